"""Timeline of the ping-pong MLP kernel (k_mlp_tc2.cu), CTA 0, layer steps 16..63
(super-tiles 1-3). Needs the hooks build:
    python tools/build_variant.py tools/var/hooks2.so k_mlp_tc2.cu -DSWR_TC_DEBUG_HOOKS
    SWR_LIB=tools/var/hooks2.so python tools/tc2_trace.py
Per step m: MMA warp [reached, waits passed, issued]; epilogue warp 0's
accumulator-ready time, its first chunk's TMEM load landed, its conversion stored, and
the last epilogue warp's conversion stored; cycles from the first stamp."""
import os, sys, numpy as np
sys.path.insert(0, ".")
os.environ["SWR_TC_DEBUG"] = "1"
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", int(sys.argv[1]) if len(sys.argv) > 1 else 1)
p01 = np.random.default_rng(0).random((256, 3)).astype(np.float32)
swr.predict_residuals(ck, p01)
import ctypes as C
t = np.zeros(8 * 48, np.int64)
f = swr.lib().swr_debug_mlp_trace2
f.argtypes = [C.c_void_p]
f(t.ctypes.data)
t = t.reshape(8, 48)
t0 = t[t > 0].min()
prev = None
for i in range(48):
    r = [int(x - t0) if x > 0 else -1 for x in t[:, i]]
    d = "" if prev is None else f" (+{r[2] - prev})"
    e = f" ld +{r[4] - r[3]:5d} st0 +{r[5] - r[3]:5d} st19 +{r[6] - r[3]:5d}" if r[3] >= 0 and r[5] >= 0 else ""
    print(f"step {i + 16:2d} (tile {(i + 16) % 2}, layer {((i + 16) // 2) % 8}): mma reached {r[0]:6d} waits {r[1]:6d} "
          f"issued {r[2]:6d}{d} | acc ready {r[3]:6d}{e}")
    prev = r[2]
if os.environ.get("TRACE_RAW"):
    print((t[3:7, :8] - t0).tolist())
