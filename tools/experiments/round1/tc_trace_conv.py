import os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["SWR_TC_DEBUG"] = os.environ.get("DBG", "8")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", 1)
p01 = np.random.default_rng(0).random((64, 3)).astype(np.float32)
swr.predict_residuals(ck, p01)
t = np.zeros(3 * 8 * 128, np.int64)
swr.lib().swr_debug_mlp_trace(t.ctypes.data)
t = t.reshape(3, 8, 128)
for l in (2, 3, 4):
    row = t[2, l]
    print(f"L{l}: per warp (first chunk): wait-done -> ld done / st done / arrived (cycles after wait)")
    for e in range(20):
        w = row[16 + e]
        if w > 0:
            print(f"  e{e:2d} grp{4 - (e >> 2)}: {row[56+e]-w:6d} {row[76+e]-w:6d} {row[36+e]-w:6d}")
