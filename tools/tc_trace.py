import ctypes, os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["SWR_TC_DEBUG"] = os.environ.get("DBG", "8")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", int(sys.argv[1]) if len(sys.argv) > 1 else 1)
pos = random_positions(64, seed=3)
p01 = swr.normalize_position(ck, pos)
swr.predict_residuals(ck, p01)
t = np.zeros(3 * 8 * 80, np.int64)
swr.lib().swr_debug_mlp_trace(t.ctypes.data)
t = t.reshape(3, 8, 80)
t0 = t[t > 0].min()
for it in range(3):
    for l in range(1, 8):
        row = t[it, l]
        rel = lambda x: (int(x - t0) if x > 0 else -1)
        mma = [rel(x) for x in row[:11]]
        wake = [rel(x) for x in row[16:32]]
        chunks = [max(rel(x) for x in row[32 + 4 * c:36 + 4 * c]) for c in range(5)]
        print(f"tile {it} L{l}: mma k-issue {mma[:5]} commit {mma[10]}")
        print(f"          epi wake min/max {min(w for w in wake if w>=0) if any(w>=0 for w in wake) else -1}/{max(wake)} chunk ready {chunks}")
