"""Per-stage timeline of the tensor-core MLP kernel (block 0), SWR_TC_DEBUG bit 8.
    DBG=8 python tools/tc_trace.py [precision]"""
import os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["SWR_TC_DEBUG"] = os.environ.get("DBG", "8")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", int(sys.argv[1]) if len(sys.argv) > 1 else 1)
p01 = np.random.default_rng(0).random((64, 3)).astype(np.float32)
swr.predict_residuals(ck, p01)
t = np.zeros(3 * 9 * 128, np.int64)
swr.lib().swr_debug_mlp_trace(t.ctypes.data)
t = t.reshape(3, 9, 128)
t0 = t[2][t[2] > 0].min()
rel = lambda x: (int(x - t0) if x > 0 else -1)
part = lambda c: 0 if c < 6 else 1
print("MMA per part: wait-start / w done / issued.  epilogue per part: [first wait done .. last conv done] (max conv duration)")
for l in range(9):
    row = t[2, l]
    parts = [f"p{p}:{rel(row[100+p])}/{rel(row[104+p])}/{rel(row[108+p])}" for p in range(2)]
    ep = {0: [], 1: [], 2: []}
    for e in range(20):
        grp = 4 - (e >> 2)
        for c, ws, cd in ((grp, 16, 36), (grp + 5, 56, 76)):
            if row[ws + e] > 0:
                ep[part(c)].append((rel(row[ws + e]), rel(row[cd + e])))
    es = []
    for p in range(3):
        if ep[p]:
            es.append(f"e{p}:[{min(x for x, _ in ep[p])}..{max(y for _, y in ep[p])}]({max(y - x for x, y in ep[p])})")
    print(f"L{l}: " + " ".join(parts) + " | " + " ".join(es))
