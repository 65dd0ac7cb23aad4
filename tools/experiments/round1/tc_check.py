"""Tensor-core MLP vs the FP64 oracle over every (Gaussian, position) of a small case.
    python tools/tc_check.py PRECISION N B"""
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
import oracle as O
prec, n, b = (int(x) for x in sys.argv[1:4])
sc = make_scene(n, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", prec)
port = O.Port(sc)
pos = random_positions(b, seed=3)
p01 = np.stack([port.normalize(p) for p in pos])
got = swr.predict_residuals(ck, p01)
worst = 0.0
for s in range(b):
    want = port.predict(p01[s], precise=True)
    for g, w in zip((got.d_center[s], got.d_response[s], got.d_atten[s]), want):
        worst = max(worst, float(np.abs(np.asarray(g) - w).max() / max(np.abs(w).max(), 1e-30)))
print(f"prec {prec} n {n} b {b}: max rel {worst:.3g}")
