"""Render-backward timing + error report (GPU box): B positions at the bench
scene (config 2), residuals from the MLP, upstream = hybrid-loss gradient."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
sc = make_scene(n, seed=1)
ck = swr.Checkpoint.from_scene(sc)
pos = random_positions(B, seed=3)
p01 = swr.normalize_position(ck, pos)
res = swr.predict_residuals(ck, p01)
pred = swr.rasterize(ck, res)
target = np.roll(pred, 5, axis=1)
terms, g = swr.hybrid_loss(ck, pred, target, 0.8)
for it in range(2):
    t0 = time.perf_counter()
    out = swr.rasterize_backward(ck, g, res)
    t1 = time.perf_counter()
    terms, g = swr.hybrid_loss(ck, pred, target, 0.8)
    t2 = time.perf_counter()
print(f"n={n} B={B}: rasterize_backward {1e3*(t1-t0):.1f} ms ({B/(t1-t0):.0f} pos/s incl. copies), "
      f"hybrid_loss {1e3*(t2-t1):.1f} ms")
if os.path.exists(O.REF_SO) and "--check" in sys.argv:
    ref = O.Reference(sc)
    for b in range(min(B, 2)):
        want = ref.rasterize_backward(g[b], (res.d_center[b], res.d_response[b], res.d_atten[b]))
        for k, _ in swr.GRAD_FIELDS:
            sc_ = max(1e-3, float(np.abs(want[k]).max()))
            print(f"  b={b} {k:12s} max|ref|={sc_:.3e} rel err={float(np.abs(out[k][b]-want[k]).max())/sc_:.2e}")
