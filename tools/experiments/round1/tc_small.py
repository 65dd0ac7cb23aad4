import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
import oracle as O
sc = make_scene(int(sys.argv[2]) if len(sys.argv) > 2 else 40, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", int(sys.argv[1]) if len(sys.argv) > 1 else 1)
port = O.Port(sc)
pos = random_positions(int(sys.argv[3]) if len(sys.argv) > 3 else 8, seed=3)
p01 = np.stack([port.normalize(p) for p in pos])
got = swr.predict_residuals(ck, p01)
want = port.predict(p01[0], precise=True)
print("dc", got.d_center[0][:3], want[0][:3])
print("max rel", [float(np.abs(g-w).max()/np.abs(w).max()) for g, w in zip((got.d_center[0], got.d_response[0], got.d_atten[0]), want)])
