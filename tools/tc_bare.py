import os, sys, numpy as np
sys.path.insert(0, ".")
os.environ["SWR_TC_DEBUG"] = os.environ.get("DBG", str(2048 | 507))
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", 1)
p01 = np.random.default_rng(0).random((64, 3)).astype(np.float32)
swr.predict_residuals(ck, p01)
t = np.zeros(3 * 8 * 80, np.int64)
swr.lib().swr_debug_mlp_trace(t.ctypes.data)
print("bare pattern in kernel: cycles/layer", t[0] / 200)
