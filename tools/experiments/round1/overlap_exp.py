import sys, numpy as np, ctypes as C
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(50000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", 1)
pos = random_positions(256, seed=3)
swr.render(ck, pos, spectra=False)
out = np.zeros(6)
L = swr.lib()
for _ in range(3):
    rc = L.swr_debug_overlap(ck.handle, out.ctypes.data_as(C.c_void_p))
    print(rc, "mlp %.2f r8 %.2f r4 %.2f mlp||r4 %.2f mlp||r8 %.2f nb %d" % tuple(out))
