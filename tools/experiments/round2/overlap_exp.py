"""MLP || raster co-residency experiment (swr_debug_overlap): times the MLP alone,
the raster alone (8- and 4-warp CTAs) and both launched on two streams."""
import sys, numpy as np, ctypes as C
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
for n, nb in ((50000, 256), (10000, 256)):
    sc = make_scene(n, seed=1)
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("chunk", nb)
    pos = random_positions(nb, seed=3)
    swr.render(ck, pos, spectra=False)
    out = np.zeros(6)
    L = swr.lib()
    for _ in range(3):
        rc = L.swr_debug_overlap(ck.handle, out.ctypes.data_as(C.c_void_p))
        print(n, rc, "mlp %.2f r2 %.2f r4 %.2f mlp||r2 %.2f mlp||r4 %.2f nb %d" % tuple(out), flush=True)
