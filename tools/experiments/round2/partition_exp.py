"""SM partition experiment: the tcgen05 MLP of one chunk on a
subset of SMs (CTA pairs capped, shared memory padded so no raster CTA fits beside
it) concurrent with the raster of another chunk on the remaining SMs, against the
two run back to back on the whole GPU. swr_debug_overlap: out[0] MLP alone, out[2]
raster alone (4 warps), out[4] MLP || raster (4 warps)."""
import sys, numpy as np, ctypes as C
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
for n, nb in ((10000, 1024), (50000, 256)):
    sc = make_scene(n, seed=1)
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("chunk", nb)
    swr.render(ck, random_positions(nb, seed=3), spectra=False)
    L = swr.lib()
    out = np.zeros(6)
    for K, pad in ((0, 0), (74, 32768), (56, 32768), (48, 32768), (40, 32768)):
        ck.set_option("mlp_max_clusters", K)
        ck.set_option("mlp_smem_pad", pad)
        best = None
        for _ in range(3):
            L.swr_debug_overlap(ck.handle, out.ctypes.data_as(C.c_void_p))
            best = out.copy() if best is None or out[4] < best[4] else best
        print(f"n {n} nb {nb} clusters {K or 'all'} pad {pad}: mlp {best[0]:.2f} raster {best[2]:.2f} "
              f"serial {best[0] + best[2]:.2f} concurrent {best[4]:.2f} ms", flush=True)
