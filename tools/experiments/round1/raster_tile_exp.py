"""Raster + binning time vs the raster tile size (the render path's internal tiling;
the parity hooks keep the reference's 16). 50k Gaussians, 256 positions, bf16x3."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
pos = random_positions(256, seed=3)
for tile in (8, 16, 24, 32):
    sc = make_scene(50000, seed=1, tile=tile)
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("mlp_precision", 1)
    swr.render(ck, pos, spectra=True)
    ck.set_option("stage_timing", 1)
    ck.set_option("stage_reset", 1)
    for _ in range(3):
        swr.render(ck, pos, spectra=True)
    st = ck.stage_times() / 3
    print(f"tile {tile}: pairs/spectrum {ck.pairs_last() / 256:.0f}  ms: setup {st[2]:.3f} bin {st[3]:.3f} raster {st[4]:.3f}")
