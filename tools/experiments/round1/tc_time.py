"""MLP stage time (ms) of one 256-position chunk at 50k Gaussians for SWR_TC_DEBUG values.
    python tools/tc_time.py 0 507 ..."""
import os, sys, numpy as np
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(50000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", 1)
pos = random_positions(256, seed=3)
for d in sys.argv[1:]:
    os.environ["SWR_TC_DEBUG"] = d
    ck.set_option("stage_timing", 1)
    ts = []
    for _ in range(3):
        ck.set_option("stage_reset", 1)
        swr.render(ck, pos, spectra=False)
        ts.append(round(float(ck.stage_times()[1]), 3))
    ck.set_option("stage_timing", 0)
    print(f"DBG {d}: mlp ms {ts}")
