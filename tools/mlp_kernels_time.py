"""MLP stage time (ms, one 256-position chunk at 50k Gaussians) of the tensor-core
kernel per precision (1 = fp16x3, 2 = fp16) and the FP32 kernel (0). SWR_LIB
selects a variant build (tools/build_variant.py)."""
import os
import sys
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(int(os.environ.get("N", 50000)), seed=1)
ck = swr.Checkpoint.from_scene(sc)
pos = random_positions(256, seed=3)
precs = [int(p) for p in os.environ.get("PRECS", "1,2").split(",")]
for prec in precs:
    ck.set_option("mlp_precision", prec)
    ck.set_option("stage_timing", 1)
    ts = []
    for _ in range(5):
        ck.set_option("stage_reset", 1)
        swr.render(ck, pos, spectra=False)
        ts.append(round(float(ck.stage_times()[1]), 3))
    ck.set_option("stage_timing", 0)
    print(f"{os.environ.get('SWR_LIB', 'default')} precision {prec}: mlp ms {ts[1:]}", flush=True)
