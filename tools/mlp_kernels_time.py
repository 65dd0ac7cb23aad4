"""MLP stage time (ms, one 256-position chunk at 50k Gaussians) for each tensor-core
kernel (1 = output parts, 2 = two-tile ping-pong) and precision (1 = bf16x3, 2 = bf16)."""
import sys
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(50000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
pos = random_positions(256, seed=3)
for kern in (1, 2):
    for prec in (1, 2):
        ck.set_option("mlp_kernel", kern)
        ck.set_option("mlp_precision", prec)
        ck.set_option("stage_timing", 1)
        ts = []
        for _ in range(4):
            ck.set_option("stage_reset", 1)
            swr.render(ck, pos, spectra=False)
            ts.append(round(float(ck.stage_times()[1]), 3))
        ck.set_option("stage_timing", 0)
        print(f"kernel {kern} precision {prec}: mlp ms {ts[1:]}", flush=True)
