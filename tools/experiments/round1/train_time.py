"""Training-loop timing (GPU box): iterations/s of the coarse and fine stages at
the reference's default TrainConfig (10000 primitives, width 156) on a 90x360
dataset simulated by the reference, vs the reference's own train() on the host."""
import os, sys, time, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ref_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
prims = int(os.environ.get("PRIMS", "10000"))
d = tempfile.mkdtemp()
t0 = time.time()
O.make_dataset(d, 90, 360, 24, 3)
print(f"dataset: {time.time() - t0:.1f} s")
ds = swr.Dataset(d)
for stage in ("coarse", "fine"):
    kw = dict(primitives=prims, coarse_iters=iters if stage == "coarse" else 0,
              fine_iters=iters if stage == "fine" else 0, anneal_threshold=10000)
    tr = swr.Trainer(swr.TrainConfig(**kw), ds)
    tr.run(5)  # warm-up (allocations, first pair counts)
    t0 = time.perf_counter()
    log, ms = tr.run(iters - 5)
    wall = time.perf_counter() - t0
    print(f"GPU {stage}: {(iters - 5) / wall:.1f} it/s wall, {(iters - 5) / (ms / 1e3):.1f} it/s device "
          f"({ms / (iters - 5):.3f} ms/it), loss {log[0, 0]:.4f} -> {log[-1, 0]:.4f}")
if "--ref" in sys.argv:
    ref = O.Reference(scene=make_scene(4, seed=1, H=12, W=16, width=24))
    for stage in ("coarse", "fine"):
        c = swr.TrainConfig(primitives=prims, coarse_iters=ref_iters if stage == "coarse" else 0,
                            fine_iters=ref_iters if stage == "fine" else 0, anneal_threshold=10000)
        t0 = time.perf_counter()
        ref.train(d, c)
        wall = time.perf_counter() - t0
        print(f"reference CPU {stage}: {ref_iters / wall:.2f} it/s ({os.cpu_count()} host threads)")
