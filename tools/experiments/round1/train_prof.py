"""A few coarse + fine training iterations for an ncu launch list (GPU box)."""
import os, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O
from paper_2506_12787_b200 import swr

d = tempfile.mkdtemp()
O.make_dataset(d, 90, 360, 24, 3)
ds = swr.Dataset(d)
stage = sys.argv[1] if len(sys.argv) > 1 else "coarse"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kw = dict(primitives=10000, coarse_iters=n_it if stage == "coarse" else 0, fine_iters=n_it if stage == "fine" else 0)
tr = swr.Trainer(swr.TrainConfig(**kw), ds)
log, ms = tr.run()
print(stage, log[:, 0], ms)
