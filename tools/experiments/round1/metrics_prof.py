"""swr_metrics_device on 256 device-resident pairs (ncu launch-list driver)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ck = swr.Checkpoint.from_scene(make_scene(100, seed=1))
pred = torch.rand((B, 90, 360, 2), device="cuda"); tgt = torch.rand((B, 90, 360, 2), device="cuda")
outs = [torch.empty(B, dtype=torch.float64, device="cuda") for _ in range(3)]
L = swr.lib()
for _ in range(2):
    swr._check(L.swr_metrics_device(ck.handle, pred.data_ptr(), tgt.data_ptr(), B, 1.0, outs[0].data_ptr(),
                                    outs[1].data_ptr(), outs[2].data_ptr(), None))
torch.cuda.synchronize()
print(outs[1][:4])
