"""Width-512 MLP (k_mlp_wide.cu) at BASELINE config 5 (1M Gaussians x 16 positions):
MLP stage time per block size (option wide_block_rows). Smaller blocks keep the
layer-to-layer activations in L2 (2 x rows x 2 KB) at the price of more launches."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(1000000, seed=0, width=512)
ck = swr.Checkpoint.from_scene(sc)
B = 16
pos = torch.from_numpy(random_positions(B, seed=1)).cuda()
sp = torch.empty((B, sc.H, sc.W, 2), device="cuda")
st = torch.cuda.Stream()
for rows in [int(a) for a in sys.argv[1:]] or [2097152, 1048576, 524288, 262144, 151552, 75776]:
    ck.set_option("wide_block_rows", rows)
    call = lambda: swr.render_device(ck, pos.data_ptr(), B, swr.OUT_SPECTRA, sp.data_ptr(), stream=st.cuda_stream)
    call()
    torch.cuda.synchronize()
    ck.set_option("stage_timing", 1)
    ck.set_option("stage_reset", 1)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ck.set_option("stage_timing", 0)
    stg = ck.stage_times() / 3
    print(f"wide_block_rows {rows:8d}: mlp {stg[1]:8.2f} ms, step {stg.sum():8.2f} ms", flush=True)
