# Launch list of small-batch calls (B = 1 and 16, 10k Gaussians; render_device on a side stream)
cat > /tmp/small.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(10000, seed=0); ck = swr.Checkpoint.from_scene(sc)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for B in (1, 16):
    pos = torch.from_numpy(random_positions(B, seed=1)).cuda()
    sp = torch.empty((B, ck.H, ck.W, 2), device="cuda")
    for _ in range(3):
        swr.render_device(ck, pos.data_ptr(), B, swr.OUT_SPECTRA, d_spec=sp.data_ptr(), stream=st.cuda_stream)
    torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python /tmp/small.py > gpurun_out/small_ncu.log 2>&1; tail -2 gpurun_out/small_ncu.log
