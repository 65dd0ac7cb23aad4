SWR_LIB=tools/var/hooks.so timeout 120 python tools/tc_time.py 0 1 2 3
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
sc = make_scene(50000, seed=1); ck = swr.Checkpoint.from_scene(sc); pos = random_positions(256, seed=3)
for prec in (1, 2):
    ck.set_option('mlp_precision', prec); ck.set_option('stage_timing', 1); ts=[]
    for _ in range(3):
        ck.set_option('stage_reset', 1); swr.render(ck, pos, spectra=False); ts.append(round(float(ck.stage_times()[1]),3))
    print('precision', prec, ts)
"
