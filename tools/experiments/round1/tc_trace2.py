"""Timeline of the tensor-core MLP kernel, CTA 0, local tile 2 (SWR_TC_DEBUG=8 clock64 stamps).
Needs a build with hooks: python tools/build_variant.py tools/var/hooks.so k_mlp_tc.cu -DSWR_TC_DEBUG_HOOKS, then SWR_LIB=tools/var/hooks.so.
Per layer and output part p: MMA [stage wait start, stage landed, part issued]; epilogue:
for the warps converting part p, [first acc seen .. last acc seen] -> [first .. last converted].
Cycles from the tile's first stamp."""
import os, sys, numpy as np
sys.path.insert(0, ".")
os.environ["SWR_TC_DEBUG"] = "8"
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene
NGRP, NPART = 6, 2
part = lambda c: 0 if c < 6 else 1
sc = make_scene(20000, seed=1)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("mlp_precision", 1)
p01 = np.random.default_rng(0).random((64, 3)).astype(np.float32)
swr.predict_residuals(ck, p01)
t = np.zeros(3 * 9 * 128, np.int64)
swr.lib().swr_debug_mlp_trace(t.ctypes.data)
t = t.reshape(3, 9, 128)
it = 2
t0 = t[it][t[it] > 0].min()
r = lambda x: int(x - t0) if x > 0 else -1
for l in range(9):
    row = t[it, l]
    print(f"L{l}")
    for p in range(NPART):
        mm = f"mma [{r(row[112+p])},{r(row[116+p])},{r(row[120+p])}]"
        acc, conv = [], []
        for e in range(4 * NGRP):
            g = NGRP - 1 - (e >> 2)
            for c, ws, cd in ((g, 16, 40), (g + NGRP, 64, 88)):
                if c < 10 and part(c) == p and row[ws + e] > 0:
                    acc.append(row[ws + e]); conv.append(row[cd + e])
        ep = f"epi acc {r(min(acc))}..{r(max(acc))} conv {r(min(conv))}..{r(max(conv))}" if acc else ""
        print(f"   p{p}: {mm} {ep}")
