"""Build a variant of libswr.so with extra -D flags for one source file.

    python tools/build_variant.py OUT.so k_mlp_tc.cu[,capi.cpp,...] -DSWR_TC_NSTAGE=4 ...

The other objects come from the regular build (paper_2506_12787_b200/_build);
bench/tests pick the variant up with SWR_LIB=OUT.so.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12787_b200 import build as b  # noqa: E402

out, srcs, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
b.build()
objs = [os.path.join(b.BUILD, os.path.basename(s) + ".o") for s in b._sources() if os.path.basename(s) not in srcs]
vobjs = []
for i, src in enumerate(srcs):
    vobj = f"{out}.{i}.o"
    lang = ["-x", "cu"] if src.endswith(".cpp") else []
    r = subprocess.run([b.NVCC] + lang + defs + b._flags() + ["-c", os.path.join(b.CSRC, src), "-o", vobj],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    vobjs.append(vobj)
r = subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-cudart", "static", "-ccbin", b.HOST_CXX, "-o", out] + objs + vobjs,
                   capture_output=True, text=True)
if r.returncode:
    raise SystemExit(r.stderr)
for v in vobjs:
    os.remove(v)
print("built", out)
