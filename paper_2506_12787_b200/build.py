"""Build libswr.so in-tree (nvcc, sm_100a only).

    python -m paper_2506_12787_b200.build          # or __graft_entry__.build()

Every .cu/.cpp under csrc/ is compiled with
`-gencode arch=compute_100a,code=sm_100a -lineinfo -O3` (host code with
-ffp-contract=off) and linked into paper_2506_12787_b200/libswr.so, which is
what the Python host (swr.py), the C++ wrapper (include/swr.hpp) and the
bench load. Objects go to paper_2506_12787_b200/_build/.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libswr.so")
BUILD = os.path.join(PKG, "_build")
# checked build: the same library with the device-side SWR_DCHECK bounds / race
# checks compiled in (tests/test_checked.py runs render cases against it)
OUT_CHECKED = os.path.join(PKG, "libswr_checked.so")
BUILD_CHECKED = os.path.join(PKG, "_build_checked")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
JSON_INC = os.environ.get(
    "SWR_JSON_INC",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_CXX = "/usr/bin/g++"


def _flags():
    extra = ["-DSWR_TC_DEBUG_WAITS"] if os.environ.get("SWR_DEBUG_WAITS") else []
    return extra + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
                   "-ccbin", HOST_CXX, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", JSON_INC,
                   "-Xptxas", "-v" if os.environ.get("SWR_PTXAS_V") else "-O3"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _digest(path: str, flags) -> str:
    h = hashlib.sha1(" ".join(flags).encode())
    for f in [path] + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))):
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _compile(src: str, flags, build_dir: str = BUILD) -> str:
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    stamp = obj + ".sha"
    dig = _digest(src, flags)
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == dig:
        return obj
    cmd = [NVCC] + flags + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-x", "cu"] + flags + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("SWR_PTXAS_V"):
        sys.stderr.write(r.stderr)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return obj


def _link(out: str, objs) -> None:
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(out) or os.path.getmtime(out) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-ccbin", HOST_CXX, "-o", out] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")


def _uses_checks(src: str) -> bool:
    with open(src) as fh:
        return "SWR_DCHECK(" in fh.read()


def build(verbose: bool = False, checked: bool = True) -> str:
    """libswr.so, and (checked=True) libswr_checked.so: the sources that hold device
    checks recompiled with -DSWR_CHECKED, linked with the other objects."""
    os.makedirs(BUILD, exist_ok=True)
    flags = _flags()
    srcs = _sources()
    jobs = [(s, flags, BUILD) for s in srcs]
    chk = [s for s in srcs if _uses_checks(s)] if checked else []
    if chk:
        os.makedirs(BUILD_CHECKED, exist_ok=True)
        jobs += [(s, ["-DSWR_CHECKED"] + flags, BUILD_CHECKED) for s in chk]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        objs = list(ex.map(lambda j: _compile(*j), jobs))
    _link(OUT, objs[:len(srcs)])
    if chk:
        repl = dict(zip(chk, objs[len(srcs):]))
        _link(OUT_CHECKED, [repl.get(s, o) for s, o in zip(srcs, objs[:len(srcs)])])
    if verbose:
        print(f"built {OUT}" + (f" and {OUT_CHECKED}" if chk else ""))
    return OUT


if __name__ == "__main__":
    build(verbose=True)
