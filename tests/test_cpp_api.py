"""The C++ host API (include/swr.hpp) compiles against the C ABI, links libswr.so,
and (on a B200) returns the same results as the Python host."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions, write_wrfc

PKG = os.path.join(ROOT, "paper_2506_12787_b200")


def build_demo(out):
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "api_demo.cpp"),
           f"-L{PKG}", "-lswr", f"-Wl,-rpath,{PKG}", "-o", out]
    subprocess.run(cmd, check=True)


def test_cpp_api_builds(tmp_path):
    build_demo(str(tmp_path / "demo"))
    assert os.path.exists(tmp_path / "demo")


@pytest.mark.gpu
def test_cpp_api_matches_python(tmp_path):
    exe = str(tmp_path / "demo")
    build_demo(exe)
    sc = make_scene(1500, seed=9)
    p = str(tmp_path / "s.wrfc")
    write_wrfc(p, sc)
    pos = random_positions(3, seed=9)
    args = [exe, p] + [f"{v:.9g}" for v in pos.ravel()]
    out = subprocess.run(args, check=True, capture_output=True, text=True).stdout.strip().splitlines()
    ck = swr.load_checkpoint(p)
    ref = swr.render(ck, pos)
    for b in range(3):
        idx, tot, pooled, row, col = out[b].split()
        assert float(tot) == pytest.approx(float(ref["spectra"][b].astype(np.float64).sum()), rel=1e-6, abs=1e-6)
        assert float(pooled) == pytest.approx(ref["pooled"][b], rel=1e-9)
        assert (int(row), int(col)) == tuple(ref["aoa_rc"][b])
    assert float(out[3].split()[1]) <= 1e-5
