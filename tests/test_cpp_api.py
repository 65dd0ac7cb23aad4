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


def build_callers(out):
    cmd = ["/usr/bin/g++", "-std=gnu++20", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "ref_callers.cpp"), f"-L{PKG}", "-lswr", f"-Wl,-rpath,{PKG}", "-o", out]
    subprocess.run(cmd, check=True)


def test_cpp_api_builds(tmp_path):
    build_demo(str(tmp_path / "demo"))
    assert os.path.exists(tmp_path / "demo")


def test_reference_callers_compile_against_the_header(tmp_path):
    """train::evaluate / tasks::eval_aoa / predict_pooled / cmd_bench call shapes
    (training.cpp:387-399, tasks.cpp:54-57,176-181, wrfsplat_cli.cpp:225-237) build
    unchanged against wrfsplat::b200 with the reference's value types."""
    build_callers(str(tmp_path / "callers"))
    assert os.path.exists(tmp_path / "callers")


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


@pytest.mark.gpu
def test_reference_callers_match_python(tmp_path):
    exe = str(tmp_path / "callers")
    build_callers(exe)
    p = os.path.join(ROOT, "tests", "golden", "scene_w32.wrfc")
    pos = random_positions(3, seed=12)
    args = [exe, p] + [f"{v:.9g}" for v in pos.ravel()]
    lines = subprocess.run(args, check=True, capture_output=True, text=True).stdout.strip().splitlines()
    ck = swr.load_checkpoint(p)
    ref = swr.render(ck, pos)
    for b in range(3):
        f = lines[b].split()
        # evaluate's predict_residuals + rasterize<float> equals render_at bit for bit (psnr clamps at 100 dB)
        assert float(f[1]) == pytest.approx(float(ref["spectra"][b].astype(np.float64).sum()), rel=1e-6, abs=1e-6)
        assert float(f[2]) == 100.0
        assert (int(f[3]), int(f[4])) == tuple(ref["aoa_rc"][b])
        assert (float(f[6]), float(f[5])) == tuple(ref["aoa_ang"][b])
        assert float(f[7]) == ref["pooled"][b]
    bench = lines[3].split()
    canon = swr.render(ck, pos[:1], residuals=False)["spectra"][0]
    off, prims = swr.bins(ck, None)[0]
    assert int(bench[1]) == len(prims) == int(bench[3])
    assert float(bench[2]) == pytest.approx(float(canon.astype(np.float64).sum()), rel=1e-6, abs=1e-6)


def build_group_demo(out):
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "group_demo.cpp"), f"-L{PKG}", "-lswr", f"-Wl,-rpath,{PKG}", "-o", out]
    subprocess.run(cmd, check=True)


def test_group_demo_builds(tmp_path):
    build_group_demo(str(tmp_path / "group_demo"))
    assert os.path.exists(tmp_path / "group_demo")


@pytest.mark.gpu
@pytest.mark.parametrize("members", [1, 3])
def test_cpp_group_render_equals_single_context(tmp_path, members):
    """A C++ caller shards a batch through train::DeviceGroup (swr_group_*); the
    spectra equal one context's render_batch bit for bit."""
    exe = str(tmp_path / "group_demo")
    build_group_demo(exe)
    sc = make_scene(1200, seed=19)
    p = str(tmp_path / "g.wrfc")
    write_wrfc(p, sc)
    pos = random_positions(7, seed=21)
    out = subprocess.run([exe, p, str(members)] + [f"{v:.9g}" for v in pos.ravel()], check=True,
                         capture_output=True, text=True).stdout.strip().splitlines()
    assert len(out) == 8
    assert out[-1] == "max-diff-vs-render_batch 0"
