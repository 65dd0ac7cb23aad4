"""The render path under device-side checks (libswr_checked.so, build.py).

compute-sanitizer is closed on the GPU pool, so the checked build stands in for
memcheck / racecheck on the render kernels: every pair slot the binning writes
lies in its position's segment and the buffer, tile keys and chunk histograms
stay in range, each raster tile list lies in its segment, every accumulator
read-modify-write stays inside its half-warp's own tile copy with no two lanes
of a warp on one cell in a sweep step (the race-freedom argument of the
no-atomics raster), and residual writes stay in the work
buffer. A failed check prints its location and traps the kernel.

The GPU parity (incl. the BASELINE-sized cases), group, backward and smoke tests are re-run against the checked
library in a subprocess (a trap ends that process only), so the same cases --
multi-chunk batches, seam / full-circle boxes, tile sizes 8-32, fp16 overflow
re-runs, the host-synchronised pair path, graph capture, multi-context groups
-- run with every check on, and must still pass their parity bars.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CHECKED = os.path.join(ROOT, "paper_2506_12787_b200", "libswr_checked.so")


def test_checked_build_has_the_checks():
    assert os.path.exists(CHECKED), "build() makes libswr_checked.so next to libswr.so"
    with open(CHECKED, "rb") as fh:
        assert b"swr check failed" in fh.read()
    with open(os.path.join(ROOT, "paper_2506_12787_b200", "libswr.so"), "rb") as fh:
        assert b"swr check failed" not in fh.read()      # compiled out of the product library


def test_render_suites_under_device_checks():
    env = dict(os.environ, SWR_LIB=CHECKED)
    files = ["tests/test_gpu_parity.py", "tests/test_gpu_at_size.py", "tests/test_group.py", "tests/test_backward.py",
             "tests/test_smoke.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider"] + files,
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-4000:]
    assert "swr check failed" not in r.stdout + r.stderr, tail
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
