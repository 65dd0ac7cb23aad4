"""CPU tests of the drop-in boundary: libswr.so loads, exports every entry
point include/swr.h declares, and refuses to run without an sm_100 device
(no CPU fallback exists)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, write_wrfc


def declared():
    text = open(os.path.join(ROOT, "include", "swr.h")).read()
    return sorted(set(re.findall(r"\b(swr_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(swr.LIB_PATH)
    names = declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "swr.h"\nint main(void){return swr_version() > 0 ? 0 : 1;}\n')
    r = os.system(f"/usr/bin/gcc -std=c99 -fsyntax-only -I{ROOT}/include {src}")
    assert r == 0


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="only meaningful without a GPU")
def test_fails_loudly_without_device(tmp_path):
    sc = make_scene(32, seed=1, width=8, H=16, W=32)
    p = str(tmp_path / "s.wrfc")
    write_wrfc(p, sc)
    with pytest.raises(swr.SwrError):
        swr.load_checkpoint(p)
    with pytest.raises(swr.SwrError):
        swr.Checkpoint.from_scene(sc)


def test_bad_checkpoint_is_runtime_error(tmp_path):
    p = tmp_path / "bad.wrfc"
    p.write_bytes(b"WRFX" + b"\0" * 60)
    with pytest.raises(swr.SwrError, match="bad magic|sm_100|device"):
        swr.load_checkpoint(str(p))


def test_host_side_validation_needs_no_device(tmp_path):
    """Argument checks of the newer entry points run before any CUDA call and map
    to the reference's exception types (invalid_argument -> SWR_EINVAL)."""
    lib = swr.lib()
    out = C.c_void_p()
    # steering: non-square arrays, empty grids (wavesim.cpp:11-19, 185-186)
    assert lib.swr_steering_create(15, 0.0625, 0.125, 10, 10, 0, C.byref(out)) == 1
    assert lib.swr_steering_create(16, 0.0625, 0.125, 0, 10, 0, C.byref(out)) == 1
    assert lib.swr_steering_create(81, 0.0625, 0.125, 10, 10, 0, C.byref(out)) == 1
    # trainer: null arguments
    cfg = swr.TrainConfig()
    assert cfg.width == 156 and cfg.primitives == 10000 and cfg.coarse_iters == 10000
    assert lib.swr_trainer_create(C.byref(cfg), None, None, 0, C.byref(out)) == 1
    # dataset: missing directory -> runtime_error (SWR_ERUNTIME)
    assert lib.swr_dataset_open(str(tmp_path / "nope").encode(), C.byref(out)) == 2
    with pytest.raises(TypeError):
        swr.TrainConfig(not_a_field=1)


def test_wrfc_peek_reads_rssi_calibration_without_a_device():
    """The trailer of an RSSI model written by the reference's save_rssi_model
    (tasks.cpp:131-137) carries the affine calibration load_rssi_model reads
    (tasks.cpp:139-150); a plain checkpoint has none."""
    gold = os.path.join(ROOT, "tests", "golden")
    m = swr.wrfc_peek(os.path.join(gold, "rssi_model_w32.wrfc"))
    assert m["rssi_cal"] == (17.25, -58.5)
    assert (m["H"], m["W"], m["n"], m["width"]) == (90, 360, 600, 32)
    assert swr.wrfc_peek(os.path.join(gold, "scene_w32.wrfc"))["rssi_cal"] is None
    with pytest.raises(swr.SwrError):
        swr.wrfc_peek(os.path.join(gold, "make_golden.py"))
