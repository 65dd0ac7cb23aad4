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
