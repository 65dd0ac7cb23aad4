import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libswr.so")


def _ensure_built():
    oracle_so = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(oracle_so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if os.path.isdir("/root/reference/proj/src") and not os.path.exists(
            os.path.join(ROOT, "oracle", "_ref", "libwrfref.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2506_12787_b200", "libswr.so")):
        from paper_2506_12787_b200 import build
        build.build()


_ensure_built()


def has_ref():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libwrfref.so"))


@pytest.fixture(scope="session")
def tmpdir_session(tmp_path_factory):
    return tmp_path_factory.mktemp("swr")
