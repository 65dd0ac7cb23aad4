"""The driver's round-end smoke entry point (__graft_entry__.smoke) runs clean."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__ as g
    g.smoke()
