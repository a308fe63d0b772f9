"""The driver's round-end smoke() must pass on the GPU (it runs it verbatim)."""
import pytest


@pytest.mark.gpu
def test_graft_entry_smoke(cuda):
    import __graft_entry__
    __graft_entry__.smoke()
