import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    assert oracle.fpenv_ok(), "FTZ/DAZ set in this process: subnormal pins would be meaningless"
    return oracle


@pytest.fixture(params=["tma", "lsu"])
def step_kernel(request, monkeypatch):
    """Run a GPU parity test through both step kernels: the bulk-copy pipeline and the per-thread
    load kernel (the library picks by launch size; MPO_STEP_KERNEL forces one, read per launch)."""
    monkeypatch.setenv("MPO_STEP_KERNEL", request.param)
    return request.param


@pytest.fixture(params=["tma", "lsu"])
def p2p_kernel(request, monkeypatch):
    """Run a P2P fused-step test through both kernels (bulk-copy pipeline / per-thread loads)."""
    monkeypatch.setenv("MPO_P2P_KERNEL", request.param)
    return request.param
