"""pytest configuration: the `gpu` marker and repo-root imports.

CPU tests (-m "not gpu") exercise the oracle against the reference's golden
values, the host-side logic and the C ABI's symbol table; GPU tests (-m gpu)
call the CUDA library through the C ABI and compare with the oracle.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    pyoracle.lib()
    return pyoracle


@pytest.fixture(scope="session")
def pcs():
    if not _has_gpu():
        pytest.skip("no CUDA device")
    import paper_1812_08491_b200 as pcs
    pcs.library()
    return pcs
