"""Shared pytest configuration.

Markers:
  gpu — needs a B200 (sm_100) GPU; deselect with -m "not gpu" on CPU boxes.
The CPU suite checks the oracle against the reference's golden vectors and
the reference library itself, the host logic, and that the C-ABI library
loads and exports every symbol include/hookcc_c.h declares.
"""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    if not O.ORACLE_SO.exists():
        O.build()
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle


@pytest.fixture(scope="session")
def capi():
    from paper_1612_01178_b200 import capi as C
    C.lib()  # fails loudly when the library is missing
    return C


@pytest.fixture(scope="session")
def ctx(capi):
    if capi.device_count() == 0:
        pytest.fail("no sm_100 GPU visible: the gpu tests need a B200 (no CPU fallback)")
    c = capi.Context(0)
    yield c
    c.close()
