"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/hookcc_c.h declares, and fails loudly (no CPU fallback) without a GPU."""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hookcc_c.h"


def declared() -> set[str]:
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(hcc_[a-z0-9_]+)\s*\(", txt)) - {"hcc_phase_cb"}


def test_header_declares_boundary():
    d = declared()
    for must in ["hcc_create", "hcc_destroy", "hcc_graph_from_edges_u64", "hcc_graph_from_edges_u32",
                 "hcc_graph_from_csr", "hcc_graph_free", "hcc_cc", "hcc_last_error",
                 "hcc_forest_download_u64", "hcc_forest_export", "hcc_rehook"]:
        assert must in d


def test_library_exports_every_declared_symbol(capi):
    lib = capi.lib()
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(capi.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hcc_[a-z0-9_]+)", out))
    assert declared() <= exported
    # only the C-ABI leaves the library
    assert all(s.startswith("hcc_") for s in exported)


def test_binding_covers_header(capi):
    assert declared() == set(capi.exported_symbols())


def test_library_is_sm100a(capi):
    out = subprocess.run(["cuobjdump", "--list-elf", str(capi.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(capi):
    assert capi.lib().hcc_abi_version() == capi.ABI_VERSION == 4


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="GPU present")
def test_no_cpu_fallback_without_gpu(capi):
    assert capi.device_count() == 0
    with pytest.raises(capi.HccError) as ei:
        capi.Context(0)
    assert ei.value.code == capi.HCC_ENODEV


def test_choose_segment_count_matches_reference(capi):
    # engines.hpp:35-41 / test_engines.cpp:20-38 / acceptance.cpp:204-218
    def s(avg, m, n=100):
        st = capi.GraphStats(n, m, 0, avg, 0)
        return capi.lib().hcc_choose_segment_count(capi.C.byref(st))
    assert s(2.41, 1000) == 2
    assert s(2.00, 1000) == 2
    assert s(14.23, 1000) == 14
    assert s(86.82, 10000) == 87
    assert s(0.0, 0) == 1
    assert s(0.0, 0, n=0) == 1
    assert s(50.0, 7) == 7
