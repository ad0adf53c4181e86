"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and the ctypes struct matches the C layout."""

import ctypes

import pytest

from paper_2308_10459_b200 import _lib as L


@pytest.fixture(scope="module")
def lib():
    return L.load()


def test_exports_every_header_symbol(lib):
    syms = L.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(L.SIGNATURES), set(syms) ^ set(L.SIGNATURES)


def test_struct_layout_and_version(lib):
    assert lib.bdem_abi_version() == 1
    assert lib.bdem_system_size() == ctypes.sizeof(L.System)


def test_workspace_queries_are_host_only(lib):
    # pure size computations: no device needed
    assert lib.bdem_broadphase_workspace(1000) > 0
    assert lib.bdem_components_workspace(1000) > 0
    assert lib.bdem_select_workspace(1000) > 0


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", L.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
