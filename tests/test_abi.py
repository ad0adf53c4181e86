"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and the ctypes struct matches the C layout."""

import ctypes

import numpy as np

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
    assert lib.bdem_abi_version() == L.ABI_VERSION == 7
    assert lib.bdem_system_size() == ctypes.sizeof(L.System)


def test_workspace_queries_are_host_only(lib):
    # pure size computations: no device needed
    assert lib.bdem_broadphase_workspace(1000) > 0
    assert lib.bdem_components_workspace(1000) > 0
    assert lib.bdem_select_workspace(1000) > 0
    assert lib.bdem_friction_workspace(1000, 500) > 0


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", L.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _schedule(lib, pairs, n):
    pairs = np.ascontiguousarray(pairs, dtype=np.int32)
    m = pairs.shape[0]
    order = np.full(m, -1, dtype=np.int32)
    wptr = np.zeros(m + 1, dtype=np.int32)
    vp = ctypes.c_void_p
    depth = lib.bdem_friction_schedule(pairs.ctypes.data_as(vp), m, n, order.ctypes.data_as(vp),
                                       wptr.ctypes.data_as(vp))
    return depth, order, wptr


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_friction_schedule_preserves_sweep_order(lib, seed):
    """Host wave scheduler behind bdem_friction (contact.py:332-340 sweep):
    pairs of one wave are element-disjoint, and every element meets its pairs
    in the reference's ascending pair order, so the wave execution applies
    the same corrections in the same order as the sequential sweep."""
    rng = np.random.default_rng(seed)
    n = 300
    a = rng.integers(0, n, 2000)
    b = rng.integers(0, n, 2000)
    keep = a != b
    pairs = np.sort(np.stack([a[keep], b[keep]], 1), axis=1)
    pairs = np.unique(pairs, axis=0)                       # ascending, like broad_phase
    depth, order, wptr = _schedule(lib, pairs, n)
    m = pairs.shape[0]
    assert sorted(order.tolist()) == list(range(m))
    wave = np.empty(m, dtype=np.int64)
    for w in range(depth):
        ids = order[wptr[w]:wptr[w + 1]]
        assert np.all(np.diff(ids) > 0)                    # ascending inside a wave
        ends = pairs[ids].reshape(-1)
        assert np.unique(ends).size == ends.size           # element-disjoint
        wave[ids] = w
    # minimal waves: 1 + latest wave of an earlier pair sharing an element
    last = np.full(n, -1)
    for k, (i, j) in enumerate(pairs):
        assert wave[k] == 1 + max(last[i], last[j])
        last[i] = last[j] = wave[k]
    assert wptr[depth] == m


def test_friction_schedule_edges(lib):
    assert _schedule(lib, np.zeros((0, 2)), 10)[0] == 0
    chain = np.stack([np.arange(9), np.arange(1, 10)], 1)
    assert _schedule(lib, chain, 10)[0] == 9                # a chain is sequential
    disjoint = np.stack([np.arange(0, 10, 2), np.arange(1, 10, 2)], 1)
    assert _schedule(lib, disjoint, 10)[0] == 1
    assert _schedule(lib, np.array([[0, 10]]), 10)[0] == -L.ERR_ARG   # out-of-range element


def test_graft_entry_build(lib):
    """The driver's build check: __graft_entry__.build() (incremental here)
    compiles, loads the library and checks its ABI version."""
    import importlib
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    entry = importlib.import_module("__graft_entry__")
    entry.build()


def test_rotation_free_pcg_switch(lib):
    """Host-only: the process-wide switch round-trips through the C ABI."""
    import paper_2308_10459_b200 as P
    prev = P.rotation_free_pcg(True)
    try:
        assert P.rotation_free_pcg(True) is True
    finally:
        P.rotation_free_pcg(prev)
    assert lib.bdem_pcg_set_rot_skip(-1) == int(prev)
