"""Load golden fixtures into host containers (shared by CPU and GPU tests)."""

import os

import numpy as np

from paper_2308_10459_b200.state import BondSet, ElementSet

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BOND_FIELDS = ("i", "j", "rest_length", "radius", "d0", "q0", "frame", "kn", "kt", "k_diag",
               "section", "second_moment", "polar_moment", "tensile_strength",
               "shear_strength", "status", "stiffness_scale", "damage", "plastic_strain",
               "sigma", "tau")
ELEM_FIELDS = ("p", "q", "v", "qdot", "mass", "radius", "pinned")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def bonds_from(d, prefix):
    return BondSet(**{f: np.array(d[prefix + f]) for f in BOND_FIELDS})


def elements_from(d, prefix):
    return ElementSet(*(np.array(d[prefix + f]) for f in ELEM_FIELDS))


def close(a, b, rtol, atol):
    """max |a-b| - (atol + rtol |b|) <= 0, with the worst offender for messages."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    assert a.shape == b.shape, (a.shape, b.shape)
    err = np.abs(a - b) - (atol + rtol * np.abs(b))
    k = int(np.argmax(err)) if err.size else 0
    ok = (not err.size) or err.flat[k] <= 0
    return ok, (a.flat[k] if err.size else None, b.flat[k] if err.size else None, k)
