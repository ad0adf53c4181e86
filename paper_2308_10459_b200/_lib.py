"""ctypes binding of ``include/bdem_sm100.h`` (the C ABI of the CUDA library).

Loading fails loudly when ``lib/libbdem_sm100.so`` is missing: there is no
CPU fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes as C
import os

from ._build import lib_path

BDEM_OK = 0
ERR_DEGENERATE_BOND, ERR_ANTIPODAL, ERR_NONFINITE, ERR_ARG, ERR_CUDA, ERR_CAPACITY = 1, 2, 3, 4, 5, 6
ERRSLOT_DEG_COUNT, ERRSLOT_DEG_FIRST, ERRSLOT_ANTI_COUNT, ERRSLOT_ANTI_FIRST = 0, 1, 2, 3
ERRSLOT_COINCIDENT = 4
ERRSLOT_COUNT = 8

# bond geometry planes
BG = dict(L0=0, D0=1, FRAME=4, KN=13, KT=14, KDIAG=15, RADIUS=18, SECTION=19, SECOND=20,
          POLAR=21, TENSILE=22, SHEAR=23, COUNT=24)
BS = dict(SCALE=0, DAMAGE=1, PLASTIC=2, SIGMA=3, TAU=4, COUNT=5)
ST = dict(KC=0, GQJ=1, D=5, A=11, COUNT=17)
IP = dict(GP=0, GQ=3, P=7, R=13, E=19, COUNT=20)
ASM_STAGE_ALL_A = 1
CF = dict(N=0, ALPHA=3, BETA=4, C=5, COUNT=14)
PS = dict(E=0, GI=1, A=4, COUNT=10)
SC = dict(F=0, GNORM2=1, CNORM2=2, MAXDEV=3, SLOPE=4, FT=5, NSING=6, EBOND=7, ECOL=8, EGRAV=9,
          EKIN=10, EPAIR=11, COUNT=32)
PCG = dict(RZ=0, PAP=1, ALPHA=2, BETA=3, RR=4, BNORM=5, REL=6, TOL=7, BOOST=8, APNORM2=9,
           PNORM2=10, K=11, MAXIT=12, STATE=13, ROTZERO=14, COUNT=16)
PCG_RUNNING, PCG_CONVERGED, PCG_BREAKDOWN, PCG_MAXIT = 0, 1, 2, 3
ABI_VERSION = 7
RED_BLOCKS = 1184
MAX_COLLIDERS = 8
N_COUNTERS = 16

_p = C.c_void_p


class Collider(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("a", C.c_double * 6)]


class System(C.Structure):
    _fields_ = [
        ("n_elem", C.c_int64), ("n_free", C.c_int64), ("n_bond", C.c_int64),
        ("n_pair", C.c_int64), ("pair_cap", C.c_int64), ("vstride", C.c_int64),
        ("sell_kmax", C.c_int64), ("sell_kjmax", C.c_int64),
        ("mass", _p), ("radius", _p), ("mp_dt2", _p), ("mq_dt2", _p), ("p_hat", _p),
        ("q_hat", _p), ("slot", _p), ("free_elem", _p),
        ("bond_i", _p), ("bond_j", _p), ("status", _p), ("geom", _p), ("bstate", _p),
        ("slice_base", _p), ("pos_oslot", _p), ("jslice_base", _p), ("jpos", _p), ("jslot", _p),
        ("row_elem", _p), ("elem_row", _p), ("slice_slot", _p), ("row_slot", _p),
        ("pair_i", _p), ("pair_j", _p), ("pi_ptr", _p), ("pj_ptr", _p), ("pj_idx", _p),
        ("stage", _p), ("scoef", _p), ("pstage", _p), ("diag", _p), ("minv", _p), ("red", _p),
        ("scalars", _p), ("pcg", _p), ("err", _p), ("counter", _p), ("clamp_list", _p),
        ("ipart", _p), ("ikpre", _p), ("grad_p", _p), ("grad_q", _p),
        ("gravity", C.c_double * 3), ("k_contact", C.c_double), ("k_element", C.c_double),
        ("n_colliders", C.c_int32), ("asm_flags", C.c_int32),
        ("colliders", Collider * MAX_COLLIDERS),
    ]


_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double
_sys = C.POINTER(System)

# name -> (restype, argtypes); mirrors include/bdem_sm100.h
SIGNATURES = {
    "bdem_abi_version": (_int, []),
    "bdem_system_size": (_i64, []),
    "bdem_device_sm": (_int, []),
    "bdem_launch_count": (_i64, []),
    "bdem_pcg_spmv": (_int, [_sys, _p, _p, _p]),
    "bdem_pcg_update": (_int, [_sys, _p, _p, _p, _p, _p, _p]),
    "bdem_bond_eval_ambient": (_int, [_sys, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _int, _p]),
    "bdem_bond_assemble": (_int, [_sys, _p, _p, _p]),
    "bdem_bond_energy": (_int, [_sys, _p, _p, _int, _p]),
    "bdem_bond_update": (_int, [_sys, _p, _p, _dbl, _p, _p, _p]),
    "bdem_pair_assemble": (_int, [_sys, _p, _int, _p]),
    "bdem_element_assemble": (_int, [_sys, _p, _p, _p, _p]),
    "bdem_reduce_finish": (_int, [_sys, _int, _int, _int, _p]),
    "bdem_trial_point": (_int, [_sys, _p, _p, _p, _p, _dbl, _p, _p, _p]),
    "bdem_element_energy": (_int, [_sys, _p, _p, _int, _p]),
    "bdem_contact_blocks": (_int, [_sys, _p, _p, _p, _p]),
    "bdem_kinetic": (_int, [_sys, _p, _p, _p]),
    "bdem_normalize_free": (_int, [_sys, _p, _p]),
    "bdem_direction": (_int, [_sys, _p, _p, _dbl, _p, _p, _p]),
    "bdem_dot": (_int, [_sys, _p, _p, _i64, _int, _p]),
    "bdem_predict": (_int, [_sys, _p, _p, _p, _p, _p, _p, _dbl, _p, _p, _p, _p, _p, _p, _p]),
    "bdem_finish_step": (_int, [_sys, _p, _p, _p, _p, _dbl, _p, _p, _p]),
    "bdem_spmv": (_int, [_sys, _p, _p, _p]),
    "bdem_pcg_init": (_int, [_sys, _p, _dbl, _p, _p, _p, _p, _dbl, _int, _dbl, _p]),
    "bdem_pcg_iterate": (_int, [_sys, _p, _p, _p, _p, _p, _int, _p]),
    "bdem_precond_apply": (_int, [_sys, _p, _p, _p]),
    "bdem_broadphase_workspace": (_i64, [_i64]),
    "bdem_broadphase": (_int, [_p, _p, _i64, _dbl, _p, _p, _p, _i64, C.POINTER(C.c_int64), _p]),
    "bdem_contact_pairs": (_int, [_p, _p, _p, _dbl, _dbl, _p, _p, _p, _p,
                                  C.POINTER(C.c_int64), _p]),
    "bdem_pair_adjacency_workspace": (_i64, [_i64, _i64]),
    "bdem_set_pairs": (_int, [_p, _p, _i64, _p, _p]),
    "bdem_event_records": (_int, [_p, _p, _i64, _p, _p]),
    "bdem_rows_copy": (_int, [_p, _i64, _p, _p, _p, _p, _p, _int, _p]),
    "bdem_reset_errors": (_int, [_p, _p]),
    "bdem_components_workspace": (_i64, [_i64]),
    "bdem_components": (_int, [_i64, _i64, _p, _p, _p, _p, _p, C.POINTER(C.c_int64), _p]),
    "bdem_select_workspace": (_i64, [_i64]),
    "bdem_select_flagged": (_int, [_p, _i64, _p, _p, C.POINTER(C.c_int64), _p]),
    "bdem_pcg_set_rot_skip": (_int, [_int]),
    "bdem_friction_workspace": (_i64, [_i64, _i64]),
    "bdem_friction": (_int, [_p, _p, _p, _p, _p, _dbl, _dbl, _dbl, _p, C.POINTER(C.c_int64), _p]),
    "bdem_friction_schedule": (_i64, [_p, _i64, _i64, _p, _p]),
    "bdem_surface_workspace": (_i64, [_i64]),
    "bdem_surface": (_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i64,
                            C.POINTER(C.c_int64), _p]),
}


class BdemLibraryError(RuntimeError):
    pass


_LIB = None


def load():
    """Load and type the library (once).  Raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise BdemLibraryError(
            f"CUDA library {path} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.bdem_abi_version() != ABI_VERSION:
        raise BdemLibraryError(f"library ABI {lib.bdem_abi_version()} != expected {ABI_VERSION}; "
                               "rebuild with __graft_entry__.build()")
    if lib.bdem_system_size() != C.sizeof(System):
        raise BdemLibraryError(f"bdem_system_t size mismatch: C {lib.bdem_system_size()} "
                               f"vs ctypes {C.sizeof(System)}")
    _LIB = lib
    return lib


def check(rc: int, what: str):
    if rc != BDEM_OK:
        raise BdemLibraryError(f"{what} failed with status {rc}")


def header_symbols() -> list[str]:
    """Function names declared in include/bdem_sm100.h."""
    import re
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "include", "bdem_sm100.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(bdem_\w+)\s*\(", text, re.M)))
