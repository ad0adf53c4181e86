"""B200-native Newton hot path of the variational bonded discrete element
method with quaternion manifold optimisation (arXiv 2308.10459).

Drop-in for the reference package ``bdem``'s stepping API: scene and bond
topology setup, ``stable_step``, the energy/gradient/Hessian entry points and
the fracture update, all computed by hand-written sm_100a FP64 CUDA kernels
in ``lib/libbdem_sm100.so`` (C ABI: ``include/bdem_sm100.h``).
"""

from .colliders import BoxCollider, HalfSpace, SphereCollider
from .newton import (IterationRecord, LineSearchError, SolveResult, SolverConfig,
                     minimize_second_order, relative_tolerance)
from .scene import FragmentLabeling, Scene, stretch_driver, twist_driver
from .state import (BROKEN, INTACT, WEAKENED, BondSet, DegenerateBondError,
                    DegenerateShearError, ElementSet, PlasticParams)

__all__ = [
    "BondSet", "BoxCollider", "DegenerateBondError", "DegenerateShearError", "ElementSet",
    "FragmentLabeling", "HalfSpace", "IterationRecord", "LineSearchError", "PlasticParams",
    "Scene", "SolveResult", "SolverConfig", "SphereCollider", "StepReport", "broad_phase",
    "energy_terms", "label_components", "minimize_second_order", "relative_tolerance",
    "stable_step", "stretch_driver", "twist_driver", "update_bond_states",
    "rotation_free_pcg", "BROKEN", "INTACT", "WEAKENED",
    "ImplicitProblem", "PotentialBlocks", "PotentialModel", "StepContext",
    "incremental_potential",
]


def rotation_free_pcg(enabled: bool = True) -> bool:
    """Switch the exact rotation-free PCG on or off (process-wide); returns
    the previous setting.  When on, a Newton system whose right-hand side has
    an identically zero rotation half (identity orientations and no
    rotational load, e.g. the BASELINE plate) is solved on its position half
    only: the rotation halves of every PCG vector stay exactly zero, so the
    iterates are bit-identical to the full solve."""
    from . import _lib
    return bool(_lib.load().bdem_pcg_set_rot_skip(1 if enabled else 0))


def __getattr__(name):
    # GPU-facing entry points import torch lazily so host-only use stays light
    if name in ("stable_step", "StepReport", "broad_phase", "label_components",
                "update_bond_states", "contact_candidates"):
        from . import step
        return getattr(step, name)
    if name == "energy_terms":
        from .bond_api import energy_terms
        return energy_terms
    if name in ("ImplicitProblem", "PotentialBlocks", "PotentialModel", "StepContext",
                "incremental_potential"):
        from . import problem
        return getattr(problem, name)
    raise AttributeError(name)
