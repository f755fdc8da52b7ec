"""B200-native (sm_100a) V-cycle / FMG hot path of the level-set geometric
multigrid Poisson solver of arXiv 2205.09411 (reference: C++ ``poissonmg``).

The product is ``libpmg_b200.so`` (C-ABI ``include/pmg_b200.h``); this package
holds its Python binding plus the host-side mesh mirror and the BASELINE
configuration generators.  There is no CPU fallback.
"""
from .mesh import (DIRICHLET, NEUMANN_ZERO, SHAPE_COMPOSITE_MIN, SHAPE_NONE, SHAPE_SPHERE,
                   VAR_OLD, VAR_PHI, VAR_RES, VAR_RHS, FaceBc, LevelSetSpec, TreeMesh,
                   build_uniform)
from .tree import DeviceTree
from .solver import (LAYOUT_INTERIOR, LAYOUT_PADDED, CycleStats, DeviceMesh, MgConfig, MgSolver,
                     StencilBuildConfig, StencilSet, build_stencils, error_norms, face_gradient, write_dump)

__all__ = [
    "TreeMesh", "build_uniform", "FaceBc", "LevelSetSpec", "DeviceMesh", "MgSolver", "MgConfig",
    "StencilBuildConfig", "StencilSet", "CycleStats", "build_stencils", "VAR_PHI", "VAR_RHS",
    "VAR_RES", "VAR_OLD", "DIRICHLET", "NEUMANN_ZERO", "SHAPE_SPHERE", "SHAPE_NONE",
    "SHAPE_COMPOSITE_MIN", "LAYOUT_PADDED", "LAYOUT_INTERIOR", "face_gradient", "error_norms", "write_dump",
    "DeviceTree",
]
