"""Shared test fixtures: the same seeded problem on the CPU oracle and the GPU."""
from __future__ import annotations

import os

import numpy as np

from oracle.oc import PORT_SO, REF_SO, Oracle
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS

ORACLES = [w for w, p in (("ref", REF_SO), ("port", PORT_SO)) if os.path.exists(p)]


def oracle_for_case(case, mesh, which="ref"):
    o = Oracle(case.dim, case.N, case.lo[:case.dim], case.hi[:case.dim], which)
    o.build_uniform(case.levels)
    if case.amr_band > 0:
        o.refine_band(case.refine_lsf.as_descs(), case.amr_band, case.max_level)
    assert o.n_blocks == mesh.n_blocks
    for d in range(2 * case.dim):
        o.set_face_bc(d, 0, 0.0)
    return o


def stencil_kwargs(case):
    return dict(w_min=case.w_min)


def interior(o, var, dim, N):
    return cfgs.interior_from_padded(o.get_field(var), dim, N)


def setup_pair(case, which="ref", gpu_stencils=False, rhs=None, phi=None, mg=None, threads=1):
    """Returns (oracle, DeviceMesh, MgSolver, mesh, stencils) with identical inputs."""
    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig
    from paper_2205_09411_b200 import build_stencils as gpu_build
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR, StencilSet

    mesh = case.build_mesh()
    o = oracle_for_case(case, mesh, which)
    o.build_stencils(case.lsf.as_descs(), **stencil_kwargs(case))
    dev = DeviceMesh(mesh)
    if gpu_stencils:
        st = gpu_build(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    else:
        st = StencilSet(o.get_stencils())
        st["phi_b"] = np.array([case.lsf.object(i).boundary_value
                                for i in range(case.lsf.n_objects())], np.float64)
    g = case.rhs_fields(mesh) if rhs is None else rhs
    dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
    o.set_field(VAR_RHS, cfgs.padded_from_interior(g, case.dim, case.N))
    if phi is not None:
        dev.set_field(VAR_PHI, phi, layout=LAYOUT_INTERIOR)
        o.set_field(VAR_PHI, cfgs.padded_from_interior(phi, case.dim, case.N))
    mgc = mg or MgConfig()
    o.solver_create(mgc.n_down, mgc.n_up, mgc.coarse_rel_tol, mgc.coarse_max_iters, threads)
    sol = MgSolver(dev, st, mgc)
    return o, dev, sol, mesh, st


def max_rel_diff(a, b):
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)


def resid_tol(r_ref, max_phi, dx_fine, dim):
    """|dr| <= 1e-6 r + 16 eps (2D/dx^2) max|phi|."""
    return 1e-6 * r_ref + 16 * 2.2e-16 * (2 * dim / dx_fine ** 2) * max_phi
