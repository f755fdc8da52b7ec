"""K5: GPU stencil build vs the reference's build_stencils (stencil.hpp:207-222).

Interface flags, row_of patterns, masks, pin/obj ids, cut distances and
coefficients must be BIT-EXACT (north star).  The heart and
astroid shapes go through cbrt, which neither glibc nor CUDA rounds correctly:
for those the patterns must still match and the values agree to 1e-12.
"""
import numpy as np
import pytest

from oracle.oc import Oracle
from paper_2205_09411_b200 import DeviceMesh, StencilBuildConfig, build_stencils, build_uniform
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import (SHAPE_ASTROID, SHAPE_COMPOSITE_MIN, SHAPE_HEART,
                                        SHAPE_NONE, SHAPE_RHOMBUS, SHAPE_ROD, SHAPE_SPHERE,
                                        SHAPE_SPHEROID, LevelSetSpec)

pytestmark = pytest.mark.gpu

KEYS_EXACT = ["boundary", "row_count", "row_of", "mask", "pin_obj", "obj", "lin"]
KEYS_VAL = ["center", "nb", "bc", "d"]


def _compare(mesh, lsf, cfg, lo, hi, exact_values=True):
    dev = DeviceMesh(mesh)
    a = build_stencils(dev, lsf, cfg)
    o = Oracle(mesh.dim, mesh.N, lo, hi)
    o.build_uniform(mesh.n_levels)
    assert o.n_blocks == mesh.n_blocks
    o.build_stencils(lsf.as_descs(), eps_tol=cfg.eps_tol, max_bracket_iters=cfg.max_bracket_iters,
                     d_min=cfg.d_min, w_min=cfg.w_min, boundary_safety=cfg.boundary_safety,
                     thin_rescue=cfg.thin_rescue)
    b = o.get_stencils()
    for k in KEYS_EXACT:
        assert np.array_equal(np.asarray(a[k]).reshape(-1), np.asarray(b[k]).reshape(-1)), k
    for k in KEYS_VAL:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if exact_values:
            assert np.array_equal(x, y), (k, np.max(np.abs(x - y)) if x.size else 0)
        else:
            assert np.allclose(x, y, rtol=1e-12, atol=0), k
    return a


@pytest.mark.parametrize("name", ["cfg1", "cfg2@4", "cfg2", "cfg4@5", "cfg5@4"])
def test_config_stencils_bit_exact(name):
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    st = _compare(mesh, case.lsf, StencilBuildConfig(w_min=case.w_min), case.lo[:case.dim],
                  case.hi[:case.dim])
    assert st.n_rows > 0


def test_amr_stencils_bit_exact():
    case = cfgs.get_case("cfg3@6")
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    a = build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    from helpers import oracle_for_case
    o = oracle_for_case(case, mesh)
    o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)
    b = o.get_stencils()
    for k in KEYS_EXACT + KEYS_VAL:
        assert np.array_equal(np.asarray(a[k]).reshape(-1), np.asarray(b[k]).reshape(-1)), k


def test_thin_rescue_virtual_boundary():
    """test_multigrid.cpp:539-561: an unresolved R=5e-3 sphere on an 8^3 grid
    gets a virtual boundary from the thin-object rescue."""
    mesh = build_uniform(3, (-0.5,) * 3, (0.5,) * 3, 8, 1)
    lsf = LevelSetSpec(shape=SHAPE_SPHERE, center=(0, 0, 0), radius=5e-3, boundary_value=1.0)
    st = _compare(mesh, lsf, StencilBuildConfig(w_min=1e-3), (-0.5,) * 3, (0.5,) * 3)
    assert np.any(np.asarray(st["d"]) < 1.0)


SHAPES_2D = [SHAPE_SPHEROID, SHAPE_RHOMBUS, SHAPE_HEART, SHAPE_ASTROID]


@pytest.mark.parametrize("shape", SHAPES_2D)
def test_sharp_shapes_2d(shape):
    mesh = build_uniform(2, (0, 0), (1, 1), 8, 5)
    lsf = LevelSetSpec(shape=shape, boundary_value=1.0)
    exact = shape not in (SHAPE_HEART, SHAPE_ASTROID)
    _compare(mesh, lsf, StencilBuildConfig(w_min=4e-3), (0, 0), (1, 1), exact_values=exact)


@pytest.mark.parametrize("shape", [SHAPE_SPHEROID, SHAPE_RHOMBUS])
def test_cylindrical_shapes_3d(shape):
    mesh = build_uniform(3, (0,) * 3, (1,) * 3, 8, 4)
    lsf = LevelSetSpec(shape=shape, boundary_value=1.0, cylindrical=True)
    _compare(mesh, lsf, StencilBuildConfig(w_min=8e-3), (0,) * 3, (1,) * 3)


def test_two_electrodes_composite():
    """harness two_electrodes geometry (harness.hpp:381-420): rod + sphere."""
    mesh = build_uniform(3, (0,) * 3, (1,) * 3, 8, 4)
    rod = LevelSetSpec(shape=SHAPE_ROD, radius=0.05, boundary_value=1.0,
                       seg_a=(0.5, 0.5, 1.0), seg_b=(0.5, 0.5, 0.8))
    sph = LevelSetSpec(shape=SHAPE_SPHERE, radius=0.25, center=(0.5, 0.5, 0.0),
                       boundary_value=0.0)
    lsf = LevelSetSpec(shape=SHAPE_COMPOSITE_MIN, children=[rod, sph])
    _compare(mesh, lsf, StencilBuildConfig(w_min=1.0 / 64), (0,) * 3, (1,) * 3)


def test_no_boundary():
    mesh = build_uniform(2, (0, 0), (1, 1), 8, 3)
    st = _compare(mesh, LevelSetSpec(shape=SHAPE_NONE), StencilBuildConfig(), (0, 0), (1, 1))
    assert st.n_rows == 0
