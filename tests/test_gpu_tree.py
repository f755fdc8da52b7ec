"""the block tree built, refined and 2:1-balanced on the device
(csrc/tree.cu, pmg_b200_tree_*) against the reference's TreeMesh
(mesh.hpp:157-320, 429-469) and refine_by_criterion (harness.hpp:295-321).

Block ids, geometry, parent / children, the level lists and both neighbour
tables must be IDENTICAL to the reference's: the ids are the order of the
reference's depth-first balancing recursion, which the device reproduces from
sorted discovery keys (tests/test_tree_model.py pins that statement on CPU).
"""
import os

import numpy as np
import pytest

from oracle.oc import REF_SO, Oracle
from paper_2205_09411_b200 import (DeviceMesh, DeviceTree, MgConfig, MgSolver, StencilBuildConfig,
                                   build_stencils)
from paper_2205_09411_b200 import _lib
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS, TreeMesh
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

pytestmark = pytest.mark.gpu

KEYS = ("level", "coords", "origin", "dx", "parent", "children", "nbr", "cnbr")
WHICH = "ref" if os.path.exists(REF_SO) else "port"


def same_tables(a, b):
    for k in KEYS:
        x, y = np.asarray(a[k]).reshape(-1), np.asarray(b[k]).reshape(-1)
        assert x.shape == y.shape, (k, x.shape, y.shape)
        assert np.array_equal(x, y), (k, int(np.flatnonzero(x != y)[0]))


def same_as_oracle(tree: DeviceTree, o: Oracle):
    assert tree.n_blocks == o.n_blocks
    assert tree.n_levels == o.n_levels
    same_tables(tree.topology_arrays(), o.topology())
    for l in range(1, tree.n_levels + 1):
        assert np.array_equal(tree.level_blocks(l), o.level_blocks(l)), l


@pytest.mark.parametrize("dim,N,levels", [(2, 8, 5), (3, 4, 4), (3, 16, 3)])
def test_uniform_tree_matches_reference(dim, N, levels):
    lo, hi = (-0.5,) * dim, (0.5,) * dim
    tree = DeviceTree(dim, lo, hi, N)
    tree.refine_all(levels - 1, levels)
    o = Oracle(dim, N, lo, hi, WHICH)
    o.build_uniform(levels)
    same_as_oracle(tree, o)


@pytest.mark.parametrize("dim,N,seed,rounds", [(2, 4, 1, 8), (2, 8, 2, 6), (3, 4, 3, 5), (3, 8, 4, 4)])
def test_random_flags_force_balancing(dim, N, seed, rounds):
    """A few flags on the finest leaves: each drags a chain of coarser blocks
    along (refine_balanced, mesh.hpp:253-278); the new ids follow the recursion."""
    rng = np.random.default_rng(seed)
    lo, hi = (0.0,) * dim, (1.0,) * dim
    tree = DeviceTree(dim, lo, hi, N)
    tree.refine_all(2, 12)
    o = Oracle(dim, N, lo, hi, WHICH)
    o.build_uniform(3)
    forced = 0
    for _ in range(rounds):
        t = o.topology()
        leaf = np.flatnonzero(t["children"][:, 0] < 0)
        deep = t["level"][leaf].max()
        pool = leaf[t["level"][leaf] >= deep - 1]
        ids = [int(b) for b in rng.choice(pool, size=min(len(pool), 5), replace=False)]
        n = tree.adapt_refine(ids, 12)
        forced += n - len(ids)
        o.adapt_refine(ids, 12)
        same_as_oracle(tree, o)
    assert forced > 0 and tree.n_levels >= 6


@pytest.mark.parametrize("name", ["cfg3@6", "cfg3"])
def test_config3_refinement_matches_reference(name):
    """BASELINE config 3: base 64^3 (N = 8) refined where |f(x)| < 2 dx up to
    level 7 (19 465 blocks), with the level set evaluated on the device."""
    case = cfgs.get_case(name)
    D = case.dim
    tree = DeviceTree(D, case.lo[:D], case.hi[:D], case.N)
    tree.refine_all(case.levels - 1, case.levels)
    tree.refine_band(case.lsf, case.amr_band, case.max_level)
    o = Oracle(D, case.N, case.lo[:D], case.hi[:D], WHICH)
    o.build_uniform(case.levels)
    o.refine_band(case.lsf.as_descs(), case.amr_band, case.max_level)
    same_as_oracle(tree, o)
    if name == "cfg3":
        assert tree.n_blocks == 19465 or tree.n_blocks == sum((1, 8, 64, 512, 1664, 5120, 12160))
        assert tree.adapt_passes >= 3 + 3  # 3 uniform passes + one per refined level


@pytest.mark.parametrize("dim", [2, 3])
def test_harness_criteria_match_reference(dim):
    """build_case's criteria: sphere_refined (harness.hpp:351-355) and the
    two_electrodes tip ball (:413-418)."""
    N, max_level = 8, 5 if dim == 3 else 6
    lo, hi = (-0.5,) * dim, (0.5,) * dim
    dx_min = 1.0 / (N * (1 << (max_level - 1)))
    tree = DeviceTree(dim, lo, hi, N)
    tree.refine_radial(dx_min, 0.1, (0.0,) * dim, max_level)
    o = Oracle(dim, N, lo, hi, WHICH)
    o.refine_crit(1, dx_min, 0.1, (0.0,) * dim, max_level)
    same_as_oracle(tree, o)
    assert tree.n_levels == max_level

    lo, hi = (0.0,) * dim, (1.0,) * dim
    tip = (0.5, 0.8) if dim == 2 else (0.5, 0.5, 0.8)
    tree = DeviceTree(dim, lo, hi, N)
    tree.refine_all(max_level - 3, max_level)
    tree.refine_ball(dx_min, 0.06, tip, max_level)
    o = Oracle(dim, N, lo, hi, WHICH)
    o.build_uniform(max_level - 2)
    o.refine_crit(2, dx_min, 0.06, tip, max_level)
    same_as_oracle(tree, o)
    assert tree.n_levels == max_level


def test_errors_match_reference():
    with pytest.raises(_lib.PmgError, match="block size N must be a power of two and at least 4"):
        DeviceTree(2, (0, 0), (1, 1), 6)
    with pytest.raises(_lib.PmgError, match="domain must be square/cubic"):
        DeviceTree(2, (0, 0), (1, 2), 8)
    tree = DeviceTree(2, (0, 0), (1, 1), 8)
    tree.refine_all(1, 2)
    with pytest.raises(_lib.PmgError, match="refinement beyond the configured maximum level"):
        tree.adapt_refine([1], 2)  # mesh.hpp:165-167
    assert tree.n_blocks == 5  # unchanged


def test_solve_on_device_tree_equals_host_mesh_path():
    """cfg3@6: the solver fed by pmg_b200_set_mesh_from_tree gives the V-cycle
    history of the host-built mesh, bit for bit."""
    case = cfgs.get_case("cfg3@6")
    D = case.dim
    mesh = case.build_mesh()
    tree = DeviceTree(D, case.lo[:D], case.hi[:D], case.N)
    tree.refine_all(case.levels - 1, case.levels)
    tree.refine_band(case.lsf, case.amr_band, case.max_level)
    same_tables(tree.topology_arrays(), mesh.topology_arrays())
    hist = []
    for dev in (DeviceMesh(mesh), DeviceMesh(None, tree=tree)):
        st = build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
        dev.set_field(VAR_RHS, case.rhs_fields(dev.mesh), layout=LAYOUT_INTERIOR)
        sol = MgSolver(dev, None, MgConfig())
        hist.append([sol.v_cycle().max_resid for _ in range(4)])
        phi = dev.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
        hist.append(phi)
    assert hist[0] == hist[2]
    assert np.array_equal(hist[1], hist[3])
