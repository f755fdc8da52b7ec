"""GPU parity against the CPU oracle (reference build, oracle/_ref/libpmgref.so).

Per-operator results are compared BIT-EXACTLY (the library is compiled with
--fmad=false and replays the reference's operation order; ghosts are evaluated
with the fill formulas of mesh.hpp:471-554).  Whole cycles differ only through
reassociated reductions (BiCGStab dot products, residual sums), so they are
compared with the tolerances of SURVEY.md §8c:
  (ii)  max|dphi| <= 1e-10 * max|phi| after the configured cycles;
  (iii) |dr_k| <= 1e-6 r_k + 16 eps (2D/dx^2) max|phi| per cycle.
"""
import os

import numpy as np
import pytest

from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_OLD, VAR_PHI, VAR_RES, VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

from helpers import ORACLES, interior, max_rel_diff, resid_tol, setup_pair

pytestmark = pytest.mark.gpu


def _random_fields(case, mesh, seed):
    rng = np.random.default_rng(seed)
    NI = case.N ** case.dim
    return rng.uniform(-1, 1, (mesh.n_blocks, NI)), rng.uniform(-1, 1, (mesh.n_blocks, NI))


def _lvl(mesh, arr, l):
    return arr[np.array(mesh.level_blocks(l))]


def _same(a, b, what):
    bad = np.nonzero(a != b)
    assert bad[0].size == 0, (f"{what}: {bad[0].size} cells differ, first at {bad[0][0]}, "
                              f"gpu {a[bad][0]!r} oracle {b[bad][0]!r}")


@pytest.mark.parametrize("name", ["cfg1@4", "cfg2@3", "cfg3@5", "cfg4@3", "amrx", "amrx16"])
def test_operators_bit_exact(name):
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    phi, g = _random_fields(case, mesh, 7)
    o, dev, sol, mesh, st = setup_pair(case, rhs=g, phi=phi)
    D, N, L = case.dim, case.N, mesh.n_levels

    def cmp(var, what, level=None):
        a = dev.get_field(var, layout=LAYOUT_INTERIOR)
        b = interior(o, var, D, N)
        if level is not None:
            a, b = _lvl(mesh, a, level), _lvl(mesh, b, level)
        _same(a, b, what)

    cmp(VAR_PHI, "init (pins)")
    for lev in (L, L - 1):
        for parity in (0, 1):
            sol.gsrb_sweep(lev, parity)
            o.gsrb_sweep(lev, parity)
            o.fill_ghosts(lev, VAR_PHI)
            cmp(VAR_PHI, f"gsrb level {lev} parity {parity}", lev)
    # level-L coarse-fine ghosts depend on level L-1, which was just swept: the
    # device evaluates ghosts from current values, the reference needs a refill
    # (MgSolver itself never reads level-L ghosts between these two points)
    o.fill_ghosts(L, VAR_PHI)
    sol.residual_level(L)
    o.residual_level(L)
    cmp(VAR_RES, "residual", L)
    sol.restrict_level(L)
    o.restrict_level(L)
    cmp(VAR_PHI, "restrict phi", L - 1)
    cmp(VAR_RHS, "FAS rhs", L - 1)
    cmp(VAR_OLD, "old snapshot", L - 1)
    for parity in (0, 1, 0, 1):
        sol.gsrb_sweep(L - 1, parity)
        o.gsrb_sweep(L - 1, parity)
        o.fill_ghosts(L - 1, VAR_PHI)
    cmp(VAR_PHI, "coarse smoothing", L - 1)
    sol.prolong_correction(L)
    o.prolong_correction(L)
    cmp(VAR_PHI, "prolong_correction", L)
    sol.restrict_level_no_guess(L)
    o.restrict_level_no_guess(L)
    cmp(VAR_PHI, "restrict_no_guess phi", L - 1)
    cmp(VAR_RHS, "restrict_no_guess rhs", L - 1)
    sol.prolong_full(L)
    o.prolong_full(L)
    cmp(VAR_PHI, "prolong_full", L)


def test_amr_block_classes():
    """cfg3 streams every block; the amrx mesh (coarse-fine faces through the
    interface) also exercises the block-per-CTA fallbacks."""
    for name, want_tile in (("cfg3@5", False), ("amrx", True), ("amrx16", True)):
        case = cfgs.get_case(name)
        o, dev, sol, mesh, st = setup_pair(case)
        L = mesh.n_levels
        cl = sol.level_classes(L)
        assert cl["blocks"] == len(mesh.level_blocks(L)) and cl["cf_faces"] > 0
        assert cl["gs_stream"] > 0 and cl["record_stream"] > 0 and cl["restrict_stream"] > 0
        tiles = cl["gs_tile"], cl["record_tile"], cl["restrict_tile"]
        assert all(t > 0 for t in tiles) if want_tile else tiles == (0, 0, 0), cl
        assert cl["restrict_stream"] + cl["restrict_tile"] == cl["blocks"]


def _run_cycles(case, which="ref", gpu_stencils=False, threads=1):
    o, dev, sol, mesh, st = setup_pair(case, which=which, gpu_stencils=gpu_stencils, threads=threads)
    D, N = case.dim, case.N
    dxf = mesh.level_dx(mesh.n_levels)
    hist = []
    a0 = sol.measure_residual()
    b0 = o.measure_residual()
    hist.append((a0, b0))
    plan = (["fmg"] if case.fmg_first else []) + ["v"] * case.v_cycles
    for kind in plan:
        a = sol.fmg_cycle() if kind == "fmg" else sol.v_cycle()
        b = o.fmg_cycle() if kind == "fmg" else o.v_cycle()
        hist.append((a, b))
    pa = dev.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
    pb = interior(o, VAR_PHI, D, N)
    maxphi = float(np.max(np.abs(pb)))
    for k, (a, b) in enumerate(hist):
        tol = resid_tol(b[0], maxphi, dxf, D)
        assert abs(a.max_resid - b[0]) <= tol, (k, a.max_resid, b[0], tol)
        tol2 = resid_tol(b[1], maxphi, dxf, D)
        assert abs(a.l2_resid - b[1]) <= tol2, (k, a.l2_resid, b[1], tol2)
    return max_rel_diff(pa, pb), hist


@pytest.mark.parametrize("name", ["cfg1", "cfg2@4", "cfg3@5", "cfg4@4", "amrx", "amrx16"])
def test_cycles_match_oracle(name):
    case = cfgs.get_case(name)
    rel, hist = _run_cycles(case)
    assert rel <= 1e-10, rel
    # the cycles converge like the reference's (residual reduction per cycle)
    assert hist[-1][0].max_resid < hist[0][0].max_resid


@pytest.mark.parametrize("name", ["cfg2@3", "cfg4@3", "cfg1@3"])
def test_coarse_bicgstab_iterations_match(name):
    """The on-chip BiCGStab replays detail::bicgstab (multigrid.hpp:208-280):
    same state in, same iteration count (+-1 for reassociated dot products),
    same converged solution within the solve tolerance."""
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    phi, g = _random_fields(case, mesh, 11)
    o, dev, sol, mesh, st = setup_pair(case, rhs=g, phi=phi)
    conv, it_ref, rel_ref = o.bicgstab_probe()
    sol.coarse_solve()
    o.coarse_solve()
    it, rel = sol.coarse_info()
    assert conv
    assert abs(it - it_ref) <= 1, (it, it_ref)
    assert rel <= 1e-6 and rel_ref <= 1e-6
    a = _lvl(mesh, dev.get_field(VAR_PHI, layout=LAYOUT_INTERIOR), 1)
    b = _lvl(mesh, interior(o, VAR_PHI, case.dim, case.N), 1)
    assert max_rel_diff(a, b) < 1e-9


def test_coarse_solve_single_level():
    """multigrid test 'single-level v_cycle is the coarse solve' (test_multigrid.cpp:382-396)."""
    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, build_uniform
    from paper_2205_09411_b200.solver import StencilSet
    mesh = build_uniform(2, (-0.5, -0.5), (0.5, 0.5), 8, 1)
    dev = DeviceMesh(mesh)
    g = np.ones((1, 64))
    dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
    st = StencilSet(boundary=np.zeros(1, np.int32), row_count=np.zeros(1, np.int32),
                    row_of=np.full((1, 64), -1, np.int32), center=np.zeros(0), nb=np.zeros(0),
                    bc=np.zeros(0), d=np.zeros(0), obj=np.zeros(0, np.int8),
                    mask=np.zeros(0, np.uint8), pin_obj=np.zeros(0, np.int8),
                    lin=np.zeros(0, np.int32), phi_b=np.zeros(0))
    sol = MgSolver(dev, st, MgConfig())
    r0 = sol.measure_residual().max_resid
    r1 = sol.v_cycle().max_resid
    assert r1 <= 1e-5 * r0


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5@6"])
def test_full_size_cycles_match_reference(name):
    """BASELINE configs 2 (256^3, FMG + 8 V, the headline), 3 (AMR, effective
    512^3, 10 V) and 4 (512^3, 32 spheres, 12 V) at full size, and config 5's
    geometry and plan (two spheres at phi_b = +-1, Gaussian g, 10 V from phi = 0)
    at 512^3, GPU stencils, against the unmodified reference solver run on the
    host's cores: residual histories within the floor-aware bound, final phi
    within 1e-10 max|phi|."""
    if "ref" not in ORACLES:
        pytest.skip("reference build (oracle/_ref) absent")
    case = cfgs.get_case(name)
    rel, hist = _run_cycles(case, which="ref", gpu_stencils=True, threads=os.cpu_count() or 1)
    assert rel <= 1e-10, rel
    assert hist[-1][0].max_resid < 1e-6 * hist[0][0].max_resid


def _host_ram_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


@pytest.mark.slow
@pytest.mark.timeout(2400)
def test_config5_1024_matches_reference():
    """BASELINE config 5 at its full 1024^3 (1.07e9 unknowns, 10 V from
    phi = 0) against the unmodified reference on the host's cores.  The
    reference's padded AoS fields need ~70 GB of host memory, so the test runs
    where the host has room (the B200 box has ~196 GB)."""
    if "ref" not in ORACLES:
        pytest.skip("reference build (oracle/_ref) absent")
    if _host_ram_gb() < 150:
        pytest.skip(f"needs ~150 GB of free host memory for the reference at 1024^3 ({_host_ram_gb():.0f} GB)")
    case = cfgs.get_case("cfg5")
    rel, hist = _run_cycles(case, which="ref", gpu_stencils=True, threads=os.cpu_count() or 1)
    assert rel <= 1e-10, rel
    assert hist[-1][0].max_resid < 1e-5 * hist[0][0].max_resid


@pytest.mark.timeout(900)
def test_config5_full_size_properties():
    """BASELINE config 5 (1024^3, two spheres at phi_b = +-1, Gaussian g) at full
    size on the GPU alone, with BASELINE's plan (10 V-cycles from phi = 0, no
    FMG): the records are finite and strictly decreasing, every cycle reduces
    the residual at the rate the reference-checked sizes show (5-6x), and ten
    cycles reduce it by more than 1e5."""
    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
    case = cfgs.get_case("cfg5")
    assert not case.fmg_first and case.v_cycles == 10
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    h = [sol.measure_residual()] + [sol.v_cycle() for _ in range(case.v_cycles)]
    r = np.array([x.max_resid for x in h])
    assert np.all(np.isfinite(r))
    assert np.all(np.diff(r) < 0), r
    red = np.exp(np.mean(np.log(r[1:-1] / r[2:])))
    assert red > 3.0, red  # about 5-6x per V-cycle at every size tested against the reference
    assert r[-1] < 1e-5 * r[0], r


def test_coarse_stall_message_matches_reference():
    """BiCGStab stall on a coarse system too large for the smoothing fallback
    (n = 3960 > 8^3 + 1; multigrid.hpp:456-465): the same std::runtime_error
    text as the reference -- iterations and unknowns exactly, the relative
    residual (std::to_string) to its printed digits up to the dot-product
    summation order."""
    import re

    from paper_2205_09411_b200 import MgConfig
    from paper_2205_09411_b200._lib import PMG_ERR_COARSE_STALL, PmgError
    case = cfgs.get_case("cfg2@3")
    o, dev, sol, mesh, st = setup_pair(case, mg=MgConfig(coarse_max_iters=1))
    with pytest.raises(PmgError) as ea:
        sol.v_cycle()
    with pytest.raises(RuntimeError) as eb:
        o.v_cycle()
    a, b = str(ea.value), str(eb.value)
    assert ea.value.code == PMG_ERR_COARSE_STALL
    pat = r"coarse solve failed: BiCGStab stalled at relative residual ([0-9.]+) after (\d+) iterations on (\d+) unknowns"
    ma, mb = re.search(pat, a), re.search(pat, b)
    assert ma and mb, (a, b)
    assert ma.group(2) == mb.group(2) == "1" and ma.group(3) == mb.group(3) == "3960", (a, b)
    assert abs(float(ma.group(1)) - float(mb.group(1))) <= 2e-6 + 1e-9 * float(mb.group(1)), (a, b)


def test_gsrb_fallback_matches_reference():
    """Config 1's coarse system (n = 52 <= 8^2 + 1) with BiCGStab capped at one
    iteration: the reference writes the iterate back and finishes with GS-RB
    sweeps (gsrb_fallback, multigrid.hpp:586-601); the GPU path does the same,
    with residual histories and phi within the SURVEY 8c bounds."""
    from paper_2205_09411_b200 import MgConfig
    case = cfgs.get_case("cfg1")
    o, dev, sol, mesh, st = setup_pair(case, mg=MgConfig(coarse_max_iters=1))
    D, N = case.dim, case.N
    dxf = mesh.level_dx(mesh.n_levels)
    hist = []
    for _ in range(4):
        hist.append((sol.v_cycle(), o.v_cycle()))
    pa = dev.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
    pb = interior(o, VAR_PHI, D, N)
    maxphi = float(np.max(np.abs(pb)))
    for k, (a, b) in enumerate(hist):
        assert abs(a.max_resid - b[0]) <= resid_tol(b[0], maxphi, dxf, D), (k, a.max_resid, b[0])
    assert max_rel_diff(pa, pb) <= 1e-10
