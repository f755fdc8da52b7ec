"""CPU: the oracle restatement (oracle/pmg_oracle.cpp) against the reference.

Two pins, both bit-exact:
  * tests/golden/*.npz, produced from the unmodified reference build by
    tools/gen_golden.py (topology, StencilSet, residual history, phi hash,
    coarse CSR) -- runs everywhere;
  * the reference build itself (oracle/_ref/libpmgref.so), operator by
    operator on random fields -- where that library was built.
"""
import glob
import hashlib
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

from oracle.oc import PORT_SO, REF_SO, Oracle  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_OLD, VAR_PHI, VAR_RES, VAR_RHS  # noqa: E402

from helpers import interior, oracle_for_case  # noqa: E402

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
needs_port = pytest.mark.skipif(not os.path.exists(PORT_SO), reason="make -C oracle port")
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build absent")


def _case_of(path):
    return os.path.basename(path)[:-4].replace("_L", "@")


@needs_port
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_port_matches_reference_golden(path):
    from gen_golden import run
    gold = np.load(path)
    name = _case_of(path)
    cycles = int(np.sum(gold["plan"] == "v"))
    out = run(name, cycles, which="port")
    assert np.array_equal(out["history"], gold["history"]), (out["history"], gold["history"])
    for k in gold.files:
        if k in ("history", "plan", "phi_sample_idx"):
            continue
        assert np.array_equal(np.asarray(out[k]), gold[k]), k


@needs_port
@needs_ref
@pytest.mark.parametrize("name", ["cfg1@3", "cfg2@3", "cfg3@5"])
def test_port_operators_bit_exact(name):
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    rng = np.random.default_rng(3)
    NI = case.N ** case.dim
    phi = cfgs.padded_from_interior(rng.uniform(-1, 1, (mesh.n_blocks, NI)), case.dim, case.N)
    g = cfgs.padded_from_interior(rng.uniform(-1, 1, (mesh.n_blocks, NI)), case.dim, case.N)
    os_ = []
    for which in ("ref", "port"):
        o = oracle_for_case(case, mesh, which)
        o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)
        o.set_field(VAR_PHI, phi)
        o.set_field(VAR_RHS, g)
        o.solver_create()
        os_.append(o)
    a, b = os_
    L = mesh.n_levels

    def same(tag):
        for var in (VAR_PHI, VAR_RHS, VAR_RES, VAR_OLD):
            assert np.array_equal(a.get_field(var), b.get_field(var)), (tag, var)

    same("init")
    for o in os_:
        for p in (0, 1):
            o.gsrb_sweep(L, p)
            o.fill_ghosts(L, VAR_PHI)
    same("gsrb")
    for o in os_:
        o.residual_level(L)
        o.restrict_level(L)
    same("restrict")
    for o in os_:
        o.prolong_correction(L)
    same("prolong")
    for o in os_:
        o.coarse_solve()
    same("coarse")
    assert a.bicgstab_probe() == b.bicgstab_probe()
    for o in os_:
        o.restrict_level_no_guess(L)
        o.prolong_full(L)
    same("fmg transfer")
    ha = [a.v_cycle() for _ in range(2)] + [a.fmg_cycle(), a.measure_residual()]
    hb = [b.v_cycle() for _ in range(2)] + [b.fmg_cycle(), b.measure_residual()]
    assert ha == hb
    same("cycles")


@needs_port
def test_port_errors_follow_reference():
    o = Oracle(2, 8, [0, 0], [1, 1], "port")
    with pytest.raises(Exception, match="n_up and n_down must be at least 1"):
        o.solver_create(n_down=0)
    with pytest.raises(Exception, match="coarse_rel_tol must be in"):
        o.solver_create(coarse_rel_tol=2.0)
    with pytest.raises(Exception, match="block size N must be a power of two"):
        Oracle(2, 6, [0, 0], [1, 1], "port")._check(1)
