"""Post-solve field kernels against the reference.

pmg::face_gradient (proj/include/pmg/fields.hpp:149-232) runs on the
unmodified reference build (oracle/_ref/libpmgref.so) after a few cycles;
its PHI (every level: coarse-fine ghosts read the parent level) is uploaded
to the GPU and the device kernels must reproduce every face value and the
cell-centred magnitude bit for bit -- regular faces, faces cut by the level
set, faces inside objects, physical and (AMR) coarse-fine ghosts.
"""
import os

import numpy as np
import pytest

from oracle.oc import REF_SO
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200 import face_gradient
from paper_2205_09411_b200.mesh import VAR_PHI
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

from helpers import interior, setup_pair

pytestmark = pytest.mark.gpu

VAR_AUX = 4  # the reference's post-processing scratch (mesh.hpp:19)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build missing (make -C oracle ref)")
@pytest.mark.parametrize("name", ["cfg1@4", "cfg2@3", "cfg3@5", "cfg4@3"])
def test_face_gradient_bit_exact(name):
    case = cfgs.get_case(name)
    o, dev, sol, mesh, st = setup_pair(case)
    o.fmg_cycle()
    for _ in range(2):
        o.v_cycle()
    phi = interior(o, VAR_PHI, case.dim, case.N)
    dev.set_field(VAR_PHI, phi, layout=LAYOUT_INTERIOR)
    ref_ids, ref_faces = o.face_gradient(VAR_PHI, VAR_AUX)
    ids, faces, mag = face_gradient(dev)
    assert np.array_equal(ids, ref_ids)
    assert faces.shape == ref_faces.shape
    bad = np.flatnonzero(faces.reshape(-1) != ref_faces.reshape(-1))
    assert bad.size == 0, (bad.size, bad[:8], faces.reshape(-1)[bad[:4]], ref_faces.reshape(-1)[bad[:4]])
    # some faces of each kind were exercised
    assert np.count_nonzero(ref_faces) > 0
    ref_mag = interior(o, VAR_AUX, case.dim, case.N)[ref_ids]
    assert np.array_equal(mag, ref_mag.reshape(mag.shape))


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build missing (make -C oracle ref)")
@pytest.mark.parametrize("name", ["cfg1@4", "cfg2@3", "cfg3@5"])
@pytest.mark.parametrize("vw", [False, True])
def test_error_norms_match_reference(name, vw):
    """pmg::error_norms against AnalyticSolution (fields.hpp:35-69).  The
    analytic sphere sits at the origin, a corner of these domains: R is small
    enough that no solved cell lies inside it.  3D evaluates sqrt and / only
    (correctly rounded on both sides: linf bit-exact); 2D adds log (CUDA's log
    vs glibc's: within an ulp); l2 sums in a different order."""
    from paper_2205_09411_b200 import error_norms

    case = cfgs.get_case(name)
    o, dev, sol, mesh, st = setup_pair(case)
    o.fmg_cycle()
    o.v_cycle()
    dev.set_field(VAR_PHI, interior(o, VAR_PHI, case.dim, case.N), layout=LAYOUT_INTERIOR)
    s3 = case.dim == 3
    ref = o.error_norms(1.0, 0.7, 1e-3, sphere3d=s3, volume_weighted=vw)
    got = error_norms(dev, 1.0, 0.7, 1e-3, sphere3d=s3, volume_weighted=vw)
    if s3:
        assert got[0] == ref[0]
    else:
        assert abs(got[0] - ref[0]) <= 4e-16 * abs(ref[0]) + 1e-300
    assert abs(got[1] - ref[1]) <= 1e-13 * abs(ref[1])


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build missing (make -C oracle ref)")
def test_error_norms_inside_raises_like_reference():
    from paper_2205_09411_b200 import error_norms
    from paper_2205_09411_b200._lib import PmgError
    from oracle.oc import OracleError

    case = cfgs.get_case("cfg2@3")
    o, dev, sol, mesh, st = setup_pair(case)
    with pytest.raises(OracleError) as e_ref:
        o.error_norms(1.0, 1.0, 0.3)
    with pytest.raises(PmgError) as e_gpu:
        error_norms(dev, 1.0, 1.0, 0.3)
    assert str(e_gpu.value) == str(e_ref.value) == "analytic solution undefined inside"


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build missing (make -C oracle ref)")
@pytest.mark.parametrize("name", ["cfg1@4", "cfg3@5"])
def test_write_dump_layout(name, tmp_path):
    """pmg_b200_write_dump (io.hpp:23-71) parsed back the way pmg::read_dump
    does (io.hpp:87-140): header fields, leaves level-major / x-major with their
    cell origins and offsets, and the raw data equal to the reference's PHI of
    those leaves.  Byte identity with the reference's own write_dump of the
    same field is checked by the C++ drop-in driver (tests/test_gpu_cpp_dropin.py)."""
    from paper_2205_09411_b200 import write_dump

    case = cfgs.get_case(name)
    o, dev, sol, mesh, st = setup_pair(case)
    o.fmg_cycle()
    o.v_cycle()
    phi = interior(o, VAR_PHI, case.dim, case.N)
    dev.set_field(VAR_PHI, phi, layout=LAYOUT_INTERIOR)
    path = tmp_path / "gpu.dump"
    write_dump(dev, str(path), "phi")
    raw = path.read_bytes()
    head, data = raw.split(b"DATA\n", 1)
    lines = head.decode().splitlines()
    assert lines[0] == "pmg dump 1" and lines[1] == "field phi" and lines[2] == f"dim {case.dim}"
    assert lines[5] == f"block_size {case.N}"
    blocks = [ln.split() for ln in lines if ln.startswith("block ")]
    leaves = [b for lvl in range(1, mesh.n_levels + 1) for b in mesh.level_blocks(lvl) if mesh.is_leaf(b)]
    assert lines[6] == f"blocks {len(leaves)}" and len(blocks) == len(leaves)
    vals = np.frombuffer(data, dtype="<f8")
    assert vals.size == len(leaves) * case.N ** case.dim
    for q, b in enumerate(leaves):
        rec = blocks[q]
        assert int(rec[1]) == mesh.level[b] and int(rec[-1]) == q * case.N ** case.dim
        assert [int(x) for x in rec[2:-1]] == [c * case.N for c in mesh.coords[b][:case.dim]]
        assert np.array_equal(vals[q * case.N ** case.dim:(q + 1) * case.N ** case.dim], phi[b])


def test_staged_upload_matches_plain_upload():
    """pmg_b200_stage_field_async + commit_staged_field (the double-buffered
    upload bench.py's e2e uses) leave exactly what upload_level_field leaves,
    also when the next stage is issued while a V-cycle is in flight."""
    import ctypes as C

    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
    from paper_2205_09411_b200.mesh import VAR_RHS

    case = cfgs.get_case("cfg2@3")
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    g = case.rhs_fields(mesh)
    dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    sol.fmg_cycle()
    L = mesh.n_levels
    rng = np.random.default_rng(7)
    blocks = np.array(mesh.level_blocks(L))
    vals = [np.ascontiguousarray(rng.standard_normal((len(blocks), case.N ** 3))) for _ in range(3)]
    dev._check(dev.lib.pmg_b200_stage_field_async(dev.h, VAR_RHS, L, C.c_void_p(vals[0].ctypes.data),
                                                  LAYOUT_INTERIOR))
    for k in range(3):
        dev._check(dev.lib.pmg_b200_commit_staged_field(dev.h))
        got = dev.get_field(VAR_RHS, layout=LAYOUT_INTERIOR)[blocks]
        assert np.array_equal(got, vals[k])
        sol.v_cycle_async()
        if k + 1 < 3:
            dev._check(dev.lib.pmg_b200_stage_field_async(dev.h, VAR_RHS, L, C.c_void_p(vals[k + 1].ctypes.data),
                                                          LAYOUT_INTERIOR))
        sol.cycle_result()
    with pytest.raises(Exception):
        dev._check(dev.lib.pmg_b200_commit_staged_field(dev.h))  # nothing staged
