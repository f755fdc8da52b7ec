"""GPU: the Morton-partitioned V-cycle (csrc/dist.h, distributed.py).

* One rank: the partitioned cycle (a CUDA graph, no transport) reproduces the
  single-GPU V-cycle bit for bit.
* Two and four ranks on ONE device: one context per rank in this process, the
  in-process transport (device copies between the contexts, one host thread
  per context), the real halo plans, the coarse-tail gather / broadcast and the
  rank-order record reduction.  Every rank's owned blocks must hold exactly the
  single-context V-cycle's phi after every cycle; the combined records match
  (max exactly, l2 up to the rank-order summation).
The NCCL transport runs the same enqueue sequence (captured into a graph) with
ncclSend / ncclRecv in place of the copies.
"""
import numpy as np
import pytest

from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.distributed import DistributedMgSolver
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS
from paper_2205_09411_b200.partition import halo_plan
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

pytestmark = pytest.mark.gpu


def case_ni(mesh):
    return mesh.N ** mesh.dim


def _setup(name):
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
    return case, mesh, dev


@pytest.mark.parametrize("name", ["cfg2@3", "cfg2@4", "cfg5@3"])
def test_distributed_vcycle_one_rank_matches(name):
    _, _, dev_a = _setup(name)
    a = MgSolver(dev_a, None, MgConfig())
    ha = [a.v_cycle() for _ in range(3)]
    phi_a = dev_a.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
    _, _, dev_b = _setup(name)
    b = DistributedMgSolver(dev_b, MgConfig(), world=1, rank=0)
    hb = [b.v_cycle() for _ in range(3)]
    phi_b = dev_b.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
    for x, y in zip(ha, hb):
        assert x.max_resid == y.max_resid and x.l2_resid == y.l2_resid, (x, y)
    assert np.array_equal(phi_a, phi_b)


@pytest.mark.parametrize("name,world", [("cfg2@4", 2), ("cfg5@4", 2), ("cfg5@4", 4), ("cfg4@4", 4)])
def test_partitioned_contexts_match_single(name, world):
    cycles = 3
    _, mesh, dev_a = _setup(name)
    a = MgSolver(dev_a, None, MgConfig())
    ha, phis = [], []
    for _ in range(cycles):
        ha.append(a.v_cycle())
        phis.append(dev_a.get_field(VAR_PHI, layout=LAYOUT_INTERIOR))
    devs = [_setup(name)[2] for _ in range(world)]
    sols = [DistributedMgSolver(d, MgConfig(), world=world, rank=r, transport="local") for r, d in enumerate(devs)]
    DistributedMgSolver.local_group(sols)
    part = sols[0].part
    assert part.split_level >= 2
    info = sols[1].info()
    assert info["world"] == world and info["transport"] == 2 and info["halo_cells"] > 0
    # the native halo plan receives exactly the cells partition.halo_plan lists
    ref = halo_plan(mesh, part, 1)
    n_ref = sum(len(v) for l in range(part.split_level, mesh.n_levels + 1)
                for c in (0, 1) for v in ref.recv.get((l, c), {}).values())
    assert info["halo_cells"] == n_ref
    # per-rank memory: the large levels map only the chunks (2 MB = 64 blocks
    # in Morton order) holding the rank's blocks and halo blocks -- at these
    # sizes the halo touches most chunks, at 1024^3 a rank maps ~1/world + 5%
    full = 4 * 8 * sum(len(mesh.level_blocks(l)) for l in range(1, mesh.n_levels + 1)) * case_ni(mesh)
    for s in sols:
        assert 0 < s.field_bytes() <= full, (s.field_bytes(), full)
    for k in range(cycles):
        hb = DistributedMgSolver.run_local(sols, lambda s: s.v_cycle())
        for r in range(world):  # every rank reports the combined records
            assert hb[r].max_resid == ha[k].max_resid, (k, r, hb[r], ha[k])
            assert abs(hb[r].l2_resid - ha[k].l2_resid) <= 1e-12 * ha[k].l2_resid, (k, r)
        for r, d in enumerate(devs):
            phi = d.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
            for l in range(part.split_level, mesh.n_levels + 1):
                ids = np.asarray(part.slots[l])[part.owner[l] == r]
                bad = np.nonzero(phi[ids] != phis[k][ids])
                assert bad[0].size == 0, f"cycle {k} rank {r} level {l}: {bad[0].size} cells differ"
