"""GPU: the Morton-partitioned V-cycle driver (distributed.py) on one rank
reproduces the single-GPU V-cycle bit for bit -- same operations, same order;
the exchanges are empty.  (The halo logic itself is covered with two gloo
ranks on CPU in tests/test_partition.py.)"""
import numpy as np
import pytest

from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.distributed import DistributedMgSolver
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

pytestmark = pytest.mark.gpu


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
    b = DistributedMgSolver(dev_b, MgConfig())
    hb = [b.v_cycle() for _ in range(3)]
    phi_b = dev_b.get_field(VAR_PHI, layout=LAYOUT_INTERIOR)
    for x, y in zip(ha, hb):
        assert x.max_resid == y.max_resid and x.l2_resid == y.l2_resid, (x, y)
    assert np.array_equal(phi_a, phi_b)
