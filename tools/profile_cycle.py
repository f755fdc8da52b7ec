"""Set up a BASELINE config on cuda:0, then run V-cycles inside a
cudaProfilerStart/Stop window (for `ncu --profile-from-start off`)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--warm", type=int, default=3)
a = ap.parse_args()
case = cfgs.get_case(a.config)
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
if case.fmg_first:
    sol.fmg_cycle()
for _ in range(a.warm):
    sol.v_cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.cycles):
    s = sol.v_cycle()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("kernels/cycle", sol.kernel_count(0), "resid", s.max_resid)
