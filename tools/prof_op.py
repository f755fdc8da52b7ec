"""Run one op (time_op code, level, reps) inside a cudaProfilerStart/Stop window
after warm-up, for `ncu --profile-from-start off`:  python tools/prof_op.py OP LEVEL REPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

op, level, reps = (int(x) for x in sys.argv[1:4])
case = cfgs.get_case(os.environ.get("CASE", "cfg2"))
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
sol.fmg_cycle()
sol.time_op(op, level, 3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sol.time_op(op, level, reps)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
