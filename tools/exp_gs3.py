import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils, LevelSetSpec, SHAPE_NONE
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
case = cfgs.get_case("cfg2")
mesh = case.build_mesh(); dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf if "sphere" in sys.argv else LevelSetSpec(shape=SHAPE_NONE), StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
L = mesh.n_levels
sol.time_op(0, L, 3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sol.time_op(0, L, 2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
