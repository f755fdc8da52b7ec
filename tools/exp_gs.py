import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
case = cfgs.get_case(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
mesh = case.build_mesh(); dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
L = mesh.n_levels
print("exp", os.environ.get("PMG_EXP", "0"), "gs finest us", 1e3 * sol.time_op(0, L, 50), "gs L-1 us", 1e3 * sol.time_op(0, L - 1, 50))
