import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils, LevelSetSpec, SHAPE_NONE
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
case = cfgs.get_case("cfg2")
mesh = case.build_mesh(); dev = DeviceMesh(mesh)
lsf = case.lsf if sys.argv[1] == "sphere" else LevelSetSpec(shape=SHAPE_NONE)
build_stencils(dev, lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
L = mesh.n_levels
print(sys.argv[1], "exp", os.environ.get("PMG_EXP", "0"), "gs finest us %.1f" % (1e3 * sol.time_op(0, L, 50)), "restrict %.1f" % (1e3 * sol.time_op(1, L, 20)), "prolong %.1f" % (1e3 * sol.time_op(2, L, 20)), "record %.1f" % (1e3 * sol.time_op(3, L, 20)))
