"""A short solve for compute-sanitizer: the case's stencils on the GPU, FMG +
two V-cycles (every kernel of the cycle graphs).  python tools/sanitize_case.py cfg2@3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

for name in sys.argv[1:]:
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    h = [sol.fmg_cycle(), sol.v_cycle(), sol.v_cycle()]
    print(name, [x.max_resid for x in h], flush=True)
