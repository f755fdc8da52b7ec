"""Coarse-solve iteration counts per cycle and the in-graph coarse-solve time (config 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

case = cfgs.get_case(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
s = sol.fmg_cycle()
print("fmg", s.max_resid, sol.coarse_info())
for k in range(8):
    s = sol.v_cycle()
    print("v", k + 1, s.max_resid, sol.coarse_info())
for r in (1, 10):
    print(f"coarse alone x{r} (graph): {1e3 * sol.time_op(104, 1, r):.1f} us")
# per-iteration cost: the coarse solve alone with capped iteration counts
for mi in (1, 2, 6, 11, 21):
    sol2 = MgSolver(dev, None, MgConfig(coarse_max_iters=mi))
    print(f"max_iters {mi:3d}: {1e3 * sol2.time_op(104, 1, 10):.1f} us")
