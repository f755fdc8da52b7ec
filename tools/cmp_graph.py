"""V-cycle time per cycle: one CUDA graph per cycle (20 launches) against
several cycles captured into ONE graph (pmg_b200_time_op 5 vs 105)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

case = cfgs.get_case(os.environ.get("CASE", "cfg2"))
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
sol.fmg_cycle()
for _ in range(10):
    sol.v_cycle()
L = mesh.n_levels
for rep in range(3):
    a = 1e3 * sol.time_op(5, L, 20)
    b = {r: 1e3 * sol.time_op(105, L, r) for r in (1, 2, 4, 20)}
    print(f"per-cycle graphs: {a:.1f} us/cycle; cycles per graph -> us/cycle: " +
          "  ".join(f"{r}: {v:.1f}" for r, v in b.items()))
