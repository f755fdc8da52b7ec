"""Per-level device times (CUDA events, back-to-back launches, pmg_b200_time_op) of the
GS half-sweep, restriction, FAS and prolongation on every level of a config."""
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
us = lambda op, lv, r=20: 1e3 * sol.time_op(op, lv, r)  # noqa: E731
for l in range(mesh.n_levels, 1, -1):
    print(f"level {l} ({len(mesh.level_blocks(l))} blocks): gs {us(0, l):7.1f}  restrict {us(7, l):7.1f}  "
          f"fas(l-1) {us(8, l):7.1f}  prolong {us(2, l):7.1f} us")
print(f"coarse {us(4, 1):.1f} us   vcycle {us(5, mesh.n_levels):.1f} us")
