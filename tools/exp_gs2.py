"""Per-phase device times of the finest level of a config (CUDA events, pmg_b200_time_op).
usage: python tools/exp_gs2.py [sphere|none] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_09411_b200 import (SHAPE_NONE, DeviceMesh, LevelSetSpec, MgConfig, MgSolver,  # noqa: E402
                                   StencilBuildConfig, build_stencils)
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

case = cfgs.get_case(sys.argv[2] if len(sys.argv) > 2 else "cfg2")
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
lsf = case.lsf if (len(sys.argv) < 2 or sys.argv[1] == "sphere") else LevelSetSpec(shape=SHAPE_NONE)
build_stencils(dev, lsf, StencilBuildConfig(w_min=case.w_min))
dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
L = mesh.n_levels
us = lambda op, lv, r: 1e3 * sol.time_op(op, lv, r)  # noqa: E731
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'sphere'} exp {os.environ.get('PMG_EXP', '0')}: "
      f"gs {us(0, L, 50):.1f}  restrict {us(7, L, 20):.1f}  fas {us(8, L, 20):.1f}  "
      f"prolong {us(2, L, 20):.1f}  record {us(3, L, 20):.1f}  coarse {us(4, 1, 20):.1f}  "
      f"vcycle {us(5, L, 20):.1f} us")
