"""Per-level in-graph op times of config 2 (each op captured 20x into one
CUDA graph): python tools/exp_ops.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
    from paper_2205_09411_b200 import configs as cfgs
    from paper_2205_09411_b200.mesh import VAR_RHS
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
    case = cfgs.get_case(os.environ.get("CASE", "cfg2"))
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    sol.fmg_cycle()
    g = 100 if os.environ.get("GRAPH", "1") == "1" else 0
    us5 = 1e3 * min(sol.time_op(5, mesh.n_levels, 20) for _ in range(3))
    us = lambda op, lv, r=20: 1e3 * min(sol.time_op(op + g, lv, r) for _ in range(3))  # noqa: E731
    print(f"  vcycle {us5:.1f} us  coarse {us(4, 1):.1f} us")
    for l in range(mesh.n_levels, 1, -1):
        print(f"  level {l} ({len(mesh.level_blocks(l))} blocks): gs {us(0, l):7.1f}  restrict {us(1, l):7.1f}"
              f"  prolong {us(2, l):7.1f}  record {us(3, l):7.1f}  fas {us(8, l):7.1f}"
              f"  smooth step {us(9, l):7.1f}  prolong(in-cycle) {us(10, l):7.1f} us")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    out = subprocess.run([sys.executable, __file__, "child"], capture_output=True, text=True)
    print(out.stdout.rstrip() if out.returncode == 0 else out.stderr[-2000:], flush=True)
