"""V-cycle graph time of config 2 with parts switched off (PMG_EXP timing
experiments, one subprocess per setting), plus the per-level op times.

    python tools/cycle_breakdown.py            # all settings
    python tools/cycle_breakdown.py child EXP  # one setting (internal)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETTINGS = [
    ("full cycle", 0),
    ("no coarse solve", 1 << 21),
    ("no GS below finest", 1 << 20),
    ("no GS on levels <= 64 blocks", 1 << 19),
    ("no coarse, no GS below finest", (1 << 20) | (1 << 21)),
]


def child(exp):
    os.environ["PMG_EXP"] = str(exp)
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
    us = lambda op, lv, r=20: 1e3 * sol.time_op(op, lv, r)  # noqa: E731
    v = min(us(5, mesh.n_levels, 20) for _ in range(3))
    print(f"RESULT {v:.1f}")
    if exp == 0:
        for l in range(mesh.n_levels, 1, -1):
            print(f"  level {l} ({len(mesh.level_blocks(l))} blocks): gs {us(0, l):7.1f}  restrict {us(1, l):7.1f}"
                  f"  prolong {us(2, l):7.1f}  record {us(3, l):7.1f} us")
        print(f"  coarse {us(4, 1):.1f} us")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(int(sys.argv[2]))
        sys.exit(0)
    for name, exp in SETTINGS:
        out = subprocess.run([sys.executable, __file__, "child", str(exp)], capture_output=True, text=True)
        lines = out.stdout.splitlines()
        res = [x for x in lines if x.startswith("RESULT")]
        print(f"{name:34s} {res[0].split()[1] if res else 'FAILED'} us/V-cycle", flush=True)
        for x in lines:
            if x.startswith("  "):
                print(x)
        if not res:
            print(out.stderr[-2000:])
