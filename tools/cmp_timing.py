"""Per-cycle device time and coarse BiCGStab iterations of config 2's plan
(FMG + V-cycles): shows how the V-cycle time depends on the solver state
(the coarse solve runs more iterations once the residual sits at round-off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS  # noqa: E402
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR  # noqa: E402

case = cfgs.get_case(os.environ.get("CASE", "cfg2"))
mesh = case.build_mesh()
dev = DeviceMesh(mesh)
build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
g = case.rhs_fields(mesh)
dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
sol = MgSolver(dev, None, MgConfig())
stream = torch.cuda.ExternalStream(dev.stream)
zero = np.zeros_like(g)
for rep in range(3):
    dev.set_field(VAR_PHI, zero, layout=LAYOUT_INTERIOR)
    dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
    sol.init()
    sol.set_have_guess(False)
    if case.fmg_first:
        sol.fmg_cycle()
    rows = []
    for k in range(26):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sol.v_cycle_async()
        e1.record(stream)
        st = sol.cycle_result()
        torch.cuda.synchronize()
        rows.append((k + 1, e0.elapsed_time(e1) * 1e3, sol.coarse_info()[0], st.max_resid))
    print("rep", rep, " ".join(f"[{k}: {t:.0f}us it={it} r={r:.1e}]" for k, t, it, r in rows))
