"""GPU parity against the committed golden fixtures of the reference
(tests/golden/*.npz, tools/gen_golden.py) -- needs no CPU oracle at run time.

  * GPU stencil build: every StencilSet array bit-exact;
  * coarse system assembly: CSR bit-exact;
  * residual history of the configuration's cycle plan within
    |dr| <= 1e-6 r + 16 eps (2D/dx^2) max|phi|;
  * final phi within 1e-10 max|phi| on a strided sample (§8c(ii)).
"""
import glob
import os

import numpy as np
import pytest

from paper_2205_09411_b200 import (DeviceMesh, MgConfig, MgSolver, StencilBuildConfig,
                                   build_stencils)
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import VAR_PHI, VAR_RHS
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

from helpers import resid_tol

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_gpu_matches_golden(path):
    gold = np.load(path)
    case = cfgs.get_case(os.path.basename(path)[:-4].replace("_L", "@"))
    mesh = case.build_mesh()
    dev = DeviceMesh(mesh)
    st = build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    for k in ("boundary", "row_count", "center", "nb", "bc", "d", "obj", "mask", "pin_obj", "lin"):
        assert np.array_equal(np.asarray(st[k]).reshape(-1), gold["st_" + k].reshape(-1)), k
    rof = np.asarray(st["row_of"])[np.asarray(st["boundary"]).astype(bool)]
    assert np.array_equal(rof, gold["st_row_of"])
    dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    cs = sol.coarse_system()
    for k in ("rp", "ci", "val", "c0", "cobj"):
        assert np.array_equal(np.asarray(cs[k]).reshape(-1), gold["cs_" + k].reshape(-1)), k
    hist = [sol.measure_residual()]
    for kind in gold["plan"]:
        hist.append(sol.fmg_cycle() if kind == "fmg" else sol.v_cycle())
    phi = dev.get_field(VAR_PHI, layout=LAYOUT_INTERIOR).reshape(-1)
    maxphi = float(gold["phi_max"][0])
    dxf = mesh.level_dx(mesh.n_levels)
    for k, (a, b) in enumerate(zip(hist, gold["history"])):
        assert abs(a.max_resid - b[0]) <= resid_tol(b[0], maxphi, dxf, case.dim), (k, a, b)
        assert abs(a.l2_resid - b[1]) <= resid_tol(b[1], maxphi, dxf, case.dim), (k, a, b)
    d = np.max(np.abs(phi[gold["phi_sample_idx"]] - gold["phi_sample"]))
    assert d <= 1e-10 * maxphi, d
