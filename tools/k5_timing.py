"""Stencil build (K5) timing, end to end: the device build +
host plan construction (pmg_b200_build_stencils) and the optional read-back
of the whole StencilSet (get_stencils).  python tools/k5_timing.py cfg2 cfg4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2205_09411_b200 import DeviceMesh, StencilBuildConfig, _lib  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402
from paper_2205_09411_b200.solver import _lsf_array  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    case = cfgs.get_case(name)
    t0 = time.perf_counter()
    mesh = case.build_mesh()
    t_mesh = time.perf_counter() - t0
    dev = DeviceMesh(mesh)
    torch.cuda.synchronize()
    cfg = StencilBuildConfig(w_min=case.w_min)
    descs = case.lsf.as_descs()
    arr = _lsf_array(descs)
    c = _lib.StencilCfgT(cfg.eps_tol, cfg.max_bracket_iters, cfg.d_min, cfg.w_min, cfg.boundary_safety,
                         int(cfg.thin_rescue))
    for rep in range(2):
        t0 = time.perf_counter()
        dev._check(dev.lib.pmg_b200_build_stencils(dev.h, C.cast(arr, C.c_void_p), len(descs), C.byref(c)))
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        st = dev.get_stencils([])
        t_get = time.perf_counter() - t0
        print(f"{name} rep {rep}: mesh {t_mesh:.3f} s  build_stencils (device + host plans) {t_build:.3f} s  "
              f"get_stencils read-back {t_get:.3f} s  rows {len(st['center'])}", flush=True)
