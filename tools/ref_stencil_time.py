"""The reference's build_stencils (oracle/_ref, unmodified reference code) timed
on the host's cores for the BASELINE configs: python tools/ref_stencil_time.py cfg2 cfg4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oc import Oracle  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    case = cfgs.get_case(name)
    o = Oracle(case.dim, case.N, case.lo[:case.dim], case.hi[:case.dim], "ref")
    o.build_uniform(case.levels)
    if case.amr_band > 0:
        o.refine_band(case.lsf.as_descs(), case.amr_band, case.max_level)
    for threads in (os.cpu_count() or 1,):
        t0 = time.perf_counter()
        o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)  # hardware_concurrency threads
        print(f"{name}: reference build_stencils {time.perf_counter() - t0:.3f} s on {threads} threads", flush=True)
