#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libpmgref.so,
built from /root/reference by `make -C oracle ref`).

Each fixture holds, for one seeded configuration at reduced size (inputs are
regenerated deterministically from paper_2205_09411_b200.configs):
  * the mesh topology (level, coords, parent, nbr, cnbr),
  * the reference's StencilSet (boundary flags, row_of, every row array),
  * the residual history of the configuration's cycle plan (measure, [FMG], V...),
  * the final phi of every block (interior, block-id order),
  * for the coarse system: n, nnz and the CSR arrays.
The fixtures pin the CPU restatement (tests/test_oracle.py) and serve the GPU
parity tests on boxes where /root/reference does not exist.

    python tools/gen_golden.py            # writes tests/golden/<case>.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import oracle_for_case  # noqa: E402
from paper_2205_09411_b200 import configs as cfgs  # noqa: E402

CASES = {"cfg1@4": 4, "cfg2@3": 3, "cfg3@5": 3, "cfg4@3": 3, "cfg5@3": 3}


def run(name, cycles, which="ref"):
    case = cfgs.get_case(name)
    mesh = case.build_mesh()
    o = oracle_for_case(case, mesh, which)
    o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)
    g = case.rhs_fields(mesh)
    o.set_field(1, cfgs.padded_from_interior(g, case.dim, case.N))
    o.solver_create()
    hist = [o.measure_residual()]
    plan = (["fmg"] if case.fmg_first else []) + ["v"] * cycles
    for k in plan:
        hist.append(o.fmg_cycle() if k == "fmg" else o.v_cycle())
    out = dict(history=np.array(hist, np.float64), plan=np.array(plan))
    t = o.topology()
    for k in ("level", "coords", "parent", "nbr", "cnbr"):
        out["topo_" + k] = t[k]
    s = o.get_stencils()
    for k, v in s.items():
        out["st_" + k] = np.asarray(v)
    out["st_row_of"] = s["row_of"][s["boundary"].astype(bool)]  # boundary blocks only
    phi = cfgs.interior_from_padded(o.get_field(0), case.dim, case.N)
    # full phi only as a hash (bit-exact port check); a strided sample and the
    # norms for tolerance checks on the GPU
    import hashlib
    out["phi_sha256"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(phi).tobytes()).digest(), np.uint8)
    out["phi_sample_idx"] = np.arange(0, phi.size, 7, dtype=np.int64)
    out["phi_sample"] = phi.reshape(-1)[out["phi_sample_idx"]]
    out["phi_max"] = np.array([np.max(np.abs(phi))])
    cs = o.coarse_system()
    for k in ("rp", "ci", "val", "c0", "cobj"):
        out["cs_" + k] = cs[k]
    return out


def main():
    d = os.path.join(ROOT, "tests", "golden")
    os.makedirs(d, exist_ok=True)
    for name, cyc in CASES.items():
        out = run(name, cyc)
        path = os.path.join(d, name.replace("@", "_L") + ".npz")
        np.savez_compressed(path, **out)
        print(f"{path}: {os.path.getsize(path) / 1e3:.0f} kB, history {out['history'][:, 0]}")


if __name__ == "__main__":
    main()
