"""ctypes front end of the CPU oracles (TEST INFRASTRUCTURE ONLY).

Loads either ``oracle/_ref/libpmgref.so`` (the unmodified reference driven by
``oracle/ref_capi.cpp``) or ``oracle/_ref/libpmgport.so`` (our restatement
``oracle/pmg_oracle.cpp``); both implement ``oracle/oc_api.h``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu baseline
and ``--impl reference``) may import this module.  The product package
``paper_2205_09411_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpmgref.so")
PORT_SO = os.path.join(HERE, "_ref", "libpmgport.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class LsfT(C.Structure):
    """pmg_lsf_t (include/pmg_types.h)."""

    _fields_ = [
        ("shape", C.c_int32),
        ("cylindrical", C.c_int32),
        ("center", C.c_double * 3),
        ("radius", C.c_double),
        ("seg_a", C.c_double * 3),
        ("seg_b", C.c_double * 3),
        ("boundary_value", C.c_double),
        ("shift_p", C.c_double),
        ("shift_q", C.c_double),
        ("scale", C.c_double),
    ]


class StencilCfgT(C.Structure):
    _fields_ = [
        ("eps_tol", C.c_double),
        ("max_bracket_iters", C.c_int32),
        ("d_min", C.c_double),
        ("w_min", C.c_double),
        ("boundary_safety", C.c_double),
        ("thin_rescue", C.c_int32),
    ]


class MgCfgT(C.Structure):
    _fields_ = [
        ("n_down", C.c_int32),
        ("n_up", C.c_int32),
        ("coarse_rel_tol", C.c_double),
        ("coarse_max_iters", C.c_int32),
        ("threads", C.c_int32),
    ]


class StatsT(C.Structure):
    _fields_ = [("max_resid", C.c_double), ("l2_resid", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def lsf_array(specs):
    """specs: list of dicts (root first, then composite children)."""
    arr = (LsfT * len(specs))()
    for i, s in enumerate(specs):
        a = arr[i]
        a.shape = int(s.get("shape", 1))
        a.cylindrical = int(s.get("cylindrical", 0))
        for k, v in enumerate(s.get("center", (0, 0, 0))):
            a.center[k] = v
        a.radius = s.get("radius", 0.25)
        for k, v in enumerate(s.get("seg_a", (0, 0, 0))):
            a.seg_a[k] = v
        for k, v in enumerate(s.get("seg_b", (0, 0, 0))):
            a.seg_b[k] = v
        a.boundary_value = s.get("boundary_value", 0.0)
        a.shift_p = s.get("shift_p", 0.5)
        a.shift_q = s.get("shift_q", 0.5)
        a.scale = s.get("scale", 4.0)
    return arr


_LIBS = {}


def load(path):
    if path in _LIBS:
        return _LIBS[path]
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    vp = C.c_void_p
    lib.oc_create.restype = vp
    lib.oc_create.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
    lib.oc_destroy.argtypes = [vp]
    lib.oc_last_error.restype = C.c_char_p
    lib.oc_last_error.argtypes = [vp]
    lib.oc_build_uniform.argtypes = [vp, C.c_int]
    lib.oc_refine_band.argtypes = [vp, C.c_void_p, C.c_int, C.c_double, C.c_int]
    lib.oc_refine_crit.argtypes = [vp, C.c_int, C.c_double, C.c_double, _f64p, C.c_int]
    lib.oc_adapt.argtypes = [vp, C.c_void_p, C.c_int, C.c_int]
    lib.oc_n_blocks.argtypes = [vp]
    lib.oc_n_levels.argtypes = [vp]
    lib.oc_get_topology.argtypes = [vp, _i32p, _i32p, _f64p, _f64p, _i32p, _i32p, _i32p, _i32p]
    lib.oc_level_blocks.argtypes = [vp, C.c_int, _i32p]
    lib.oc_set_face_bc.argtypes = [vp, C.c_int, C.c_int, C.c_double, _f64p]
    lib.oc_set_field.argtypes = [vp, C.c_int, _f64p]
    lib.oc_get_field.argtypes = [vp, C.c_int, _f64p]
    lib.oc_build_stencils.argtypes = [vp, C.c_void_p, C.c_int, C.POINTER(StencilCfgT)]
    lib.oc_stencil_summary.argtypes = [vp, _i32p, _i32p]
    lib.oc_get_stencils.argtypes = [vp, _i32p, _f64p, _f64p, _f64p, _f64p, _i8p, _u8p, _i8p, _i32p]
    lib.oc_set_stencils.argtypes = [vp, _i32p, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p, _i8p,
                                    _u8p, _i8p, _i32p, C.c_int, _f64p]
    lib.oc_set_boundary_value.argtypes = [vp, C.c_int, C.c_double]
    lib.oc_solver_create.argtypes = [vp, C.POINTER(MgCfgT)]
    for n in ("oc_init", "oc_coarse_solve"):
        getattr(lib, n).argtypes = [vp]
    for n in ("oc_v_cycle", "oc_fmg_cycle", "oc_measure_residual"):
        getattr(lib, n).argtypes = [vp, C.POINTER(StatsT)]
    for n in ("oc_gsrb_sweep", "oc_fill_ghosts"):
        getattr(lib, n).argtypes = [vp, C.c_int, C.c_int]
    for n in ("oc_apply_pins", "oc_residual_level", "oc_restrict_level",
              "oc_restrict_level_no_guess", "oc_prolong_correction", "oc_prolong_full",
              "oc_set_have_guess"):
        getattr(lib, n).argtypes = [vp, C.c_int]
    lib.oc_coarse_sizes.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32)]
    lib.oc_coarse_get.argtypes = [vp, _i32p, _i32p, _f64p, _f64p, _f64p, _i32p, _i32p]
    lib.oc_bicgstab_probe.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_double)]
    _LIBS[path] = lib
    return lib


class Oracle:
    """One oracle context: a reference TreeMesh + StencilSet + MgSolver."""

    def __init__(self, dim, N, lo, hi, which="ref"):
        path = {"ref": REF_SO, "port": PORT_SO}.get(which, which)
        self.lib = load(path)
        self.dim, self.N = dim, N
        self.h = self.lib.oc_create(dim, N, np.ascontiguousarray(lo, np.float64),
                                    np.ascontiguousarray(hi, np.float64))
        self._check(0)
        self.F = 2 * dim
        self.S = (N + 2) ** dim
        self.NI = N ** dim

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.oc_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.oc_last_error(self.h).decode())
        err = self.lib.oc_last_error(self.h)
        if err:
            raise OracleError(-1, err.decode())

    # ---- mesh ---------------------------------------------------------------
    def build_uniform(self, levels):
        self._check(self.lib.oc_build_uniform(self.h, levels))

    def refine_band(self, lsf_specs, band, max_level):
        arr = lsf_array(lsf_specs)
        self._check(self.lib.oc_refine_band(self.h, C.cast(arr, C.c_void_p), len(lsf_specs),
                                            band, max_level))

    def refine_crit(self, kind, p0, p1, centre, max_level):
        c = np.zeros(3)
        c[:len(centre)] = centre
        self._check(self.lib.oc_refine_crit(self.h, kind, p0, p1, c, max_level))

    def adapt_refine(self, ids, max_level):
        flags = np.zeros(self.n_blocks, np.uint8)
        flags[np.asarray(list(ids), np.int64)] = 1
        self._check(self.lib.oc_adapt(self.h, flags.ctypes.data_as(C.c_void_p), flags.size, max_level))

    @property
    def n_blocks(self):
        return self.lib.oc_n_blocks(self.h)

    @property
    def n_levels(self):
        return self.lib.oc_n_levels(self.h)

    def topology(self):
        nb = self.n_blocks
        t = dict(level=np.zeros(nb, np.int32), coords=np.zeros((nb, 3), np.int32),
                 origin=np.zeros((nb, 3)), dx=np.zeros(nb), parent=np.zeros(nb, np.int32),
                 children=np.zeros((nb, 8), np.int32), nbr=np.zeros((nb, 6), np.int32),
                 cnbr=np.zeros((nb, 6), np.int32))
        self._check(self.lib.oc_get_topology(self.h, t["level"], t["coords"], t["origin"],
                                             t["dx"], t["parent"], t["children"], t["nbr"],
                                             t["cnbr"]))
        return t

    def level_blocks(self, level):
        ids = np.zeros(max(self.n_blocks, 1), np.int32)
        n = self.lib.oc_level_blocks(self.h, level, ids)
        return ids[:n].copy()

    def set_face_bc(self, d, typ=0, c=0.0, g=(0.0, 0.0, 0.0)):
        self._check(self.lib.oc_set_face_bc(self.h, d, typ, c, np.asarray(g, np.float64)))

    def set_field(self, var, buf):
        buf = np.ascontiguousarray(buf, np.float64).reshape(-1)
        assert buf.size == self.n_blocks * self.S
        self._check(self.lib.oc_set_field(self.h, var, buf))

    def face_gradient(self, var=0, var_out=4):
        """pmg::face_gradient on the reference build (fields.hpp:149-232): (leaf_ids,
        faces[leaf, axis, face_index]); the magnitude lands in field var_out."""
        fn = getattr(self.lib, "oc_face_gradient", None)
        if fn is None:
            raise NotImplementedError("face_gradient: reference build only")
        fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        nl = fn(self.h, var, var_out, None, None)
        if nl < 0:
            self._check(-1)
        pa = (self.N + 1) * self.N ** (self.dim - 1)
        faces = np.zeros((nl, self.dim, pa))
        ids = np.zeros(nl, np.int32)
        if fn(self.h, var, var_out, faces.ctypes.data, ids.ctypes.data) != nl:
            self._check(-1)
        return ids, faces

    def error_norms(self, phi_b, a=1.0, R=0.25, sphere3d=True, volume_weighted=False, var=0):
        """pmg::error_norms against pmg::AnalyticSolution on the reference build."""
        fn = getattr(self.lib, "oc_error_norms", None)
        if fn is None:
            raise NotImplementedError("error_norms: reference build only")
        fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_void_p]
        out = np.zeros(2)
        if fn(self.h, var, 1 if sphere3d else 0, phi_b, a, R, int(volume_weighted), out.ctypes.data) != 0:
            self._check(-1)
        return float(out[0]), float(out[1])

    def get_field(self, var):
        buf = np.zeros(self.n_blocks * self.S)
        self._check(self.lib.oc_get_field(self.h, var, buf))
        return buf.reshape(self.n_blocks, self.S)

    # ---- stencils -------------------------------------------------------------
    def build_stencils(self, lsf_specs, eps_tol=1e-8, max_bracket_iters=45, d_min=1e-4,
                       w_min=1e-3, boundary_safety=1.5, thin_rescue=True):
        arr = lsf_array(lsf_specs)
        cfg = StencilCfgT(eps_tol, max_bracket_iters, d_min, w_min, boundary_safety,
                          int(thin_rescue))
        self._check(self.lib.oc_build_stencils(self.h, C.cast(arr, C.c_void_p),
                                               len(lsf_specs), C.byref(cfg)))

    def get_stencils(self):
        nb, F = self.n_blocks, self.F
        boundary = np.zeros(nb, np.int32)
        rc = np.zeros(nb, np.int32)
        R = self.lib.oc_stencil_summary(self.h, boundary, rc)
        if R < 0:
            self._check(-R)
        R1 = max(R, 1)
        s = dict(boundary=boundary, row_count=rc, row_of=np.zeros(nb * self.NI, np.int32),
                 center=np.zeros(R1), nb=np.zeros(R1 * F), bc=np.zeros(R1 * F),
                 d=np.zeros(R1 * F), obj=np.zeros(R1 * F, np.int8), mask=np.zeros(R1, np.uint8),
                 pin_obj=np.zeros(R1, np.int8), lin=np.zeros(R1, np.int32))
        self._check(self.lib.oc_get_stencils(self.h, s["row_of"], s["center"], s["nb"], s["bc"],
                                             s["d"], s["obj"], s["mask"], s["pin_obj"],
                                             s["lin"]))
        for k in ("center", "mask", "pin_obj", "lin"):
            s[k] = s[k][:R]
        for k in ("nb", "bc", "d", "obj"):
            s[k] = s[k][:R * F]
        s["row_of"] = s["row_of"].reshape(nb, self.NI)
        return s

    def set_stencils(self, s, phi_b):
        F = self.F
        R = int(np.sum(s["row_count"]))
        R1 = max(R, 1)

        def pad(a, n, dt):
            out = np.zeros(n, dt)
            a = np.asarray(a, dt).reshape(-1)
            out[:a.size] = a
            return out
        self._check(self.lib.oc_set_stencils(
            self.h, np.ascontiguousarray(s["boundary"], np.int32),
            np.ascontiguousarray(s["row_count"], np.int32),
            np.ascontiguousarray(np.asarray(s["row_of"]).reshape(-1), np.int32),
            pad(s["center"], R1, np.float64), pad(s["nb"], R1 * F, np.float64),
            pad(s["bc"], R1 * F, np.float64), pad(s["d"], R1 * F, np.float64),
            pad(s["obj"], R1 * F, np.int8), pad(s["mask"], R1, np.uint8),
            pad(s["pin_obj"], R1, np.int8), pad(s["lin"], R1, np.int32), len(phi_b),
            np.ascontiguousarray(phi_b, np.float64)))

    def set_boundary_value(self, obj, v):
        self._check(self.lib.oc_set_boundary_value(self.h, obj, v))

    # ---- solver ---------------------------------------------------------------
    def solver_create(self, n_down=2, n_up=2, coarse_rel_tol=1e-6, coarse_max_iters=2000,
                      threads=1):
        cfg = MgCfgT(n_down, n_up, coarse_rel_tol, coarse_max_iters, threads)
        self._check(self.lib.oc_solver_create(self.h, C.byref(cfg)))

    def _stats(self, fn):
        st = StatsT()
        self._check(fn(self.h, C.byref(st)))
        return st.max_resid, st.l2_resid

    def init(self):
        self._check(self.lib.oc_init(self.h))

    def v_cycle(self):
        return self._stats(self.lib.oc_v_cycle)

    def fmg_cycle(self):
        return self._stats(self.lib.oc_fmg_cycle)

    def measure_residual(self):
        return self._stats(self.lib.oc_measure_residual)

    def gsrb_sweep(self, level, parity):
        self._check(self.lib.oc_gsrb_sweep(self.h, level, parity))

    def fill_ghosts(self, level, var=0):
        self._check(self.lib.oc_fill_ghosts(self.h, level, var))

    def apply_pins(self, level):
        self._check(self.lib.oc_apply_pins(self.h, level))

    def residual_level(self, level):
        self._check(self.lib.oc_residual_level(self.h, level))

    def restrict_level(self, level):
        self._check(self.lib.oc_restrict_level(self.h, level))

    def restrict_level_no_guess(self, level):
        self._check(self.lib.oc_restrict_level_no_guess(self.h, level))

    def prolong_correction(self, level):
        self._check(self.lib.oc_prolong_correction(self.h, level))

    def prolong_full(self, level):
        self._check(self.lib.oc_prolong_full(self.h, level))

    def coarse_solve(self):
        self._check(self.lib.oc_coarse_solve(self.h))

    def set_have_guess(self, v):
        self._check(self.lib.oc_set_have_guess(self.h, int(bool(v))))

    def bicgstab_probe(self):
        c, it, rel = C.c_int32(), C.c_int32(), C.c_double()
        self._check(self.lib.oc_bicgstab_probe(self.h, C.byref(c), C.byref(it), C.byref(rel)))
        return bool(c.value), it.value, rel.value

    def coarse_system(self):
        n, nnz, no = C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self.lib.oc_coarse_sizes(self.h, C.byref(n), C.byref(nnz), C.byref(no)))
        n, nnz, no = n.value, nnz.value, no.value
        cs = dict(n=n, rp=np.zeros(n + 1, np.int32), ci=np.zeros(max(nnz, 1), np.int32),
                  val=np.zeros(max(nnz, 1)), c0=np.zeros(max(n, 1)),
                  cobj=np.zeros(max(no * n, 1)), unk_block=np.zeros(max(n, 1), np.int32),
                  unk_lin=np.zeros(max(n, 1), np.int32))
        self._check(self.lib.oc_coarse_get(self.h, cs["rp"], cs["ci"], cs["val"], cs["c0"],
                                           cs["cobj"], cs["unk_block"], cs["unk_lin"]))
        cs["ci"], cs["val"] = cs["ci"][:nnz], cs["val"][:nnz]
        cs["c0"], cs["unk_block"], cs["unk_lin"] = cs["c0"][:n], cs["unk_block"][:n], cs["unk_lin"][:n]
        cs["cobj"] = cs["cobj"][:no * n].reshape(no, n)
        return cs
