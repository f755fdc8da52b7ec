"""Python mirror of the reference's solver API over the B200 C-ABI.

    mesh = build_uniform(3, lo, hi, 16, 5)              # host topology (mesh.py)
    dev = DeviceMesh(mesh)                              # fields live in HBM
    stencils = build_stencils(dev, lsf, StencilBuildConfig(w_min=...))  # GPU (K5)
    solver = MgSolver(dev, stencils, MgConfig())        # multigrid.hpp:295-299
    stats = solver.v_cycle()                            # CycleStats

Names, argument meaning and error behaviour follow pmg::MgSolver
(proj/include/pmg/multigrid.hpp:292-792), pmg::build_stencils
(stencil.hpp:207-222) and TreeMesh::field (mesh.hpp:118-125).  Errors raise
``PmgError`` carrying the reference's exception text.
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Mapping
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mesh import DIRICHLET, VAR_OLD, VAR_PHI, VAR_RES, VAR_RHS, LevelSetSpec, TreeMesh

LAYOUT_PADDED, LAYOUT_INTERIOR = 0, 1


@dataclass
class CycleStats:
    max_resid: float = 0.0
    l2_resid: float = 0.0


def face_gradient(dev: "DeviceMesh", var: int = 0, magnitude: bool = True):
    """pmg::face_gradient (fields.hpp:149-232) on the device: the staggered
    gradient of PHI on the faces of every leaf cell, leaves in dump order.

    Returns (leaf_ids, faces, mag): faces[leaf, axis, FaceField::face_index]
    with (N+1) N^(dim-1) faces per axis; mag[leaf, i + N (j + N k)] the
    cell-centred magnitude the reference writes to var_out (None if not asked).
    """
    lib, h = dev.lib, dev.h
    nl = lib.pmg_b200_n_leaves(h)
    pa = (dev.N + 1) * dev.N ** (dev.dim - 1)
    faces = np.zeros((nl, dev.dim, pa))
    mag = np.zeros((nl, dev.NI)) if magnitude else None
    ids = np.zeros(nl, np.int32)
    dev._check(lib.pmg_b200_face_gradient(h, var, faces.reshape(-1),
                                          mag.ctypes.data if magnitude else None, ids.ctypes.data))
    return ids, faces, mag


def write_dump(dev: "DeviceMesh", path: str, field_name: str = "phi", var: int = 0):
    """pmg::write_dump (io.hpp:23-71) straight from the device: the "pmg dump 1"
    file of the leaf blocks, byte-identical to the reference's."""
    dev._check(dev.lib.pmg_b200_write_dump(dev.h, var, os.fsencode(path), field_name.encode()))


def error_norms(dev: "DeviceMesh", phi_b: float, a: float = 1.0, R: float = 0.25, sphere3d: bool = True,
                volume_weighted: bool = False, var: int = 0):
    """pmg::error_norms against pmg::AnalyticSolution (fields.hpp:9-69) on the
    device: (linf, l2) of PHI minus phi_b + a (1 - R/r) (3D) or
    phi_b + a log(r/R) (2D) over the solved leaf cells."""
    linf, l2 = C.c_double(), C.c_double()
    dev._check(dev.lib.pmg_b200_error_norms(dev.h, var, 1 if sphere3d else 0, phi_b, a, R, int(volume_weighted),
                                            C.byref(linf), C.byref(l2)))
    return linf.value, l2.value


@dataclass
class MgConfig:
    """pmg::MgConfig (multigrid.hpp:12-28); threads is accepted and ignored."""

    n_down: int = 2
    n_up: int = 2
    coarse_rel_tol: float = 1e-6
    coarse_max_iters: int = 2000
    threads: int = 1


@dataclass
class StencilBuildConfig:
    """pmg::StencilBuildConfig + RootSearchConfig (stencil.hpp:115-120, levelset.hpp:170-183)."""

    eps_tol: float = 1e-8
    max_bracket_iters: int = 45
    d_min: float = 1e-4
    w_min: float = 1e-3
    boundary_safety: float = 1.5
    thin_rescue: bool = True


class StencilSet(dict):
    """Host image of pmg::StencilSet: boundary, row_count, row_of (nb x N^D),
    center, nb, bc, d, obj, mask, pin_obj, lin (rows in block-id order), phi_b."""

    @property
    def n_rows(self):
        return int(np.sum(self["row_count"]))

    def set_boundary_value(self, obj, value):
        self["phi_b"][obj] = value


def _lsf_array(descs):
    arr = (_lib.LsfT * len(descs))()
    for i, s in enumerate(descs):
        a = arr[i]
        a.shape = int(s["shape"])
        a.cylindrical = int(s.get("cylindrical", 0))
        for k in range(3):
            a.center[k] = s["center"][k]
            a.seg_a[k] = s["seg_a"][k]
            a.seg_b[k] = s["seg_b"][k]
        a.radius = s["radius"]
        a.boundary_value = s["boundary_value"]
        a.shift_p, a.shift_q, a.scale = s["shift_p"], s["shift_q"], s["scale"]
    return arr


class DeviceMesh:
    """A TreeMesh bound to one GPU context: topology, face BCs and every cell
    field (VAR_PHI/RHS/RES/OLD) in HBM."""

    def __init__(self, mesh: TreeMesh, device: int = 0, tree=None):
        """mesh: the host TreeMesh mirror.  tree: a DeviceTree (tree.py) -- the
        topology then comes from the device tables (pmg_b200_set_mesh_from_tree)
        and `mesh` may be None (a mirror is filled from the same tables)."""
        self.lib = _lib.load()
        if tree is not None and mesh is None:
            mesh = tree.to_host_mesh()
        self.mesh = mesh
        self.dim, self.N = mesh.dim, mesh.N
        self.NI = self.N ** self.dim
        self.S = (self.N + 2) ** self.dim
        lo = np.zeros(3)
        hi = np.zeros(3)
        lo[:self.dim], hi[:self.dim] = mesh.lo, mesh.hi
        self.h = self.lib.pmg_b200_create(self.dim, self.N, lo, hi, device)
        if not self.h:
            raise MemoryError("pmg_b200_create failed")
        self._check_err()
        if tree is not None:
            self._check(self.lib.pmg_b200_set_mesh_from_tree(self.h, tree.h))
        else:
            t = mesh.topology_arrays()
            self._check(self.lib.pmg_b200_set_mesh(self.h, mesh.n_blocks, t["level"], t["coords"],
                                                   t["origin"], t["dx"], t["parent"],
                                                   t["children"], t["nbr"], t["cnbr"]))
        self.sync_face_bc()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.pmg_b200_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check_err(self):
        e = self.lib.pmg_b200_last_error(self.h)
        if e:
            raise _lib.PmgError(_lib.PMG_ERR_INVALID_ARG, e.decode())

    def _check(self, rc):
        if rc != 0:
            raise _lib.PmgError(rc, self.lib.pmg_b200_last_error(self.h).decode())

    def sync_face_bc(self):
        """Push mesh.face_bc (types + evaluated Dirichlet values) to the device."""
        for d in range(2 * self.dim):
            fb = self.mesh.face_bc[d]
            vals = self.mesh.face_bc_values(d) if fb.type == DIRICHLET else None
            ptr = None
            if vals is not None:
                vals = np.ascontiguousarray(vals, np.float64)
                self._bcvals = getattr(self, "_bcvals", {})
                self._bcvals[d] = vals
                ptr = vals.ctypes.data_as(C.c_void_p)
            self._check(self.lib.pmg_b200_set_face_bc(self.h, d, fb.type, ptr))

    @property
    def stream(self):
        return self.lib.pmg_b200_stream(self.h)

    # ---- fields (TreeMesh::field) -------------------------------------------
    def set_field(self, var, values, layout=LAYOUT_PADDED, level=0):
        per = self.S if layout == LAYOUT_PADDED else self.NI
        nb = self.mesh.n_blocks if level == 0 else len(self.mesh.level_blocks(level))
        v = np.ascontiguousarray(values, np.float64)
        if v.size != nb * per:
            raise ValueError(f"field has {v.size} values, expected {nb * per}")
        if level == 0:
            self._check(self.lib.pmg_b200_upload_field(self.h, var, v.ctypes.data_as(C.c_void_p), layout))
        else:
            self._check(self.lib.pmg_b200_upload_level_field(self.h, var, level,
                                                             v.ctypes.data_as(C.c_void_p), layout))

    def get_field(self, var, layout=LAYOUT_PADDED, level=0):
        per = self.S if layout == LAYOUT_PADDED else self.NI
        nb = self.mesh.n_blocks if level == 0 else len(self.mesh.level_blocks(level))
        out = np.zeros(nb * per)
        if level == 0:
            self._check(self.lib.pmg_b200_download_field(self.h, var, out.ctypes.data_as(C.c_void_p), layout))
        else:
            self._check(self.lib.pmg_b200_download_level_field(self.h, var, level,
                                                               out.ctypes.data_as(C.c_void_p), layout))
        return out.reshape(nb, per)

    # ---- stencils -------------------------------------------------------------
    def set_stencils(self, st: StencilSet):
        F = 2 * self.dim
        R = st.n_rows
        R1 = max(R, 1)

        def pad(a, n, dt):
            out = np.zeros(n, dt)
            a = np.asarray(a, dt).reshape(-1)
            out[:a.size] = a
            return out
        phi_b = np.ascontiguousarray(st["phi_b"], np.float64)
        self._check(self.lib.pmg_b200_set_stencils(
            self.h, np.ascontiguousarray(st["boundary"], np.int32),
            np.ascontiguousarray(st["row_count"], np.int32),
            np.ascontiguousarray(np.asarray(st["row_of"]).reshape(-1), np.int32),
            pad(st["center"], R1, np.float64), pad(st["nb"], R1 * F, np.float64),
            pad(st["bc"], R1 * F, np.float64), pad(st["d"], R1 * F, np.float64),
            pad(st["obj"], R1 * F, np.int8), pad(st["mask"], R1, np.uint8),
            pad(st["pin_obj"], R1, np.int8), pad(st["lin"], R1, np.int32), len(phi_b),
            phi_b if phi_b.size else np.zeros(1)))

    def get_stencils(self, phi_b=None) -> StencilSet:
        nb, F = self.mesh.n_blocks, 2 * self.dim
        boundary = np.zeros(nb, np.int32)
        rc = np.zeros(nb, np.int32)
        R = self.lib.pmg_b200_stencil_summary(self.h, boundary, rc)
        if R < 0:
            self._check(-R)
        R1 = max(R, 1)
        s = StencilSet(boundary=boundary, row_count=rc, row_of=np.zeros(nb * self.NI, np.int32),
                       center=np.zeros(R1), nb=np.zeros(R1 * F), bc=np.zeros(R1 * F),
                       d=np.zeros(R1 * F), obj=np.zeros(R1 * F, np.int8),
                       mask=np.zeros(R1, np.uint8), pin_obj=np.zeros(R1, np.int8),
                       lin=np.zeros(R1, np.int32))
        self._check(self.lib.pmg_b200_get_stencils(self.h, s["row_of"], s["center"], s["nb"],
                                                   s["bc"], s["d"], s["obj"], s["mask"],
                                                   s["pin_obj"], s["lin"]))
        for k in ("center", "mask", "pin_obj", "lin"):
            s[k] = s[k][:R]
        for k in ("nb", "bc", "d", "obj"):
            s[k] = s[k][:R * F]
        s["row_of"] = s["row_of"].reshape(nb, self.NI)
        s["phi_b"] = np.array(phi_b if phi_b is not None else [], np.float64)
        return s


class DeviceStencils(Mapping):
    """The StencilSet built on the device (build_stencils).  The solver reads
    the device copy; the host image (a StencilSet) is read back only when an
    item is first accessed (parity checks, the C++ drop-in's bit comparison)."""

    def __init__(self, dev: DeviceMesh, phi_b):
        self._dev, self._phi_b, self._s = dev, list(phi_b), None

    def host(self) -> StencilSet:
        if self._s is None:
            self._s = self._dev.get_stencils(self._phi_b)
        return self._s

    def __getitem__(self, k):
        return self.host()[k]

    def __setitem__(self, k, v):
        self.host()[k] = v

    def __iter__(self):
        return iter(self.host())

    def __len__(self):
        return len(self.host())

    @property
    def n_rows(self):
        return self.host().n_rows


def build_stencils(dev: DeviceMesh, lsf: LevelSetSpec, cfg: StencilBuildConfig) -> DeviceStencils:
    """pmg::build_stencils (stencil.hpp:207-222), evaluated on the GPU."""
    descs = lsf.as_descs()
    arr = _lsf_array(descs)
    c = _lib.StencilCfgT(cfg.eps_tol, cfg.max_bracket_iters, cfg.d_min, cfg.w_min,
                         cfg.boundary_safety, int(cfg.thin_rescue))
    dev._check(dev.lib.pmg_b200_build_stencils(dev.h, C.cast(arr, C.c_void_p), len(descs),
                                               C.byref(c)))
    phi_b = [lsf.object(i).boundary_value for i in range(lsf.n_objects())]
    return DeviceStencils(dev, phi_b)


class MgSolver:
    """pmg::MgSolver<Dim> on the B200 (multigrid.hpp:292-792)."""

    def __init__(self, dev: DeviceMesh, stencils: StencilSet | None, cfg: MgConfig | None = None):
        self.dev = dev
        self.lib = dev.lib
        self.h = dev.h
        if stencils is not None and not (isinstance(stencils, DeviceStencils) and stencils._dev is dev):
            dev.set_stencils(stencils if not isinstance(stencils, DeviceStencils) else stencils.host())
        self.stencils = stencils
        cfg = cfg or MgConfig()
        self.cfg = cfg
        c = _lib.MgCfgT(cfg.n_down, cfg.n_up, cfg.coarse_rel_tol, cfg.coarse_max_iters,
                        cfg.threads)
        dev._check(self.lib.pmg_b200_solver_create(self.h, C.byref(c)))

    def _stats(self, fn):
        st = _lib.StatsT()
        self.dev._check(fn(self.h, C.byref(st)))
        return CycleStats(st.max_resid, st.l2_resid)

    def init(self):
        self.dev._check(self.lib.pmg_b200_init(self.h))

    def run_cycle(self, fmg=False):
        return self.fmg_cycle() if fmg else self.v_cycle()

    def v_cycle(self):
        return self._stats(self.lib.pmg_b200_v_cycle)

    def fmg_cycle(self):
        return self._stats(self.lib.pmg_b200_fmg_cycle)

    def measure_residual(self):
        return self._stats(self.lib.pmg_b200_measure_residual)

    def v_cycle_async(self):
        self.dev._check(self.lib.pmg_b200_v_cycle_async(self.h))

    def fmg_cycle_async(self):
        self.dev._check(self.lib.pmg_b200_fmg_cycle_async(self.h))

    def cycle_result(self):
        return self._stats(self.lib.pmg_b200_cycle_result)

    def gsrb_sweep(self, level, parity):
        self.dev._check(self.lib.pmg_b200_gsrb_sweep(self.h, level, parity))

    def fill_ghosts(self, level, var=VAR_PHI):
        self.dev._check(self.lib.pmg_b200_fill_ghosts(self.h, level, var))

    def apply_pins(self, level):
        self.dev._check(self.lib.pmg_b200_apply_pins(self.h, level))

    def residual_level(self, level):
        self.dev._check(self.lib.pmg_b200_residual_level(self.h, level))

    def restrict_level(self, level):
        self.dev._check(self.lib.pmg_b200_restrict_level(self.h, level))

    def restrict_level_no_guess(self, level):
        self.dev._check(self.lib.pmg_b200_restrict_level_no_guess(self.h, level))

    def prolong_correction(self, level):
        self.dev._check(self.lib.pmg_b200_prolong_correction(self.h, level))

    def prolong_full(self, level):
        self.dev._check(self.lib.pmg_b200_prolong_full(self.h, level))

    def coarse_solve(self):
        self.dev._check(self.lib.pmg_b200_coarse_solve(self.h))

    def set_have_guess(self, v):
        self.dev._check(self.lib.pmg_b200_set_have_guess(self.h, int(bool(v))))

    def set_boundary_value(self, obj, value):
        self.dev._check(self.lib.pmg_b200_set_boundary_value(self.h, obj, value))

    def kernel_count(self, kind=0):
        k = self.lib.pmg_b200_cycle_kernel_count(self.h, kind)
        if k < 0:
            self.dev._check(-k)
        return k

    def level_classes(self, level):
        """How the kernels split the blocks of ``level`` (pmg_b200_level_classes)."""
        out = np.zeros(8, np.int32)
        self.dev._check(self.lib.pmg_b200_level_classes(self.h, level, out))
        keys = ("blocks", "cf_faces", "gs_stream", "gs_tile", "record_stream", "record_tile",
                "restrict_stream", "restrict_tile")
        return dict(zip(keys, (int(v) for v in out)))

    def coarse_info(self):
        """(iterations, relative residual) of the last BiCGStab coarse solve."""
        it, rel = C.c_int32(), C.c_double()
        self.dev._check(self.lib.pmg_b200_coarse_info(self.h, C.byref(it), C.byref(rel)))
        return it.value, rel.value

    def time_op(self, op, level=0, reps=10):
        """Average device ms of one phase (pmg_b200_time_op)."""
        ms = C.c_double()
        self.dev._check(self.lib.pmg_b200_time_op(self.h, op, level, reps, C.byref(ms)))
        return ms.value

    def coarse_system(self):
        n, nnz, no = C.c_int32(), C.c_int32(), C.c_int32()
        self.dev._check(self.lib.pmg_b200_coarse_sizes(self.h, C.byref(n), C.byref(nnz), C.byref(no)))
        n, nnz, no = n.value, nnz.value, no.value
        cs = dict(n=n, rp=np.zeros(n + 1, np.int32), ci=np.zeros(max(nnz, 1), np.int32),
                  val=np.zeros(max(nnz, 1)), c0=np.zeros(max(n, 1)), cobj=np.zeros(max(no * n, 1)),
                  unk_block=np.zeros(max(n, 1), np.int32), unk_lin=np.zeros(max(n, 1), np.int32))
        self.dev._check(self.lib.pmg_b200_coarse_get(self.h, cs["rp"], cs["ci"], cs["val"], cs["c0"],
                                                     cs["cobj"], cs["unk_block"], cs["unk_lin"]))
        cs["ci"], cs["val"] = cs["ci"][:nnz], cs["val"][:nnz]
        cs["c0"], cs["unk_block"], cs["unk_lin"] = cs["c0"][:n], cs["unk_block"][:n], cs["unk_lin"][:n]
        cs["cobj"] = cs["cobj"][:no * n].reshape(no, n)
        return cs
