"""The block tree on the device (csrc/tree.cu): the Python face of
``pmg_b200_tree_*`` (include/pmg_b200.h).

Mirrors the part of the reference's ``TreeMesh`` that builds and refines the
mesh -- the constructor, ``refine_all``, ``adapt`` with refine flags and the
2:1 balance (mesh.hpp:66-82, 157-175, 206-216, 253-320), ``rebuild_topology``
(mesh.hpp:429-469) -- and ``refine_by_criterion`` (harness.hpp:295-321) with
the criterion evaluated by a kernel.  Block ids, level lists and neighbour
tables are the reference's, bit for bit (tests/test_gpu_tree.py).  There is
no CPU fallback: every call runs kernels on the GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .mesh import FaceBc, LevelSetSpec, TreeMesh

CRIT_BAND, CRIT_RADIAL, CRIT_BALL = 0, 1, 2


class DeviceTree:
    def __init__(self, dim, lo, hi, N, device: int = 0):
        self.lib = _lib.load()
        self.dim, self.N, self.device = dim, N, device
        self.lo = np.zeros(3)
        self.hi = np.zeros(3)
        self.lo[:dim], self.hi[:dim] = np.asarray(lo, np.float64)[:dim], np.asarray(hi, np.float64)[:dim]
        self.h = self.lib.pmg_b200_tree_create(dim, N, self.lo, self.hi, device)
        if not self.h:
            raise MemoryError("pmg_b200_tree_create failed")
        e = self.lib.pmg_b200_tree_last_error(self.h)
        if e:
            msg = e.decode()
            self.lib.pmg_b200_tree_destroy(self.h)
            self.h = None
            raise _lib.PmgError(_lib.PMG_ERR_INVALID_ARG, msg)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.pmg_b200_tree_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise _lib.PmgError(rc, self.lib.pmg_b200_tree_last_error(self.h).decode())

    # ---- queries (mesh.hpp:94-105) --------------------------------------------
    @property
    def n_blocks(self):
        return self.lib.pmg_b200_tree_n_blocks(self.h)

    @property
    def n_levels(self):
        return self.lib.pmg_b200_tree_n_levels(self.h)

    @property
    def adapt_passes(self):
        return self.lib.pmg_b200_tree_adapt_passes(self.h)

    def level_blocks(self, l):
        n = C.c_int(0)
        self._check(self.lib.pmg_b200_tree_level_blocks(self.h, l, None, C.byref(n)))
        ids = np.zeros(max(n.value, 1), np.int32)
        self._check(self.lib.pmg_b200_tree_level_blocks(self.h, l, ids.ctypes.data_as(C.c_void_p), C.byref(n)))
        return ids[:n.value]

    def topology_arrays(self):
        """The Block table in the layout of pmg_b200_set_mesh (as TreeMesh.topology_arrays)."""
        nb = self.n_blocks
        t = dict(level=np.zeros(nb, np.int32), coords=np.zeros((nb, 3), np.int32),
                 origin=np.zeros((nb, 3)), dx=np.zeros(nb), parent=np.zeros(nb, np.int32),
                 children=np.zeros((nb, 8), np.int32), nbr=np.zeros((nb, 6), np.int32),
                 cnbr=np.zeros((nb, 6), np.int32))
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(self.lib.pmg_b200_tree_get(self.h, p(t["level"]), p(t["coords"]), p(t["origin"]),
                                               p(t["dx"]), p(t["parent"]), p(t["children"]),
                                               p(t["nbr"]), p(t["cnbr"])))
        return t

    # ---- refinement ---------------------------------------------------------------
    def refine_all(self, times, max_level):
        self._check(self.lib.pmg_b200_tree_refine_all(self.h, times, max_level))

    def adapt_refine(self, refine_ids, max_level):
        """adapt() with refine flags (mesh.hpp:157-175,198); returns the number of blocks refined."""
        flags = np.zeros(self.n_blocks, np.uint8)
        flags[np.asarray(list(refine_ids), np.int64)] = 1
        n = C.c_int(0)
        self._check(self.lib.pmg_b200_tree_adapt(self.h, flags.ctypes.data_as(C.c_void_p), flags.size, 0,
                                                 max_level, C.byref(n)))
        return n.value

    def refine_band(self, lsf: LevelSetSpec, band, max_level):
        """refine_by_criterion with want(b, x) = |f(x)| < band * b.dx."""
        from .solver import _lsf_array
        arr = _lsf_array(lsf.as_descs())
        self._check(self.lib.pmg_b200_tree_refine_by_criterion(
            self.h, CRIT_BAND, C.cast(arr, C.c_void_p), len(arr), float(band), 0.0, None, max_level))

    def _refine_centre(self, kind, p0, p1, centre, max_level):
        c = np.zeros(3)
        c[:self.dim] = np.asarray(centre, np.float64)[:self.dim]
        self._check(self.lib.pmg_b200_tree_refine_by_criterion(
            self.h, kind, None, 0, float(p0), float(p1), c.ctypes.data_as(C.c_void_p), max_level))

    def refine_radial(self, dx_min, R, centre, max_level):
        """want(b, x) = b.dx > dx_min * max(1, ||x - centre|| / R)  (harness.hpp:351-355)."""
        self._refine_centre(CRIT_RADIAL, dx_min, R, centre, max_level)

    def refine_ball(self, dx_tip, r_tip, tip, max_level):
        """want(b, x) = b.dx > dx_tip and ||x - tip|| < r_tip  (harness.hpp:413-418)."""
        self._refine_centre(CRIT_BALL, dx_tip, r_tip, tip, max_level)

    # ---- hand-over -----------------------------------------------------------------
    def to_host_mesh(self) -> TreeMesh:
        """Host mirror filled from the device tables (nothing recomputed): the
        Python helpers that generate fields and face values read it."""
        t = self.topology_arrays()
        D = self.dim
        m = TreeMesh.__new__(TreeMesh)
        m.dim, m.N = D, self.N
        m.lo, m.hi = self.lo[:D].copy(), self.hi[:D].copy()
        m.level = [int(v) for v in t["level"]]
        m.coords = [tuple(int(v) for v in r[:D]) for r in t["coords"]]
        m.origin = [tuple(float(v) for v in r[:D]) for r in t["origin"]]
        m.dx = [float(v) for v in t["dx"]]
        m.parent = [int(v) for v in t["parent"]]
        m.children = [[int(v) for v in r[:1 << D]] for r in t["children"]]
        m.nbr = [[int(v) for v in r[:2 * D]] for r in t["nbr"]]
        m.cnbr = [[int(v) for v in r[:2 * D]] for r in t["cnbr"]]
        m.face_bc = [FaceBc() for _ in range(2 * D)]
        L = self.n_levels
        m._levels = [[]] + [[int(v) for v in self.level_blocks(l)] for l in range(1, L + 1)]
        m._maps = [None] + [{m.coords[b]: b for b in m._levels[l]} for l in range(1, L + 1)]
        return m
