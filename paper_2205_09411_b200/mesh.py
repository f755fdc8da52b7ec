"""Host mirror of the reference's block-tree mesh (topology and geometry only).

Mirrors ``pmg::TreeMesh<Dim>`` (proj/include/pmg/mesh.hpp:60-561) for the parts
the solver path consumes: block table (level, coords, origin, dx, parent,
children), per-level block lists in the reference's x-major order
(mesh.hpp:101-105, 439-447), neighbour tables (rebuild_topology,
mesh.hpp:429-469), uniform construction (build_uniform, mesh.hpp:565-572) and
criterion-driven refinement with 2:1 balance (adapt/refine_balanced/do_refine,
mesh.hpp:157-199, 252-320; refine_by_criterion, harness.hpp:295-321).
Block ids follow the reference's creation order, so ids, level lists and
neighbour tables are identical to the reference's for the same sequence of
operations (checked against the reference in tests/test_mesh_host.py).

Cell fields do not live here: they live on the device context
(``paper_2205_09411_b200.solver.DeviceMesh``).  Coarsening (``adapt`` with
coarsen flags, ``compact``) is mesh construction outside the hot path and is
not mirrored.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

VAR_PHI, VAR_RHS, VAR_RES, VAR_OLD, VAR_AUX = 0, 1, 2, 3, 4
DIRICHLET, NEUMANN_ZERO = 0, 1


@dataclass
class FaceBc:
    """pmg::FaceBc (mesh.hpp:22-32): type + optional value(x) (None means 0)."""

    type: int = DIRICHLET
    value: Optional[Callable[[np.ndarray], np.ndarray]] = None  # vectorised over rows of x


def dir_axis(d):
    return d // 2


def dir_sign(d):
    return 1 if d & 1 else -1


class TreeMesh:
    """Block-structured quadtree/octree: all blocks hold N^D cells."""

    def __init__(self, dim, lo, hi, N):
        if N < 4 or (N & (N - 1)) != 0:
            raise ValueError("block size N must be a power of two and at least 4")
        self.dim = dim
        self.lo = np.array(lo, np.float64)[:dim]
        self.hi = np.array(hi, np.float64)[:dim]
        ext = self.hi[0] - self.lo[0]
        for k in range(dim):
            if abs((self.hi[k] - self.lo[k]) - ext) > 1e-12 * abs(ext):
                raise ValueError("domain must be square/cubic")
        if not ext > 0:
            raise ValueError("domain extent must be positive")
        self.N = N
        self.level = [1]
        self.coords = [(0,) * dim]
        self.origin = [tuple(float(v) for v in self.lo)]
        self.dx = [ext / N]
        self.parent = [-1]
        self.children = [[-1] * (1 << dim)]
        self.face_bc = [FaceBc() for _ in range(2 * dim)]
        self._maps = [None, {(0,) * dim: 0}]
        self._rebuild_topology()

    # ------------------------------------------------------------------ queries
    @property
    def n_blocks(self):
        return len(self.level)

    @property
    def n_levels(self):
        return len(self._levels) - 1

    def level_blocks(self, l):
        return self._levels[l]

    def level_dx(self, l):
        return (self.hi[0] - self.lo[0]) / (self.N * (1 << (l - 1)))

    def is_leaf(self, b):
        return self.children[b][0] < 0

    def leaves(self):
        """Leaf ids in dump order: level-major, lexicographic (mesh.hpp:229-235)."""
        return [b for l in range(1, self.n_levels + 1) for b in self._levels[l] if self.is_leaf(b)]

    def find_block(self, level, coords):
        if level < 1 or level >= len(self._maps):
            return -1
        return self._maps[level].get(tuple(coords), -1)

    def cell_centers(self, b):
        """(N^D, D) cell centres of block b in for_box order (x fastest):
        origin + (i + 0.5) dx (mesh.hpp:139-143)."""
        N, D = self.N, self.dim
        idx = np.indices((N,) * D)[::-1].reshape(D, -1).T  # x fastest
        o = np.array(self.origin[b])
        return o[None, :] + (idx + 0.5) * self.dx[b]

    # ------------------------------------------------------------------ refinement
    def _in_bounds(self, level, c):
        nb = 1 << (level - 1)
        return all(0 <= v < nb for v in c)

    def _do_refine(self, b):
        D, N = self.dim, self.N
        lvl = self.level[b] + 1
        while len(self._maps) <= lvl:
            self._maps.append({})
        for c in range(1 << D):
            bits = [(c >> k) & 1 for k in range(D)]
            cid = self.n_blocks
            self.level.append(lvl)
            self.coords.append(tuple(2 * self.coords[b][k] + bits[k] for k in range(D)))
            self.origin.append(tuple(self.origin[b][k] + bits[k] * (0.5 * N * self.dx[b])
                                     for k in range(D)))
            self.dx.append(0.5 * self.dx[b])
            self.parent.append(b)
            self.children.append([-1] * (1 << D))
            self.children[b][c] = cid
            self._maps[lvl][self.coords[cid]] = cid

    def _refine_balanced(self, b, max_level):
        if not self.is_leaf(b):
            return
        level = self.level[b]
        if level >= max_level:
            raise RuntimeError("2:1 balancing forced refinement beyond the maximum level")
        D = self.dim
        # enumerate_offsets order: axis 0 outermost (mesh.hpp:280-290)
        for off in itertools.product((-1, 0, 1), repeat=D):
            if all(o == 0 for o in off):
                continue
            nc = tuple(self.coords[b][k] + off[k] for k in range(D))
            if not self._in_bounds(level, nc):
                continue
            if self.find_block(level, nc) >= 0:
                continue
            pid = self.find_block(level - 1, tuple(v >> 1 for v in nc))
            assert pid >= 0, "2:1 balance invariant violated"
            if self.is_leaf(pid):
                self._refine_balanced(pid, max_level)
        self._do_refine(b)

    def adapt_refine(self, refine_ids, max_level):
        """adapt() with refine flags only (mesh.hpp:157-175,198)."""
        todo = []
        for b in refine_ids:
            if self.is_leaf(b):
                if self.level[b] >= max_level:
                    raise RuntimeError("refinement beyond the configured maximum level")
                todo.append(b)
        todo.sort(key=lambda b: (self.level[b], b))
        for b in todo:
            self._refine_balanced(b, max_level)
        self._rebuild_topology()

    def refine_all(self, times, max_level):
        for _ in range(times):
            self.adapt_refine([b for b in range(self.n_blocks) if self.is_leaf(b)], max_level)

    def refine_by_criterion(self, max_level, want):
        """harness.hpp:295-321.  want(mesh, b, x[N^D, D]) -> bool array over cells."""
        while True:
            flags = []
            for b in self.leaves():
                if self.level[b] >= max_level:
                    continue
                if np.any(want(self, b, self.cell_centers(b))):
                    flags.append(b)
            if not flags:
                return
            self.adapt_refine(flags, max_level)

    # ------------------------------------------------------------------ topology
    def _rebuild_topology(self):
        D = self.dim
        L = max(self.level)
        self._levels = [[] for _ in range(L + 1)]
        self._maps = [None] + [{} for _ in range(L)]
        for b in range(self.n_blocks):
            self._levels[self.level[b]].append(b)
            self._maps[self.level[b]][self.coords[b]] = b
        for lv in self._levels:
            lv.sort(key=lambda b: self.coords[b])  # x-major (mesh.hpp:439-447)
        self.nbr = [[-1] * (2 * D) for _ in range(self.n_blocks)]
        self.cnbr = [[-1] * (2 * D) for _ in range(self.n_blocks)]
        for b in range(self.n_blocks):
            for d in range(2 * D):
                nc = list(self.coords[b])
                nc[dir_axis(d)] += dir_sign(d)
                if not self._in_bounds(self.level[b], nc):
                    continue
                nid = self.find_block(self.level[b], nc)
                if nid >= 0:
                    self.nbr[b][d] = nid
                else:
                    cid = self.find_block(self.level[b] - 1, [v >> 1 for v in nc])
                    if cid < 0:
                        raise RuntimeError("ghost region has no covering block")
                    self.cnbr[b][d] = cid

    def topology_arrays(self):
        """Arrays in the C-ABI layout of pmg_b200_set_mesh."""
        nb, D = self.n_blocks, self.dim
        t = dict(level=np.array(self.level, np.int32),
                 coords=np.zeros((nb, 3), np.int32), origin=np.zeros((nb, 3)),
                 dx=np.array(self.dx, np.float64), parent=np.array(self.parent, np.int32),
                 children=np.full((nb, 8), -1, np.int32), nbr=np.full((nb, 6), -1, np.int32),
                 cnbr=np.full((nb, 6), -1, np.int32))
        t["coords"][:, :D] = np.array(self.coords, np.int32)
        t["origin"][:, :D] = np.array(self.origin, np.float64)
        t["children"][:, :1 << D] = np.array(self.children, np.int32)
        t["nbr"][:, :2 * D] = np.array(self.nbr, np.int32)
        t["cnbr"][:, :2 * D] = np.array(self.cnbr, np.int32)
        return t

    def face_bc_values(self, d):
        """Dirichlet ghost-face values bc(x_f) for every block with a physical face
        d, in block-id order (mesh.hpp:538-552); None if the face value is null."""
        fb = self.face_bc[d]
        if fb.value is None:
            return None
        D, N = self.dim, self.N
        axis, side = dir_axis(d), d & 1
        out = []
        idx = np.indices((N,) * (D - 1))[::-1].reshape(D - 1, -1).T  # lower axis fastest
        for b in range(self.n_blocks):
            if self.nbr[b][d] >= 0 or self.cnbr[b][d] >= 0:
                continue
            i1 = np.zeros((idx.shape[0], D), np.int64)
            others = [k for k in range(D) if k != axis]
            for q, k in enumerate(others):
                i1[:, k] = idx[:, q]
            i1[:, axis] = N - 1 if side else 0
            o = np.array(self.origin[b])
            xf = o[None, :] + (i1 + 0.5) * self.dx[b]
            half = 0.5 * self.dx[b] * dir_sign(d)
            xf[:, axis] += half
            out.append(np.asarray(fb.value(xf), np.float64).reshape(-1))
        return np.concatenate(out) if out else np.zeros(0)

    def lin(self, i):
        """Padded index (mesh.hpp:128-137)."""
        s = self.N + 2
        r, mul = i[0] + 1, s
        for k in range(1, self.dim):
            r += (i[k] + 1) * mul
            mul *= s
        return r


def build_uniform(dim, lo, hi, N, levels):
    """mesh.hpp:565-572."""
    if levels < 1:
        raise ValueError("levels must be at least 1")
    m = TreeMesh(dim, lo, hi, N)
    m.refine_all(levels - 1, levels)
    return m


# ---------------------------------------------------------------------- level sets
SHAPE_NONE, SHAPE_SPHERE, SHAPE_SPHEROID, SHAPE_RHOMBUS, SHAPE_HEART, SHAPE_ASTROID, \
    SHAPE_ROD, SHAPE_COMPOSITE_MIN = range(8)


@dataclass
class LevelSetSpec:
    """pmg::LevelSetSpec (levelset.hpp:31-52)."""

    shape: int = SHAPE_SPHERE
    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 0.25
    seg_a: tuple = (0.0, 0.0, 0.0)
    seg_b: tuple = (0.0, 0.0, 0.0)
    boundary_value: float = 0.0
    shift_p: float = 0.5
    shift_q: float = 0.5
    scale: float = 4.0
    cylindrical: bool = False
    children: list = field(default_factory=list)

    def n_objects(self):
        return len(self.children) if self.shape == SHAPE_COMPOSITE_MIN else 1

    def object(self, i):
        return self.children[i] if self.shape == SHAPE_COMPOSITE_MIN else self

    def as_descs(self):
        """pmg_lsf_t array: root first, then composite children."""
        d = lambda s: dict(shape=s.shape, cylindrical=int(s.cylindrical),
                           center=tuple(s.center) + (0.0,) * (3 - len(s.center)),
                           radius=s.radius, seg_a=tuple(s.seg_a) + (0.0,) * (3 - len(s.seg_a)),
                           seg_b=tuple(s.seg_b) + (0.0,) * (3 - len(s.seg_b)),
                           boundary_value=s.boundary_value, shift_p=s.shift_p,
                           shift_q=s.shift_q, scale=s.scale)
        out = [d(self)]
        if self.shape == SHAPE_COMPOSITE_MIN:
            out += [d(c) for c in self.children]
        return out


def lsf_eval_sphere(spec, x):
    """||x - c|| - R with the reference's sequential dot (core.hpp:57-67,
    levelset.hpp:85); x is (n, D)."""
    D = x.shape[1]
    s = np.zeros(x.shape[0])
    for k in range(D):
        a = x[:, k] - spec.center[k]
        s = s + a * a
    return np.sqrt(s) - spec.radius


def lsf_eval(spec, x):
    """Vectorised lsf_eval for sphere / composite-of-spheres / none (host-side
    mesh criteria only; the stencil build runs on the GPU)."""
    if spec.shape == SHAPE_NONE:
        return np.ones(x.shape[0])
    if spec.shape == SHAPE_SPHERE:
        return lsf_eval_sphere(spec, x)
    if spec.shape == SHAPE_COMPOSITE_MIN:
        f = np.full(x.shape[0], np.inf)
        for ch in spec.children:
            e = lsf_eval(ch, x)
            f = np.where(e < f, e, f)  # std::min(f, e)
        return f
    raise NotImplementedError("host-side lsf_eval supports sphere/composite/none")
