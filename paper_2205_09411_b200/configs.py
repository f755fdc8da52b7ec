"""The BASELINE.json configurations as seeded, host-generated synthetic inputs.

BASELINE names no public dataset: every input is synthetic, generated here on
the host (counter-based splitmix64) and uploaded, so the CPU
oracle and the GPU see bit-identical data.

  cfg1  2D [0,1]^2, 256^2 in 8^2 blocks (L=6), circle c=(.5,.5) R=.25 phi_b=1, g=0, 10 V
  cfg2  3D [0,1]^3, 256^3 in 16^3 blocks (L=5), sphere c=.5 R=.2 phi_b=1,
        g = 1e-2*U[-1,1) (seeded), FMG + 8 V                      <- headline
  cfg3  3D AMR: base 64^3 (N=8, L=4) + refinement to level 7 (effective 512^3)
        where |f(x)| < 2 dx_block; sphere c=.5 R=.25 phi_b=1 ("same as config 1"), g=0, 10 V
  cfg4  3D 512^3 in 16^3 blocks (L=6), min over 32 spheres (centres U[.15,.85]^3,
        R U[.01,.06], seeded), phi_b=1, g=0, 12 V
  cfg5  3D 1024^3 in 16^3 blocks (L=7), spheres (.3,.5,.5)/(.7,.5,.5) R=.15 with
        phi_b=+1/-1, g ~ N(0, 1e-3^2) (seeded), 10 V
All physical faces are Dirichlet 0; w_min = finest dx (harness.hpp:515-516).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import (SHAPE_COMPOSITE_MIN, SHAPE_SPHERE, LevelSetSpec, TreeMesh, build_uniform,
                   lsf_eval)

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED_CFG2 = 2205094112
SEED_CFG4 = 2205094114
SEED_CFG5 = 2205094115


def splitmix64(seed, k):
    """k-th output of a splitmix64 stream: state = seed + (k+1)*golden (public finaliser)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.asarray(k, np.uint64) + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01(seed, k):
    return (splitmix64(seed, k) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclass
class Case:
    name: str
    dim: int
    N: int
    levels: int               # uniform levels (or AMR base levels)
    max_level: int
    lsf: LevelSetSpec
    rhs: str = "zero"         # zero | uniform | gauss
    rhs_amp: float = 0.0
    seed: int = 0
    fmg_first: bool = False
    v_cycles: int = 10
    amr_band: float = 0.0     # >0: refine where |f(x)| < band * block dx
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def refine_lsf(self):
        """Level set the AMR band follows (the case's own unless extra['refine_lsf'])."""
        return self.extra.get("refine_lsf", self.lsf)

    @property
    def w_min(self):
        return 1.0 / (self.N * (1 << (self.max_level - 1)))

    def build_mesh(self) -> TreeMesh:
        m = build_uniform(self.dim, self.lo[:self.dim], self.hi[:self.dim], self.N, self.levels)
        if self.amr_band > 0:
            band = self.amr_band
            lsf = self.refine_lsf
            m.refine_by_criterion(self.max_level,
                                  lambda mesh, b, x: np.abs(lsf_eval(lsf, x)) < band * mesh.dx[b])
        return m

    def rhs_fields(self, mesh: TreeMesh, only=None, chunk=2048):
        """Interior RHS (n_blocks, N^D) for leaf blocks, zeros elsewhere.

        ``only``: boolean mask over block ids -- values are generated for those
        leaves alone (a rank of the partitioned solve needs its own blocks; the
        counter-based generator makes every cell's value independent of which
        others are drawn).  Blocks are processed ``chunk`` at a time, so the
        temporaries stay small at 1024^3 (the untouched rows of the zero array
        are never committed)."""
        nb, NI = mesh.n_blocks, self.N ** self.dim
        out = np.zeros((nb, NI))
        if self.rhs == "zero":
            return out
        N, D = self.N, self.dim
        idx = np.indices((N,) * D)[::-1].reshape(D, -1).T  # x fastest
        for l in range(1, mesh.n_levels + 1):
            n = N << (l - 1)
            ids_all = [b for b in mesh.level_blocks(l) if mesh.is_leaf(b) and (only is None or only[b])]
            for c0 in range(0, len(ids_all), chunk):
                ids = ids_all[c0:c0 + chunk]
                crd = np.array([mesh.coords[b] for b in ids], np.int64)  # (nl, D)
                g = crd[:, None, :] * N + idx[None, :, :]                 # (nl, NI, D)
                k = g[..., 0].astype(np.uint64)
                mul = np.uint64(n)
                for a in range(1, D):
                    k = k + mul * g[..., a].astype(np.uint64)
                    mul = mul * np.uint64(n)
                if self.rhs == "uniform":
                    u = uniform01(self.seed, k)
                    vals = self.rhs_amp * (2.0 * u - 1.0)
                else:  # gauss: Box-Muller on draws 2k, 2k+1
                    u1 = uniform01(self.seed, np.uint64(2) * k)
                    u2 = uniform01(self.seed, np.uint64(2) * k + np.uint64(1))
                    vals = self.rhs_amp * np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * np.pi * u2)
                out[np.array(ids)] = vals
        return out

    def leaf_cells(self, mesh: TreeMesh):
        return len(mesh.leaves()) * self.N ** self.dim


def _sphere(c, r, phi_b):
    return LevelSetSpec(shape=SHAPE_SPHERE, center=tuple(c), radius=r, boundary_value=phi_b)


def spheres32(seed=SEED_CFG4):
    ch = []
    for i in range(32):
        u = uniform01(seed, np.arange(4 * i, 4 * i + 4, dtype=np.uint64))
        c = 0.15 + 0.7 * u[:3]
        r = 0.01 + 0.05 * u[3]
        ch.append(_sphere(tuple(float(v) for v in c), float(r), 1.0))
    return LevelSetSpec(shape=SHAPE_COMPOSITE_MIN, children=ch)


def get_case(name: str) -> Case:
    if name == "cfg1":
        return Case("cfg1", 2, 8, 6, 6, _sphere((0.5, 0.5, 0.0), 0.25, 1.0), v_cycles=10,
                    notes="2D 256^2, N=8, circle R=.25, 10 V")
    if name == "cfg2":
        return Case("cfg2", 3, 16, 5, 5, _sphere((0.5, 0.5, 0.5), 0.2, 1.0), rhs="uniform",
                    rhs_amp=1e-2, seed=SEED_CFG2, fmg_first=True, v_cycles=8,
                    notes="3D 256^3, N=16, sphere R=.2, g=1e-2 U[-1,1), FMG + 8 V")
    if name == "cfg3":
        return Case("cfg3", 3, 8, 4, 7, _sphere((0.5, 0.5, 0.5), 0.25, 1.0), amr_band=2.0,
                    v_cycles=10, notes="3D AMR base 64^3 (N=8) -> level 7 (eff. 512^3), R=.25")
    if name == "cfg4":
        return Case("cfg4", 3, 16, 6, 6, spheres32(), v_cycles=12,
                    notes="3D 512^3, N=16, min of 32 seeded spheres, 12 V")
    if name == "cfg5":
        lsf = LevelSetSpec(shape=SHAPE_COMPOSITE_MIN,
                           children=[_sphere((0.3, 0.5, 0.5), 0.15, 1.0),
                                     _sphere((0.7, 0.5, 0.5), 0.15, -1.0)])
        return Case("cfg5", 3, 16, 7, 7, lsf, rhs="gauss", rhs_amp=1e-3, seed=SEED_CFG5,
                    v_cycles=10, notes="3D 1024^3, N=16, two spheres +-1, g ~ N(0,1e-6)")
    if name == "amrx":
        # test mesh: the refined band follows a SHIFTED sphere, so coarse-fine
        # faces cut through the interface of the real one (cut rows on and next
        # to coarse-fine faces: the block-per-CTA fallbacks of the AMR path)
        return Case("amrx", 3, 8, 3, 5, _sphere((0.5, 0.5, 0.5), 0.25, 1.0), amr_band=2.0, v_cycles=6,
                    extra={"refine_lsf": _sphere((0.35, 0.5, 0.5), 0.2, 1.0)},
                    notes="3D AMR base 32^3 (N=8) -> level 5, band around a shifted sphere")
    if name == "amrx16":  # the same with 16^3 blocks (the N = 16 kernels' coarse-fine paths)
        return Case("amrx16", 3, 16, 2, 4, _sphere((0.5, 0.5, 0.5), 0.25, 1.0), amr_band=2.0, v_cycles=6,
                    extra={"refine_lsf": _sphere((0.35, 0.5, 0.5), 0.2, 1.0)},
                    notes="3D AMR base 32^3 (N=16) -> level 4, band around a shifted sphere")
    # reduced variants for quick parity (same geometry / generator, fewer levels)
    if name.startswith("cfg") and "@" in name:
        base, lv = name.split("@")
        c = get_case(base)
        lv = int(lv)
        c.name = name
        if c.amr_band > 0:
            c.max_level = lv
        else:
            c.levels = c.max_level = lv
        return c
    raise KeyError(name)


def padded_from_interior(arr, dim, N):
    """(nb, N^D) interior -> (nb, (N+2)^D) padded with zero ghosts."""
    nb = arr.shape[0]
    s = N + 2
    out = np.zeros((nb,) + (s,) * dim)
    a = arr.reshape((nb,) + (N,) * dim)  # axes reversed: (z, y, x)
    if dim == 2:
        out[:, 1:-1, 1:-1] = a
    else:
        out[:, 1:-1, 1:-1, 1:-1] = a
    return out.reshape(nb, -1)


def interior_from_padded(arr, dim, N):
    nb = arr.shape[0]
    s = N + 2
    a = arr.reshape((nb,) + (s,) * dim)
    if dim == 2:
        return a[:, 1:-1, 1:-1].reshape(nb, -1)
    return a[:, 1:-1, 1:-1, 1:-1].reshape(nb, -1)
