"""Morton-partitioned V-cycle over several GPUs.

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  Every rank
holds the whole block tree and full-size level arrays (the DeviceMesh
context), computes only the blocks ``partition.morton_partition`` gives it, and
copies in the face layers its blocks read from other ranks' blocks after each
phase that changes them (``partition.exchange``: after a GS-RB half-sweep the
colour just updated, after restriction / FAS / prolongation both colours).
Levels below the split level are the coarse tail: their blocks belong to rank
0, which receives the restricted values of the split level's parents, runs the
tail of the V-cycle (down to the coarse solve and back) alone and broadcasts
the corrected level for the prolongation.  Records are reduced in rank order.

The V-cycle is the reference's (multigrid.hpp:483-499) operation for
operation; on one rank it reproduces ``MgSolver.v_cycle`` bit for bit
(tests/test_gpu_distributed.py).  It is driven from the host, one C-ABI call
per operation (no CUDA graph), so its per-level launch overhead is higher than
the single-GPU graph's.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .mesh import VAR_OLD, VAR_PHI, VAR_RHS
from .partition import exchange, halo_plan, morton_partition
from .solver import CycleStats, DeviceMesh, MgConfig, MgSolver


class _Cuda:
    """__cuda_array_interface__ wrapper of a device pointer (for torch.as_tensor)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class DistributedMgSolver:
    def __init__(self, dev: DeviceMesh, cfg: MgConfig | None = None, group=None, min_blocks_per_rank=8):
        import torch.distributed as dist
        self.dev = dev
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.mesh = dev.mesh
        self.cfg = cfg or MgConfig()
        self.part = morton_partition(self.mesh, self.world, min_blocks_per_rank)
        self.plan = halo_plan(self.mesh, self.part, self.rank)
        self.lib = _lib.load()
        self.h = dev.h
        L = self.mesh.n_levels
        for l in range(1, L + 1):
            mask = (self.part.owner[l] == self.rank).astype(np.uint8)
            dev._check(self.lib.pmg_b200_set_owned(self.h, l, mask.ctypes.data))
        self.solver = MgSolver(dev, None, self.cfg)
        self.NI = self.mesh.N ** self.mesh.dim
        self._views = {}

    # ---- device arrays as torch tensors
    def field(self, var, level):
        key = (var, level)
        if key not in self._views:
            import torch
            ptr = self.lib.pmg_b200_level_field_ptr(self.h, var, level)
            n = len(self.part.slots[level]) * self.NI
            self._views[key] = torch.as_tensor(_Cuda(ptr, n), device="cuda")
        return self._views[key]

    def _xchg(self, var, level, colours=(0, 1)):
        if self.world > 1 and level >= self.part.split_level:
            import torch
            torch.cuda.synchronize()
            exchange(self.field(var, level), self.plan, level, colours, self.group)

    def _parents_to_root(self, level):
        """Restricted phi / r of the split level's parents (level-1, owned by rank 0):
        every rank's parent cells go to rank 0."""
        if self.world == 1:
            return
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        own = np.repeat(self.part.owner[level] == self.rank, 1)
        # parent slots of this rank's level blocks
        slots_c = self.part.slots[level - 1]
        slot_of = {b: s for s, b in enumerate(slots_c)}
        mine = sorted({slot_of[self.mesh.parent[b]] for b, o in zip(self.part.slots[level], own) if o})
        idx = torch.as_tensor(np.concatenate([np.arange(s * self.NI, (s + 1) * self.NI) for s in mine])
                              if mine else np.zeros(0, np.int64), device="cuda")
        for var in (VAR_PHI, VAR_RHS):
            arr = self.field(var, level - 1)
            if self.rank == 0:
                for src in range(1, self.world):
                    n = torch.zeros(1, dtype=torch.int64, device="cuda")
                    dist.recv(n, src, self.group)
                    ridx = torch.empty(int(n.item()), dtype=torch.int64, device="cuda")
                    dist.recv(ridx, src, self.group)
                    buf = torch.empty(len(ridx), dtype=arr.dtype, device="cuda")
                    dist.recv(buf, src, self.group)
                    arr[ridx] = buf
            else:
                dist.send(torch.tensor([len(idx)], dtype=torch.int64, device="cuda"), 0, self.group)
                dist.send(idx, 0, self.group)
                dist.send(arr[idx].contiguous(), 0, self.group)

    def _bcast_level(self, level):
        if self.world == 1:
            return
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        for var in (VAR_PHI, VAR_OLD):
            dist.broadcast(self.field(var, level), 0, self.group)

    # ---- the cycle
    def _smooth(self, l, steps):
        for _ in range(steps):
            for c in (0, 1):
                self.dev._check(self.lib.pmg_b200_gsrb_sweep(self.h, l, c))
                self._xchg(VAR_PHI, l, (c,))

    def _record(self, l, recs):
        out = np.zeros(3)
        self.dev._check(self.lib.pmg_b200_level_record(self.h, l, out))
        recs[l] = out

    def _tail(self, top, recs):
        """v_cycle_span(top) on rank 0 only (levels <= top are the coarse tail)."""
        if self.rank != 0:
            return
        for l in range(top, 1, -1):
            self._smooth(l, self.cfg.n_down)
            self.dev._check(self.lib.pmg_b200_restrict_level(self.h, l))
        self.dev._check(self.lib.pmg_b200_coarse_solve(self.h))
        if self.mesh.is_leaf(self.part.slots[1][0]):
            self._record(1, recs)
        for l in range(2, top + 1):
            self.dev._check(self.lib.pmg_b200_prolong_correction(self.h, l))
            self._smooth(l, self.cfg.n_up)
            self._record(l, recs)

    def v_cycle(self):
        L, g = self.mesh.n_levels, self.part.split_level
        recs = {}
        if g == 1 or self.world == 1 and g > L:
            g = 1
        for l in range(L, max(g, 2) - 1, -1):
            self._smooth(l, self.cfg.n_down)
            self.dev._check(self.lib.pmg_b200_restrict_only(self.h, l))
            if l - 1 >= g:
                self._xchg(VAR_PHI, l - 1)
                self.dev._check(self.lib.pmg_b200_fas_level(self.h, l - 1))
                self._xchg(VAR_OLD, l - 1)
            else:  # the split level's parents: coarse tail on rank 0
                self._parents_to_root(l)
                if self.rank == 0:
                    self.dev._check(self.lib.pmg_b200_apply_pins(self.h, l - 1))
                    self.dev._check(self.lib.pmg_b200_fas_level(self.h, l - 1))
        if g >= 2:
            self._tail(g - 1, recs)
            self._bcast_level(g - 1)
        else:
            self.dev._check(self.lib.pmg_b200_coarse_solve(self.h))
            if self.mesh.is_leaf(self.part.slots[1][0]):
                self._record(1, recs)
        for l in range(max(g, 2), L + 1):
            self.dev._check(self.lib.pmg_b200_prolong_correction(self.h, l))
            self._xchg(VAR_PHI, l)
            self._smooth(l, self.cfg.n_up)
            self._record(l, recs)
        self.dev._check(self.lib.pmg_b200_set_have_guess(self.h, 1))
        return self._combine(recs)

    def _combine(self, recs):
        """combine_records (multigrid.hpp:564-575) over levels, records reduced over ranks in rank order."""
        L = self.mesh.n_levels
        loc = np.zeros((L + 1, 3))
        for l, r in recs.items():
            loc[l] = r
        if self.world > 1:
            import torch
            import torch.distributed as dist
            t = torch.tensor(loc, dtype=torch.float64, device="cuda")
            allr = [torch.zeros_like(t) for _ in range(self.world)]
            dist.all_gather(allr, t, group=self.group)
            tot = np.zeros((L + 1, 3))
            for a in allr:  # rank order
                a = a.cpu().numpy()
                tot[:, 0] = np.maximum(tot[:, 0], a[:, 0])
                tot[:, 1] += a[:, 1]
                tot[:, 2] += a[:, 2]
            loc = tot
        m, s, c = 0.0, 0.0, 0.0
        for l in range(0, L + 1):
            m = max(m, loc[l, 0])
            s += loc[l, 1]
            c += loc[l, 2]
        return CycleStats(m, math.sqrt(s / c) if c > 0 else 0.0)
