"""Morton-partitioned V-cycle over several GPUs.

One process per GPU (torchrun), one DeviceMesh context per process.  The
partition is ``partition.morton_partition`` (Morton ranges of the split level,
subtrees follow, the coarse tail on rank 0); everything else is native
(csrc/dist.h): the library restricts every kernel to the rank's blocks, builds
device-resident halo plans per level, peer and colour, and runs the whole
V-cycle -- halo pack / unpack kernels, grouped NCCL send / receive, the
coarse-tail gather and broadcast, the record all-gather -- as one CUDA graph on
the context's stream.  The host only launches the graph and reads the stats.

Transports:
  * ``"nccl"``  -- one process per GPU; the NCCL unique id is made on rank 0 by
    the library and broadcast with ``torch.distributed`` (any backend).
  * ``"local"`` -- several contexts of one process (``local_group``), each
    driven by its own host thread; device copies ordered by events.  This is
    how the decomposition is checked against the single-context cycle on one
    GPU (tests/test_gpu_distributed.py).
  * world == 1  -- no transport: the partitioned cycle is the single-GPU one.

The V-cycle is the reference's (multigrid.hpp:483-499) operation for
operation; its result is bit-identical to ``MgSolver.v_cycle`` (records up to
the rank-order summation of the sums of squares).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from .partition import morton_partition
from .solver import CycleStats, DeviceMesh, MgConfig, MgSolver


def owner_of_blocks(mesh, part):
    """Owner rank of every block id (levels below the split level: 0)."""
    owner = np.zeros(mesh.n_blocks, np.int32)
    for l in range(part.split_level, mesh.n_levels + 1):
        owner[np.asarray(part.slots[l], np.int64)] = part.owner[l]
    return owner


class DistributedMgSolver:
    """pmg::MgSolver<Dim>::v_cycle over a Morton partition of the block tree.

    ``dev`` holds the whole mesh and its stencils (build them first);
    ``world`` / ``rank`` default to torch.distributed's.  ``transport`` is
    ``"nccl"`` (default for world > 1 under torch.distributed) or ``"local"``
    (then call ``DistributedMgSolver.local_group`` with all ranks' solvers)."""

    def __init__(self, dev: DeviceMesh, cfg: MgConfig | None = None, world: int | None = None,
                 rank: int | None = None, transport: str | None = None, group=None,
                 min_blocks_per_rank: int = 8):
        if world is None or rank is None:
            import torch.distributed as dist
            init = dist.is_available() and dist.is_initialized()
            world = dist.get_world_size(group) if init else 1
            rank = dist.get_rank(group) if init else 0
        self.dev, self.world, self.rank = dev, world, rank
        self.lib = _lib.load()
        self.h = dev.h
        self.mesh = dev.mesh
        self.cfg = cfg or MgConfig()
        self.part = morton_partition(self.mesh, world, min_blocks_per_rank)
        owner = owner_of_blocks(self.mesh, self.part)
        dev._check(self.lib.pmg_b200_set_partition(self.h, world, rank, self.part.split_level,
                                                   owner.ctypes.data))
        self.solver = MgSolver(dev, None, self.cfg)
        self.transport = transport or ("nccl" if world > 1 else None)
        if world > 1 and self.transport == "nccl":
            self._init_nccl(group)

    def _init_nccl(self, group):
        import torch.distributed as dist
        uid = (C.c_ubyte * 128)()
        if self.rank == 0:
            self.dev._check(self.lib.pmg_b200_nccl_unique_id(uid))
        box = [bytes(uid) if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        C.memmove(uid, box[0], 128)
        self.dev._check(self.lib.pmg_b200_dist_init_nccl(self.h, uid))

    @staticmethod
    def local_group(solvers):
        """Bind the solvers of one process (solvers[r] is rank r) to the
        in-process transport."""
        lib = _lib.load()
        hs = (C.c_void_p * len(solvers))(*[s.h for s in solvers])
        rc = lib.pmg_b200_dist_local_group(len(solvers), hs)
        if rc != 0:
            solvers[0].dev._check(rc)
        for s in solvers:
            s.transport = "local"

    @staticmethod
    def run_local(solvers, fn):
        """Call fn(solver) for every solver of a local group on its own thread
        (the in-process transport needs one host thread per context)."""
        out, err = [None] * len(solvers), []

        def body(i):
            try:
                out[i] = fn(solvers[i])
            except BaseException as e:  # noqa: BLE001 -- re-raised below
                err.append(e)

        ts = [threading.Thread(target=body, args=(i,)) for i in range(len(solvers))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        return out

    def info(self):
        out = (C.c_int32 * 6)()
        self.dev._check(self.lib.pmg_b200_dist_info(self.h, out))
        return dict(world=out[0], split_level=out[1], transport=out[2], halo_cells=out[3],
                    graph_kernels=out[4], graph=out[5])

    def field_bytes(self) -> float:
        """Device bytes of this rank's field arrays (its blocks + halo on the
        large levels, the coarse tail whole)."""
        out = C.c_double()
        self.dev._check(self.lib.pmg_b200_field_bytes(self.h, C.byref(out)))
        return out.value

    def v_cycle(self) -> CycleStats:
        st = _lib.StatsT()
        self.dev._check(self.lib.pmg_b200_dist_v_cycle(self.h, C.byref(st)))
        return CycleStats(st.max_resid, st.l2_resid)

    def v_cycle_async(self):
        self.dev._check(self.lib.pmg_b200_dist_v_cycle_async(self.h))

    def cycle_result(self) -> CycleStats:
        return self.solver.cycle_result()
