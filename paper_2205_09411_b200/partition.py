"""Multi-GPU decomposition of the block tree.

* **Partition** -- Morton (Z-order) ranges.  The blocks of one *split level*
  ``g`` (the coarsest level with at least ``min_blocks_per_rank`` blocks per
  rank) are cut into ``world`` contiguous Morton ranges, balanced by the number
  of cells in each block's subtree; every finer block belongs to the rank of
  its level-``g`` ancestor.  A parent and its 2^D children therefore always
  share a rank, so restriction and prolongation above the split level need no
  communication.  Levels coarser than ``g`` (the coarse tail, a few hundred
  blocks at most) are owned by rank 0: the restricted level-``g`` values are
  gathered there and the corrected values broadcast back.
* **Halo plan** -- every rank keeps full-size level arrays (the colour-split
  block layout of the device context) and computes only its own blocks; the
  face layers its blocks read from other ranks' blocks are copied in after
  each phase that changes them.  After a GS half-sweep of colour ``c`` only the
  colour-``c`` cells of those face layers move (the colour-split exchange of
  §8e); residual-type phases move both colours.  For a rank pair the cells are
  listed in one canonical order, so the sender's gather list is the
  receiver's scatter list (``HaloPlan.pairs``).
* **Exchange** -- the solver's exchange is native (``csrc/dist.h``: the halo
  plans live on the device, pack / unpack kernels and NCCL run on the
  context's own stream inside the cycle graph).  ``exchange()`` here is the
  host-side statement of the same plan over ``torch.distributed``
  point-to-point calls; the world-size-2 ``gloo`` test drives it on CPU
  tensors (``tests/test_partition.py``).  Records are reduced with
  ``reduce_records()`` in rank order (deterministic).

Uniform (dense) levels and AMR levels without coarse-fine faces across a
partition boundary are supported; a coarse-fine face between two ranks raises
``NotImplementedError`` (AMR meshes run as replicas).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import TreeMesh


def morton_key(coords, dim):
    """Interleaved coordinate bits, x lowest (capi.cu morton)."""
    key = 0
    for b in range(21):
        for k in range(dim):
            key |= ((int(coords[k]) >> b) & 1) << (b * dim + k)
    return key


def level_slots(mesh: TreeMesh, l):
    """Block ids of level ``l`` in device slot order (Morton order of coords)."""
    ids = list(mesh.level_blocks(l))
    return sorted(ids, key=lambda b: morton_key(mesh.coords[b], mesh.dim))


def colour_addr(i, j, k, N, dim):
    """Colour-split address of interior cell (i,j,k) inside one block (capi.cu cs_addr)."""
    NI = N ** dim
    H = NI // 2
    return ((i + j + k) & 1) * H + ((i + N * (j + N * k)) >> 1)


@dataclass
class Partition:
    world: int
    split_level: int
    owner: dict = field(default_factory=dict)   # level -> np.int32[n blocks of level] in slot order
    slots: dict = field(default_factory=dict)   # level -> list of block ids in slot order

    def owned(self, level, rank):
        return self.owner[level] == rank


def morton_partition(mesh: TreeMesh, world: int, min_blocks_per_rank: int = 8) -> Partition:
    L = mesh.n_levels
    slots = {l: level_slots(mesh, l) for l in range(1, L + 1)}
    g = L
    for l in range(1, L + 1):
        if len(slots[l]) >= world * min_blocks_per_rank:
            g = l
            break
    # subtree cell weights of the split-level blocks
    NI = mesh.N ** mesh.dim

    def weight(b):
        w = NI
        for c in mesh.children[b]:
            if c >= 0:
                w += weight(c)
        return w

    ws = np.array([weight(b) for b in slots[g]], np.float64)
    cum = np.concatenate([[0.0], np.cumsum(ws)])
    total = cum[-1]
    own_g = np.zeros(len(slots[g]), np.int32)
    for s in range(len(slots[g])):
        mid = 0.5 * (cum[s] + cum[s + 1])
        own_g[s] = min(world - 1, int(mid * world / total))
    part = Partition(world=world, split_level=g, slots=slots)
    by_block = {}
    for s, b in enumerate(slots[g]):
        by_block[b] = int(own_g[s])
    for l in range(g + 1, L + 1):
        for b in slots[l]:
            by_block[b] = by_block[mesh.parent[b]]
    for l in range(1, L + 1):
        part.owner[l] = np.array([by_block.get(b, 0) if l >= g else 0 for b in slots[l]], np.int32)
    return part


@dataclass
class HaloPlan:
    """Per level and colour, for this rank: for each peer, the cell addresses
    (level-array indices, block slot * N^D + colour-split address) to send and
    to receive, in the canonical order shared by both ends."""
    rank: int
    send: dict = field(default_factory=dict)   # (level, colour) -> {peer: np.int64[]}
    recv: dict = field(default_factory=dict)   # (level, colour) -> {peer: np.int64[]}


def _face_cells(N, dim, d):
    """Interior cells (i,j,k) adjacent to face d of a block, transverse order lower axis fastest."""
    ax, side = d // 2, d & 1
    out = []
    rng = range(N)
    if dim == 2:
        for t in rng:
            c = [0, 0, 0]
            c[ax] = N - 1 if side else 0
            c[1 - ax] = t
            out.append(tuple(c))
    else:
        others = [a for a in range(3) if a != ax]
        for t1 in rng:
            for t0 in rng:
                c = [0, 0, 0]
                c[ax] = N - 1 if side else 0
                c[others[0]] = t0
                c[others[1]] = t1
                out.append(tuple(c))
    return out


def halo_plan(mesh: TreeMesh, part: Partition, rank: int) -> HaloPlan:
    dim, N = mesh.dim, mesh.N
    NI = N ** dim
    plan = HaloPlan(rank=rank)
    faces = {d: _face_cells(N, dim, d) for d in range(2 * dim)}
    for l in range(1, mesh.n_levels + 1):
        own = part.owner[l]
        slot_of = {b: s for s, b in enumerate(part.slots[l])}
        # canonical list per ordered pair (src owner p -> dst owner q): cells of
        # p's blocks that q's blocks read across a shared face
        pairs = {}
        for s, b in enumerate(part.slots[l]):
            p = int(own[s])
            for d in range(2 * dim):
                nb = mesh.nbr[b][d]
                if nb < 0:
                    if mesh.cnbr[b][d] >= 0:
                        q_c = int(part.owner[l - 1][part.slots[l - 1].index(mesh.cnbr[b][d])])
                        if q_c != p:
                            raise NotImplementedError("coarse-fine face across a partition boundary")
                    continue
                q = int(own[slot_of[nb]])
                if q == p:
                    continue
                # q's block nb reads b's face layer on b's side d
                for (i, j, k) in faces[d]:
                    pairs.setdefault((p, q), []).append((s, i, j, k))
        for c in (0, 1):
            send, recv = {}, {}
            for (p, q), cells in pairs.items():
                sel = [s * NI + colour_addr(i, j, k, N, dim) for (s, i, j, k) in cells
                       if ((i + j + k) & 1) == c]
                arr = np.array(sel, np.int64)
                if p == rank:
                    send[q] = arr
                if q == rank:
                    recv[p] = arr
            plan.send[(l, c)] = send
            plan.recv[(l, c)] = recv
    return plan


def exchange(arr, plan: HaloPlan, level: int, colours=(0, 1), group=None):
    """Copy the halo cells of `arr` (torch tensor, one level's field, flat) from
    their owners into this rank's copy.  Point-to-point, batched."""
    import torch
    import torch.distributed as dist
    ops, bufs = [], []
    for c in colours:
        for q, idx in sorted(plan.send.get((level, c), {}).items()):
            if len(idx) == 0:
                continue
            t = torch.as_tensor(idx, device=arr.device)
            ops.append(dist.P2POp(dist.isend, arr[t].contiguous(), q, group))
        for p, idx in sorted(plan.recv.get((level, c), {}).items()):
            if len(idx) == 0:
                continue
            buf = torch.empty(len(idx), dtype=arr.dtype, device=arr.device)
            bufs.append((idx, buf))
            ops.append(dist.P2POp(dist.irecv, buf, p, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for idx, buf in bufs:
        arr[torch.as_tensor(idx, device=arr.device)] = buf
    if arr.is_cuda:
        # the library's kernels run on the context's own non-blocking stream,
        # which does not wait for torch's: finish the writes before returning
        torch.cuda.current_stream(arr.device).synchronize()
    return arr


def reduce_records(rec, group=None):
    """(max|r|, sum r^2, count) of every rank, combined in rank order on all ranks."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([rec[0], rec[1], float(rec[2])], dtype=torch.float64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    mx, ss, cnt = 0.0, 0.0, 0.0
    for o in out:  # rank order: deterministic
        mx = max(mx, float(o[0]))
        ss += float(o[1])
        cnt += float(o[2])
    return mx, ss, int(cnt)
