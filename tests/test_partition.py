"""CPU: the multi-GPU decomposition (paper_2205_09411_b200/partition.py) --
Morton partition properties, and the halo exchange / a partitioned GS-RB sweep
over world_size-2 gloo process groups, checked bit-for-bit against the
single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_09411_b200.mesh import build_uniform
from paper_2205_09411_b200.partition import (colour_addr, exchange, halo_plan, level_slots, morton_partition,
                                             reduce_records)


def _mesh():
    return build_uniform(3, (0, 0, 0), (1, 1, 1), 8, 4)  # 8 x 8 x 8 blocks of 8^3 on the finest level


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_keeps_subtrees_and_balances(world):
    m = _mesh()
    p = morton_partition(m, world)
    g = p.split_level
    for l in range(2, m.n_levels + 1):
        own = {b: int(o) for b, o in zip(p.slots[l], p.owner[l])}
        ownp = {b: int(o) for b, o in zip(p.slots[l - 1], p.owner[l - 1])}
        for b in p.slots[l]:
            if l > g:  # parent and children share a rank above the split level
                assert own[b] == ownp[m.parent[b]]
    # contiguous Morton ranges, balanced on the finest level
    own = p.owner[m.n_levels]
    assert np.all(np.diff(own) >= 0)
    counts = np.bincount(own, minlength=world)
    assert counts.max() - counts.min() <= 8 ** (m.n_levels - g)
    assert set(np.unique(own)) == set(range(world))
    for l in range(1, g):
        assert np.all(p.owner[l] == 0)  # coarse tail on rank 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gs_tables(m, l):
    """Per cell of level l (slot order): the 6 neighbour addresses; -1 marks a
    physical Dirichlet-0 face (ghost -f1)."""
    N, dim = m.N, m.dim
    NI = N ** dim
    slots = level_slots(m, l)
    slot_of = {b: s for s, b in enumerate(slots)}
    nb_addr = np.full((len(slots) * NI, 6), -1, np.int64)
    for s, b in enumerate(slots):
        for k in range(N):
            for j in range(N):
                for i in range(N):
                    a = s * NI + colour_addr(i, j, k, N, dim)
                    for d in range(6):
                        ax, sg = d // 2, (1 if d & 1 else -1)
                        q = [i, j, k]
                        q[ax] += sg
                        if 0 <= q[ax] < N:
                            nb_addr[a, d] = s * NI + colour_addr(*q, N, dim)
                        elif m.nbr[b][d] >= 0:
                            q[ax] = 0 if sg > 0 else N - 1
                            nb_addr[a, d] = slot_of[m.nbr[b][d]] * NI + colour_addr(*q, N, dim)
    return nb_addr


def _half_sweep(phi, g, nb_addr, colour, owned_cells, h2):
    """Uniform GS-RB half-sweep (multigrid.hpp:651-653) on the given cells of one colour."""
    cells = owned_cells[colour]
    p = np.where(nb_addr[cells] >= 0, phi[np.maximum(nb_addr[cells], 0)], -phi[cells][:, None])
    phi[cells] = (p[:, 0] + p[:, 1] + p[:, 2] + p[:, 3] + p[:, 4] + p[:, 5] - h2 * g[cells]) / 6.0


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _mesh()
        L = m.n_levels
        p = morton_partition(m, world)
        plan = halo_plan(m, p, rank)
        N, NI = m.N, m.N ** 3
        nbk = len(p.slots[L])
        rng = np.random.default_rng(7)
        glob = rng.uniform(-1, 1, nbk * NI)
        g = rng.uniform(-1, 1, nbk * NI)
        # 1) exchange: non-owned values start as NaN; every cell an owned block reads must arrive
        own_blk = p.owner[L] == rank
        mine = np.repeat(own_blk, NI)
        loc = torch.tensor(np.where(mine, glob, np.nan))
        exchange(loc, plan, L, colours=(0, 1))
        nb_addr = _gs_tables(m, L)
        reads = np.unique(nb_addr[mine][nb_addr[mine] >= 0])
        ok_ex = bool(np.array_equal(loc.numpy()[reads], glob[reads]))
        # 2) two GS-RB sweeps, partitioned (sweep own cells, exchange the colour just updated)
        colour_of = np.array([((a % NI) // (NI // 2)) for a in range(nbk * NI)])
        owned_cells = {c: np.nonzero(mine & (colour_of == c))[0] for c in (0, 1)}
        all_cells = {c: np.nonzero(colour_of == c)[0] for c in (0, 1)}
        h2 = m.level_dx(L) ** 2
        ser = glob.copy()
        par = torch.tensor(np.where(mine, glob, np.nan))
        exchange(par, plan, L, colours=(0, 1))
        for _ in range(2):
            for c in (0, 1):
                _half_sweep(ser, g, nb_addr, c, all_cells, h2)
                arr = par.numpy()
                _half_sweep(arr, g, nb_addr, c, owned_cells, h2)
                exchange(par, plan, L, colours=(c,))
        ok_gs = bool(np.array_equal(par.numpy()[mine], ser[mine]))
        # 3) record reduction in rank order
        r = par.numpy()[mine]
        mx, ss, cnt = reduce_records((float(np.max(np.abs(r))), float(np.sum(r * r)), int(r.size)))
        ok_rec = cnt == nbk * NI and mx == float(np.max(np.abs(ser)))
        out[rank] = (ok_ex, ok_gs, ok_rec)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_partitioned_gs_matches_serial_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (True, True, True), (r, out[r])
