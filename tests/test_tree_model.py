"""CPU checks behind the device tree (csrc/tree.cu).

1. The host mirror's adapt (mesh.py, the sequential recursion of
   mesh.hpp:157-175, 253-320) against the reference build on random refine
   flags that force 2:1 balancing -- the order of the new block ids is what
   the device has to reproduce.
2. A Python model of the DEVICE algorithm (lexicographically smallest
   discovery path per refined block, level by level, then a sort with
   "a prefix sorts after its extensions") against that recursion: the model
   is the statement csrc/tree.cu implements, kernel by kernel.
"""
import itertools
import os

import numpy as np
import pytest

from oracle.oc import PORT_SO, REF_SO, Oracle
from paper_2205_09411_b200.mesh import TreeMesh

PAD = 31


def model_adapt_order(m: TreeMesh, refine_ids, max_level):
    """The blocks an adapt refines, in do_refine order, by the device algorithm."""
    D = m.dim
    K = {}
    for b in refine_ids:
        if m.is_leaf(b):
            assert m.level[b] < max_level
            K[b] = ((m.level[b] << 27) | b,)  # root key: the reference's (level, id) order
    offs = list(itertools.product((-1, 0, 1), repeat=D))  # enumerate_offsets order
    for l in range(m.n_levels - 1, 0, -1):
        for v in m.level_blocks(l):
            if not m.is_leaf(v):
                continue
            best = K.get(v)
            vc = m.coords[v]
            side = 1 << l
            for a in itertools.product(range(4), repeat=D):
                if all(x in (1, 2) for x in a):
                    continue
                uc = tuple(2 * vc[k] - 1 + a[k] for k in range(D))
                if not all(0 <= x < side for x in uc):
                    continue
                u = m.find_block(l + 1, uc)
                if u < 0 or u not in K:
                    continue
                o = tuple(1 if a[k] == 0 else 0 if a[k] == 1 else -1 for k in range(D))
                cand = K[u] + (offs.index(o),)
                if best is None or cand < best:
                    best = cand
            if best is not None:
                K[v] = best
    depth = max((len(k) for k in K.values()), default=1)
    order = sorted(K, key=lambda b: K[b] + (PAD,) * (depth - len(K[b])))
    return order


def sequential_order(m: TreeMesh, refine_ids, max_level):
    """do_refine order of the sequential recursion (the parents of the new blocks)."""
    nb0 = m.n_blocks
    m.adapt_refine(refine_ids, max_level)
    return [m.parent[b] for b in range(nb0, m.n_blocks, 1 << m.dim)]


def clone(m: TreeMesh):
    import copy
    return copy.deepcopy(m)


@pytest.mark.parametrize("dim,N,seed", [(2, 4, 1), (2, 4, 2), (2, 8, 3), (3, 4, 4), (3, 4, 5)])
def test_device_order_model_matches_recursion(dim, N, seed):
    rng = np.random.default_rng(seed)
    m = TreeMesh(dim, (0.0,) * dim, (1.0,) * dim, N)
    m.refine_all(2, 12)
    max_level = 9
    for _ in range(6 if dim == 2 else 4):
        leaves = [b for b in m.leaves() if m.level[b] < max_level]
        # few flags on the finest leaves: each drags a chain of coarser blocks along
        deep = max(m.level[b] for b in leaves)
        pool = [b for b in leaves if m.level[b] >= deep - 1]
        ids = [int(b) for b in rng.choice(pool, size=min(len(pool), 5), replace=False)]
        expect_model = model_adapt_order(m, ids, max_level)
        got = sequential_order(m, ids, max_level)
        assert got == expect_model
    assert m.n_levels >= 6  # the chains really forced coarser refinement


@pytest.mark.parametrize("dim,N,seed", [(2, 4, 11), (3, 4, 12)])
def test_host_adapt_matches_reference_on_random_flags(dim, N, seed):
    which = "ref" if os.path.exists(REF_SO) else "port"
    if not os.path.exists(REF_SO if which == "ref" else PORT_SO):
        pytest.skip("no CPU oracle built")
    rng = np.random.default_rng(seed)
    m = TreeMesh(dim, (0.0,) * dim, (1.0,) * dim, N)
    m.refine_all(2, 12)
    o = Oracle(dim, N, (0.0,) * 3, (1.0,) * 3, which)
    o.build_uniform(3)
    for _ in range(5 if dim == 2 else 3):
        leaves = m.leaves()
        deep = max(m.level[b] for b in leaves)
        pool = [b for b in leaves if m.level[b] >= deep - 1]
        ids = [int(b) for b in rng.choice(pool, size=min(len(pool), 4), replace=False)]
        m.adapt_refine(ids, 12)
        o.adapt_refine(ids, 12)
        t, r = m.topology_arrays(), o.topology()
        for k in ("level", "coords", "origin", "dx", "parent", "children", "nbr", "cnbr"):
            assert np.array_equal(np.asarray(t[k]).reshape(-1), np.asarray(r[k]).reshape(-1)), k
        for l in range(1, m.n_levels + 1):
            assert list(m.level_blocks(l)) == list(o.level_blocks(l))
