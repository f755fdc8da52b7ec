// tree.cu -- the block tree (TreeMesh topology) built, refined and balanced on
// the device.
//
// Replaces, for the topology the solver reads:
//   TreeMesh::TreeMesh / refine_all            mesh.hpp:66-82, 206-216
//   TreeMesh::adapt (refine flags)             mesh.hpp:157-175, 198
//   refine_balanced / do_refine                mesh.hpp:253-320
//   rebuild_topology                           mesh.hpp:429-469
//   refine_by_criterion                        harness.hpp:295-321
//
// The reference refines sequentially: the flagged leaves in (level, id) order,
// each through a depth-first recursion that first refines every coarser leaf
// whose region touches the block (2:1 balance over faces, edges and corners,
// the 3^D - 1 offsets in enumerate_offsets order), then appends the block's
// 2^D children -- so the new block ids are the post-order of that recursion.
// The device reproduces the ids exactly without running the recursion:
//
//   * Every recursive call lands on a block of the mesh as it was BEFORE the
//     adapt (a balanced mesh has no leaf two levels coarser than a
//     neighbour), so the recursion is a depth-first search over a static DAG:
//     nodes = leaves, edge u -> v (label e = offset index, 0..3^D-1) when
//     offset e of u has no block on u's level and v is the leaf covering it.
//     Every edge goes one level down, so the DAG has depth < n_levels.
//   * In a DAG the path by which an ordered depth-first search discovers a
//     node is the lexicographically smallest (root, e1, e2, ...) path to it,
//     and the order in which the calls complete (= the order of do_refine)
//     is the order of those paths with "a prefix sorts after its extensions".
//   * So: K(v) = min over in-edges (u, e) of K(u).e, and (root key of v) when v
//     is flagged, computed level by level from the finest (one gather kernel
//     per level, no atomics); the blocks with a finite K are exactly the ones
//     the reference refines; sorting them by K (unused slots padded with the
//     largest label) gives the order of do_refine.  A root key is (level, id),
//     the reference's sort order of the flagged leaves.
//
// Keys are 128 bits: 32 for the root, 18 labels of 5 bits (max_level <= 19).
// Lookups (find_block, mesh.hpp:112-116) are binary searches in the blocks
// sorted by (level, coords[0], coords[1], coords[2]) -- the order of
// level_blocks (mesh.hpp:439-447) -- by a bitonic sort.  All arithmetic on
// origin / dx / cell centres follows the reference's expressions, so the
// geometry is bit-identical (mesh.hpp:78, 296-303, 139-143).
#include <algorithm>
#include <cstring>
#include <functional>

#include "stencil_build.cuh"

using pmghost::DevBuf;
using pmghost::PmgError;

namespace pmgdev {

struct TreeView {
  int dim, N, nb;
  int32_t *level, *coords, *parent, *children, *nbr, *cnbr;
  double *origin, *dx;
  // blocks sorted by (level, coords): key, id
  const unsigned long long* skey;
  const int32_t* sid;
};

constexpr int kCoordBits = 19;
__host__ __device__ __forceinline__ unsigned long long tree_key(int level, int c0, int c1, int c2) {
  return ((unsigned long long)level << (3 * kCoordBits)) | ((unsigned long long)c0 << (2 * kCoordBits)) |
         ((unsigned long long)c1 << kCoordBits) | (unsigned long long)c2;
}

// find_block (mesh.hpp:112-116): id of the block (level, c) or -1
__device__ __forceinline__ int tree_find(const TreeView& T, int level, const int* c) {
  const unsigned long long key = tree_key(level, c[0], c[1], T.dim == 3 ? c[2] : 0);
  int lo = 0, hi = T.nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (T.skey[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo < T.nb && T.skey[lo] == key ? T.sid[lo] : -1;
}

__global__ void k_tree_keys(TreeView T, unsigned long long* key, int32_t* id, int npad) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= npad) return;
  if (b < T.nb) {
    key[b] = tree_key(T.level[b], T.coords[3 * b], T.coords[3 * b + 1], T.dim == 3 ? T.coords[3 * b + 2] : 0);
    id[b] = b;
  } else {
    key[b] = ~0ull;
    id[b] = -1;
  }
}

// one compare-exchange step of a bitonic sorting network over (key, id)
__global__ void k_bitonic64(unsigned long long* key, int32_t* id, int n, int j, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = i ^ j;
  if (p <= i) return;
  const bool up = (i & k) == 0;
  const unsigned long long a = key[i], b = key[p];
  if ((a > b) == up) {
    key[i] = b, key[p] = a;
    const int32_t t = id[i];
    id[i] = id[p], id[p] = t;
  }
}

struct Key128 {
  unsigned long long hi, lo;
};
__device__ __forceinline__ bool key_less(const Key128& a, const Key128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
// K.e: label e into slot `depth` (slots hold 31 until used)
__device__ __forceinline__ Key128 key_append(Key128 k, int depth, int e) {
  const unsigned long long d = (unsigned long long)(31 - e);
  if (depth < 6) k.hi -= d << (27 - 5 * depth);
  else k.lo -= d << (59 - 5 * (depth - 6));
  return k;
}

__global__ void k_bitonic128(Key128* key, int32_t* id, int n, int j, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = i ^ j;
  if (p <= i) return;
  const bool up = (i & k) == 0;
  const Key128 a = key[i], b = key[p];
  if (key_less(b, a) == up) {
    key[i] = b, key[p] = a;
    const int32_t t = id[i];
    id[i] = id[p], id[p] = t;
  }
}

// Roots of an adapt: the flagged leaves (mesh.hpp:160-170).  err[0] counts
// flagged leaves at or beyond max_level.
__global__ void k_tree_roots(TreeView T, const uint8_t* __restrict__ flags, int nflags, int max_level, Key128* K,
                             int* err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= T.nb) return;
  Key128 k{~0ull, ~0ull};
  if (b < nflags && flags[b] == 1 && T.children[8 * b] < 0) {
    if (T.level[b] >= max_level) atomicAdd(err, 1);
    else k.hi = ((unsigned long long)(((unsigned)T.level[b] << 27) | (unsigned)b) << 32) | 0xffffffffull;
  }
  K[b] = k;
}

// K of the leaves of level l from the refined blocks of level l + 1 whose
// offsets they cover (refine_balanced, mesh.hpp:253-278).  One thread per
// block; list = the ids of level l.
__global__ void k_tree_close(TreeView T, const int32_t* __restrict__ list, int n, int l, Key128* K) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int v = list[q];
  if (T.children[8 * v] >= 0) return;  // not a leaf: nothing to force
  const int D = T.dim;
  const int side = 1 << l;  // blocks per axis on level l + 1
  int vc[3] = {T.coords[3 * v], T.coords[3 * v + 1], D == 3 ? T.coords[3 * v + 2] : 0};
  Key128 best = K[v];
  const int n2 = D == 3 ? 4 : 1;
  for (int a0 = 0; a0 < 4; ++a0)
    for (int a1 = 0; a1 < 4; ++a1)
      for (int a2 = 0; a2 < n2; ++a2) {
        const int a[3] = {a0, a1, D == 3 ? a2 : 1};
        // candidate u on level l + 1 next to (not inside) v
        if ((a[0] == 1 || a[0] == 2) && (a[1] == 1 || a[1] == 2) && (a[2] == 1 || a[2] == 2)) continue;
        int uc[3] = {0, 0, 0};
        bool in = true;
        int e = 0;
        for (int k = 0; k < D; ++k) {
          uc[k] = 2 * vc[k] - 1 + a[k];
          in = in && uc[k] >= 0 && uc[k] < side;
          // smallest offset o with (uc + o) >> 1 == vc: +1 below v, 0 on its
          // lower half, -1 on its upper half and above (enumerate_offsets
          // order: axis 0 outermost, -1, 0, 1)
          const int o = a[k] == 0 ? 1 : a[k] == 1 ? 0 : -1;
          e = 3 * e + (o + 1);
        }
        if (!in) continue;
        const int u = tree_find(T, l + 1, uc);
        if (u < 0) continue;
        const Key128 ku = K[u];
        if (ku.hi == ~0ull) continue;  // u is not refined
        const int depth = (int)(ku.hi >> 59) - (l + 1);  // root level - level of u
        const Key128 cand = key_append(ku, depth, e);
        if (key_less(cand, best)) best = cand;
      }
  K[v] = best;
}

// the refined set: (K, id) of every block with a finite K, compacted by an
// atomic counter (the order is fixed afterwards by the sort)
__global__ void k_tree_collect(int nb, const Key128* __restrict__ K, Key128* key, int32_t* id, int npad, int* count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= npad) return;
  if (b < nb && K[b].hi != ~0ull) {
    const int p = atomicAdd(count, 1);
    key[p] = K[b];
    id[p] = b;
  }
}
__global__ void k_tree_pad128(Key128* key, int32_t* id, int from, int npad) {
  const int i = from + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  key[i] = Key128{~0ull, ~0ull};
  id[i] = -1;
}

// do_refine (mesh.hpp:292-320) of the p-th refined block: children
// nb0 + 2^D p + c
__global__ void k_tree_children(TreeView T, const int32_t* __restrict__ order, int ns, int nb0) {
  const int D = T.dim, NC = 1 << D;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ns * NC) return;
  const int p = q / NC, c = q % NC;
  const int id = order[p];
  const int cid = nb0 + q;
  T.level[cid] = T.level[id] + 1;
  T.parent[cid] = id;
  const double pdx = T.dx[id];
  T.dx[cid] = 0.5 * pdx;
  for (int k = 0; k < 3; ++k) {
    const int bit = k < D ? (c >> k) & 1 : 0;
    T.coords[3 * cid + k] = k < D ? 2 * T.coords[3 * id + k] + bit : 0;
    T.origin[3 * cid + k] = k < D ? T.origin[3 * id + k] + bit * (0.5 * T.N * pdx) : 0.0;
  }
  for (int k = 0; k < 8; ++k) T.children[8 * cid + k] = -1;
  T.children[8 * id + c] = cid;
}

// rebuild_topology's neighbour tables (mesh.hpp:449-468); err[1] counts ghost
// regions without a covering block
__global__ void k_tree_nbrs(TreeView T, int* err) {
  const int D = T.dim;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= T.nb * 6) return;
  const int b = q / 6, dir = q % 6;
  int nb_ = -1, cn = -1;
  if (dir < 2 * D) {
    const int level = T.level[b];
    int nc[3] = {T.coords[3 * b], T.coords[3 * b + 1], T.coords[3 * b + 2]};
    nc[dir >> 1] += (dir & 1) ? 1 : -1;
    const int side = 1 << (level - 1);
    if (nc[dir >> 1] >= 0 && nc[dir >> 1] < side) {
      nb_ = tree_find(T, level, nc);
      if (nb_ < 0) {
        int pc[3] = {nc[0] >> 1, nc[1] >> 1, nc[2] >> 1};
        cn = level > 1 ? tree_find(T, level - 1, pc) : -1;
        if (cn < 0) atomicAdd(err + 1, 1);
      }
    }
  }
  T.nbr[q] = nb_;
  T.cnbr[q] = cn;
}

// first sorted position of every level (level_blocks segments); lvl_start has L + 2 entries
__global__ void k_tree_level_starts(const unsigned long long* __restrict__ skey, int nb, int* lvl_start, int nl) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l > nl + 1) return;
  const unsigned long long key = (unsigned long long)l << (3 * kCoordBits);
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (skey[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  lvl_start[l] = lo;
}

// refine_by_criterion's flags (harness.hpp:301-316): a leaf below max_level
// is flagged when any of its cell centres satisfies the criterion.
//   0 band:   |f(x)| < p0 * b.dx                      (the level set f)
//   1 radial: b.dx > p0 * max(1, ||x - c|| / p1)      (harness.hpp:351-355)
//   2 ball:   b.dx > p0 && ||x - c|| < p1             (harness.hpp:413-418)
struct TreeCrit {
  int kind;
  double p0, p1, c[3];
};
template <int D>
__global__ void __launch_bounds__(128) k_tree_flag(TreeView T, TreeCrit C, LsfDev lsf, int max_level, uint8_t* flags,
                                                   int* count) {
  const int b = blockIdx.x;
  __shared__ int hit;
  if (threadIdx.x == 0) hit = 0;
  __syncthreads();
  const bool cand = T.children[8 * b] < 0 && T.level[b] < max_level;
  if (cand) {
    const int N = T.N, NI = D == 3 ? N * N * N : N * N;
    const double dx = T.dx[b];
    for (int base = 0; base < NI; base += blockDim.x) {
      const int ii = base + threadIdx.x;
      if (ii < NI) {
        const int i[3] = {ii % N, (ii / N) % N, ii / (N * N)};
        double x[3];
        for (int k = 0; k < D; ++k) x[k] = T.origin[3 * b + k] + (i[k] + 0.5) * dx;  // mesh.hpp:139-143
        bool w;
        if (C.kind == 0) {
          w = fabs(lsf_eval<D>(lsf, x)) < C.p0 * dx;
        } else {
          double d[3];
          for (int k = 0; k < D; ++k) d[k] = x[k] - C.c[k];
          const double r = vnorm<D>(d);
          if (C.kind == 1) {
            const double m = r / C.p1;
            w = dx > C.p0 * (1.0 < m ? m : 1.0);  // std::max(1.0, m)
          } else {
            w = dx > C.p0 && r < C.p1;
          }
        }
        if (w) hit = 1;
      }
      __syncthreads();
      if (hit) break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    flags[b] = hit ? 1 : 0;
    if (hit) atomicAdd(count, 1);
  }
}

__global__ void k_tree_flag_leaves(TreeView T, uint8_t* flags) {  // refine_all: every leaf (mesh.hpp:206-216)
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < T.nb) flags[b] = T.children[8 * b] < 0 ? 1 : 0;
}

__global__ void k_tree_max_level(TreeView T, int* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < T.nb) atomicMax(out, T.level[b]);
}

}  // namespace pmgdev

// ------------------------------------------------------------------ host side
struct pmg_b200_tree {
  int dim = 0, N = 0, device = 0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  int nb = 0, cap = 0, L = 1;
  cudaStream_t stream = nullptr;
  DevBuf<int32_t> level, coords, parent, children, nbr, cnbr, sid;
  DevBuf<double> origin, dx;
  DevBuf<unsigned long long> skey;
  DevBuf<int> lvl_start, scal;  // scal: [0] err max-level, [1] err topology, [2] count, [3] max level
  std::vector<int> h_lvl_start;
  std::string err;
  int adapt_passes = 0;

  pmgdev::TreeView view() const {
    pmgdev::TreeView T;
    T.dim = dim, T.N = N, T.nb = nb;
    T.level = level.p, T.coords = coords.p, T.parent = parent.p, T.children = children.p;
    T.nbr = nbr.p, T.cnbr = cnbr.p, T.origin = origin.p, T.dx = dx.p;
    T.skey = skey.p, T.sid = sid.p;
    return T;
  }
};

namespace {

using namespace pmghost;

inline unsigned grid1(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }
inline int pow2_ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

template <typename T>
void grow(DevBuf<T>& b, size_t old_n, size_t new_n, cudaStream_t s) {
  DevBuf<T> nb_;
  nb_.alloc(new_n);
  if (b.p && old_n) PMG_CUDA(cudaMemcpyAsync(nb_.p, b.p, old_n * sizeof(T), cudaMemcpyDeviceToDevice, s));
  PMG_CUDA(cudaStreamSynchronize(s));
  b = std::move(nb_);
}

void reserve(pmg_b200_tree& t, int want) {
  if (want <= t.cap) return;
  const int cap = std::max(want, std::max(64, 2 * t.cap));
  grow(t.level, (size_t)t.nb, (size_t)cap, t.stream);
  grow(t.coords, (size_t)t.nb * 3, (size_t)cap * 3, t.stream);
  grow(t.origin, (size_t)t.nb * 3, (size_t)cap * 3, t.stream);
  grow(t.dx, (size_t)t.nb, (size_t)cap, t.stream);
  grow(t.parent, (size_t)t.nb, (size_t)cap, t.stream);
  grow(t.children, (size_t)t.nb * 8, (size_t)cap * 8, t.stream);
  grow(t.nbr, (size_t)t.nb * 6, (size_t)cap * 6, t.stream);
  grow(t.cnbr, (size_t)t.nb * 6, (size_t)cap * 6, t.stream);
  t.cap = cap;
}

// (key, id) of every block sorted by (level, coords): find_block's index and
// the level_blocks lists at once (mesh.hpp:431-447)
void sort_blocks(pmg_b200_tree& t) {
  const int npad = pow2_ceil(std::max(t.nb, 2));
  if ((size_t)npad > t.skey.n) {
    t.skey.alloc((size_t)npad);
    t.sid.alloc((size_t)npad);
  }
  pmgdev::k_tree_keys<<<grid1(npad), 256, 0, t.stream>>>(t.view(), t.skey.p, t.sid.p, npad);
  for (int k = 2; k <= npad; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1)
      pmgdev::k_bitonic64<<<grid1(npad), 256, 0, t.stream>>>(t.skey.p, t.sid.p, npad, j, k);
  PMG_CUDA(cudaGetLastError());
}

void rebuild_topology(pmg_b200_tree& t) {
  sort_blocks(t);
  PMG_CUDA(cudaMemsetAsync(t.scal.p + 1, 0, sizeof(int), t.stream));
  PMG_CUDA(cudaMemsetAsync(t.scal.p + 3, 0, sizeof(int), t.stream));
  pmgdev::k_tree_nbrs<<<grid1((long long)t.nb * 6), 256, 0, t.stream>>>(t.view(), t.scal.p);
  pmgdev::k_tree_max_level<<<grid1(t.nb), 256, 0, t.stream>>>(t.view(), t.scal.p + 3);
  int h[4];
  PMG_CUDA(cudaMemcpyAsync(h, t.scal.p, sizeof(h), cudaMemcpyDeviceToHost, t.stream));
  PMG_CUDA(cudaStreamSynchronize(t.stream));
  if (h[1] != 0) throw PmgError(PMG_ERR_TOPOLOGY, "ghost region has no covering block");  // mesh.hpp:464
  t.L = h[3];
  if ((size_t)(t.L + 2) > t.lvl_start.n) t.lvl_start.alloc((size_t)t.L + 2 + 8);
  pmgdev::k_tree_level_starts<<<1, 64, 0, t.stream>>>(t.skey.p, t.nb, t.lvl_start.p, t.L);
  t.h_lvl_start.assign((size_t)t.L + 2, 0);
  PMG_CUDA(cudaMemcpyAsync(t.h_lvl_start.data(), t.lvl_start.p, (size_t)(t.L + 2) * sizeof(int),
                           cudaMemcpyDeviceToHost, t.stream));
  PMG_CUDA(cudaStreamSynchronize(t.stream));
}

// adapt with refine flags on the device (flags: one byte per block id, 1 = refine).
// Returns the number of blocks refined.
int adapt_device(pmg_b200_tree& t, const uint8_t* d_flags, int nflags, int max_level) {
  if (max_level > 19) throw PmgError(PMG_ERR_INVALID_ARG, "device tree: max_level must be at most 19");
  const int nb0 = t.nb;
  DevBuf<pmgdev::Key128> K, skeys;
  DevBuf<int32_t> sids;
  K.alloc((size_t)nb0);
  PMG_CUDA(cudaMemsetAsync(t.scal.p, 0, 3 * sizeof(int), t.stream));
  pmgdev::k_tree_roots<<<grid1(nb0), 256, 0, t.stream>>>(t.view(), d_flags, nflags, max_level, K.p, t.scal.p);
  // forced refinement, one level at a time from the finest: the leaves of
  // level l that a refined block of level l + 1 touches
  for (int l = t.L - 1; l >= 1; --l) {
    const int s0 = t.h_lvl_start[(size_t)l], n = t.h_lvl_start[(size_t)l + 1] - s0;
    if (n > 0) pmgdev::k_tree_close<<<grid1(n, 128), 128, 0, t.stream>>>(t.view(), t.sid.p + s0, n, l, K.p);
  }
  const int npad0 = pow2_ceil(std::max(nb0, 2));
  skeys.alloc((size_t)npad0);
  sids.alloc((size_t)npad0);
  pmgdev::k_tree_collect<<<grid1(nb0), 256, 0, t.stream>>>(nb0, K.p, skeys.p, sids.p, nb0, t.scal.p + 2);
  int h[3];
  PMG_CUDA(cudaMemcpyAsync(h, t.scal.p, sizeof(h), cudaMemcpyDeviceToHost, t.stream));
  PMG_CUDA(cudaStreamSynchronize(t.stream));
  if (h[0] != 0) throw PmgError(PMG_ERR_INVALID_ARG, "refinement beyond the configured maximum level");
  const int ns = h[2];
  if (ns == 0) return 0;
  const int npad = pow2_ceil(std::max(ns, 2));
  pmgdev::k_tree_pad128<<<grid1(npad - ns + 1), 256, 0, t.stream>>>(skeys.p, sids.p, ns, npad);
  for (int k = 2; k <= npad; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1)
      pmgdev::k_bitonic128<<<grid1(npad), 256, 0, t.stream>>>(skeys.p, sids.p, npad, j, k);
  const int NC = 1 << t.dim;
  reserve(t, nb0 + ns * NC);
  t.nb = nb0 + ns * NC;
  pmgdev::k_tree_children<<<grid1((long long)ns * NC), 256, 0, t.stream>>>(t.view(), sids.p, ns, nb0);
  PMG_CUDA(cudaGetLastError());
  rebuild_topology(t);
  ++t.adapt_passes;
  return ns;
}

int guard(pmg_b200_tree* t, const std::function<void()>& f) {
  if (!t) return PMG_ERR_INVALID_ARG;
  try {
    PMG_CUDA(cudaSetDevice(t->device));
    f();
    return PMG_OK;
  } catch (const PmgError& e) {
    t->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    t->err = e.what();
    return PMG_ERR_INVALID_ARG;
  }
}

}  // namespace

extern "C" {

pmg_b200_tree* pmg_b200_tree_create(int dim, int N, const double* lo, const double* hi, int device) {
  auto* t = new (std::nothrow) pmg_b200_tree();
  if (!t) return nullptr;
  t->dim = dim, t->N = N, t->device = device;
  const int rc = guard(t, [&] {
    // TreeMesh::TreeMesh (mesh.hpp:66-82), the reference's messages
    if (dim != 2 && dim != 3) throw PmgError(PMG_ERR_INVALID_ARG, "dimension must be 2 or 3");
    if (!(N > 0 && (N & (N - 1)) == 0 && N >= 4))
      throw PmgError(PMG_ERR_INVALID_ARG, "block size N must be a power of two and at least 4");
    const double ext = hi[0] - lo[0];
    for (int k = 0; k < dim; ++k) {
      t->lo[k] = lo[k], t->hi[k] = hi[k];
      if (!(std::abs((hi[k] - lo[k]) - ext) <= 1e-12 * std::abs(ext)))
        throw PmgError(PMG_ERR_INVALID_ARG, "domain must be square/cubic");
    }
    if (!(ext > 0)) throw PmgError(PMG_ERR_INVALID_ARG, "domain extent must be positive");
    PMG_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    t->scal.alloc(4);
    reserve(*t, 64);
    // the root block
    const int32_t lvl = 1, par = -1;
    int32_t c3[3] = {0, 0, 0}, m8[8], m6[6];
    std::fill(m8, m8 + 8, -1);
    std::fill(m6, m6 + 6, -1);
    double o3[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) o3[k] = lo[k];
    const double dx = ext / N;
    PMG_CUDA(cudaMemcpyAsync(t->level.p, &lvl, sizeof(lvl), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->parent.p, &par, sizeof(par), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->coords.p, c3, sizeof(c3), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->origin.p, o3, sizeof(o3), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->dx.p, &dx, sizeof(dx), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->children.p, m8, sizeof(m8), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->nbr.p, m6, sizeof(m6), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaMemcpyAsync(t->cnbr.p, m6, sizeof(m6), cudaMemcpyHostToDevice, t->stream));
    PMG_CUDA(cudaStreamSynchronize(t->stream));
    t->nb = 1;
    rebuild_topology(*t);
  });
  (void)rc;
  return t;
}

void pmg_b200_tree_destroy(pmg_b200_tree* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  if (t->stream) cudaStreamDestroy(t->stream);
  delete t;
}

const char* pmg_b200_tree_last_error(pmg_b200_tree* t) { return t ? t->err.c_str() : "null tree"; }
int pmg_b200_tree_n_blocks(pmg_b200_tree* t) { return t ? t->nb : 0; }
int pmg_b200_tree_n_levels(pmg_b200_tree* t) { return t ? t->L : 0; }
int pmg_b200_tree_adapt_passes(pmg_b200_tree* t) { return t ? t->adapt_passes : 0; }

int pmg_b200_tree_refine_all(pmg_b200_tree* t, int times, int max_level) {
  return guard(t, [&] {
    for (int i = 0; i < times; ++i) {
      DevBuf<uint8_t> flags;
      flags.alloc((size_t)t->nb);
      pmgdev::k_tree_flag_leaves<<<grid1(t->nb), 256, 0, t->stream>>>(t->view(), flags.p);
      adapt_device(*t, flags.p, t->nb, max_level);
    }
  });
}

int pmg_b200_tree_adapt(pmg_b200_tree* t, const uint8_t* flags, int n_flags, int flags_on_device, int max_level,
                        int* n_refined) {
  return guard(t, [&] {
    const int n = std::min(n_flags, t->nb);
    DevBuf<uint8_t> tmp;
    const uint8_t* d = flags;
    if (!flags_on_device) {
      tmp.alloc((size_t)std::max(n, 1));
      if (n > 0) PMG_CUDA(cudaMemcpyAsync(tmp.p, flags, (size_t)n, cudaMemcpyHostToDevice, t->stream));
      d = tmp.p;
    }
    const int ns = adapt_device(*t, d, n, max_level);
    if (n_refined) *n_refined = ns;
  });
}

int pmg_b200_tree_refine_by_criterion(pmg_b200_tree* t, int kind, const pmg_lsf_t* lsf, int n_lsf, double p0,
                                      double p1, const double* centre, int max_level) {
  return guard(t, [&] {
    if (kind < 0 || kind > 2) throw PmgError(PMG_ERR_INVALID_ARG, "unknown refinement criterion");
    pmgdev::TreeCrit C;
    C.kind = kind, C.p0 = p0, C.p1 = p1;
    for (int k = 0; k < 3; ++k) C.c[k] = centre && k < t->dim ? centre[k] : 0.0;
    DevBuf<pmg_lsf_t> dl;
    pmgdev::LsfDev L{0, nullptr};
    if (kind == 0) {
      if (!lsf || n_lsf < 1) throw PmgError(PMG_ERR_INVALID_ARG, "band criterion needs a level set");
      dl.upload(std::vector<pmg_lsf_t>(lsf, lsf + n_lsf), t->stream);
      L.n = n_lsf, L.d = dl.p;
    }
    for (;;) {  // harness.hpp:299-320
      DevBuf<uint8_t> flags;
      flags.alloc((size_t)t->nb);
      PMG_CUDA(cudaMemsetAsync(t->scal.p + 2, 0, sizeof(int), t->stream));
      if (t->dim == 2)
        pmgdev::k_tree_flag<2><<<t->nb, 128, 0, t->stream>>>(t->view(), C, L, max_level, flags.p, t->scal.p + 2);
      else
        pmgdev::k_tree_flag<3><<<t->nb, 128, 0, t->stream>>>(t->view(), C, L, max_level, flags.p, t->scal.p + 2);
      int any = 0;
      PMG_CUDA(cudaMemcpyAsync(&any, t->scal.p + 2, sizeof(int), cudaMemcpyDeviceToHost, t->stream));
      PMG_CUDA(cudaStreamSynchronize(t->stream));
      if (!any) return;
      adapt_device(*t, flags.p, t->nb, max_level);
    }
  });
}

int pmg_b200_tree_get(pmg_b200_tree* t, int32_t* level, int32_t* coords, double* origin, double* dx,
                      int32_t* parent, int32_t* children, int32_t* nbr, int32_t* cnbr) {
  return guard(t, [&] {
    const size_t n = (size_t)t->nb;
    auto get = [&](void* dst, const void* src, size_t bytes) {
      if (dst) PMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, t->stream));
    };
    get(level, t->level.p, n * 4);
    get(coords, t->coords.p, n * 12);
    get(origin, t->origin.p, n * 24);
    get(dx, t->dx.p, n * 8);
    get(parent, t->parent.p, n * 4);
    get(children, t->children.p, n * 32);
    get(nbr, t->nbr.p, n * 24);
    get(cnbr, t->cnbr.p, n * 24);
    PMG_CUDA(cudaStreamSynchronize(t->stream));
  });
}

int pmg_b200_tree_level_blocks(pmg_b200_tree* t, int level, int32_t* ids, int* n) {
  return guard(t, [&] {
    if (level < 1 || level > t->L) throw PmgError(PMG_ERR_INVALID_ARG, "level out of range");
    const int s0 = t->h_lvl_start[(size_t)level], cnt = t->h_lvl_start[(size_t)level + 1] - s0;
    if (n) *n = cnt;
    if (ids && cnt > 0) {
      PMG_CUDA(cudaMemcpyAsync(ids, t->sid.p + s0, (size_t)cnt * 4, cudaMemcpyDeviceToHost, t->stream));
      PMG_CUDA(cudaStreamSynchronize(t->stream));
    }
  });
}

/* device pointers of the block table (level, coords[3], origin[3], dx, parent,
 * children[8], nbr[6], cnbr[6]) for consumers on the same device */
int pmg_b200_tree_device_arrays(pmg_b200_tree* t, const void** out8) {
  return guard(t, [&] {
    out8[0] = t->level.p, out8[1] = t->coords.p, out8[2] = t->origin.p, out8[3] = t->dx.p;
    out8[4] = t->parent.p, out8[5] = t->children.p, out8[6] = t->nbr.p, out8[7] = t->cnbr.p;
  });
}

/* hands the tree to a solver context: pmg_b200_set_mesh from the device tables */
int pmg_b200_set_mesh_from_tree(pmg_b200_ctx* ctx, pmg_b200_tree* t) {
  if (!ctx || !t) return PMG_ERR_INVALID_ARG;
  const size_t n = (size_t)t->nb;
  std::vector<int32_t> level(n), coords(n * 3), parent(n), children(n * 8), nbr(n * 6), cnbr(n * 6);
  std::vector<double> origin(n * 3), dx(n);
  const int rc = pmg_b200_tree_get(t, level.data(), coords.data(), origin.data(), dx.data(), parent.data(),
                                   children.data(), nbr.data(), cnbr.data());
  if (rc != PMG_OK) return rc;
  return pmg_b200_set_mesh(ctx, t->nb, level.data(), coords.data(), origin.data(), dx.data(), parent.data(),
                           children.data(), nbr.data(), cnbr.data());
}

}  // extern "C"
