// dist.h -- the Morton-partitioned V-cycle over several GPUs,
// included by capi.cu (it drives the same enqueue functions).
//
// One context per GPU (one process per GPU under torchrun, NCCL transport),
// or several contexts of one process (the in-process transport: the parity
// test of the decomposition on one device, one host thread per context).
//
// * Ownership (pmg_b200_set_partition): every block of the split level g and
//   its whole subtree belongs to one rank (the caller's Morton ranges,
//   partition.py); the levels below g -- the coarse tail -- belong to rank 0.
//   Every kernel plan, cut-row table and pin list is restricted to the owned
//   blocks (set_owned's machinery).
// * Halo plans, built here once from the topology: for every level >= g and
//   every peer, the face-layer cells of this rank's blocks a peer's blocks
//   read (send) and of the peer's blocks this rank's blocks read (receive),
//   each in ONE canonical order both ends derive (blocks in slot order, faces
//   in direction order, face cells lower axis fastest); per colour and for both
//   colours.  The cell addresses live on the device: an exchange is one pack
//   kernel, the transport, one unpack kernel, all on the context's stream --
//   no host synchronisation, nothing re-uploaded.
// * Exchanges: after a GS-RB half-sweep only the colour just updated moves
//   (the colour-split exchange); after restriction (phi) and FAS (OLD) of a
//   level >= g, and after prolongation, both colours.
// * Coarse tail: the split level's restriction writes its parents' octants on
//   the children's ranks; they are gathered to rank 0 (phi and the restricted
//   residual), which pins them, forms the FAS right-hand side and runs the
//   V-cycle of levels <= g - 1 alone, then broadcasts phi and OLD of level
//   g - 1 for the prolongation into level g.
// * Records: every rank records its owned leaves; the per-level records of
//   all ranks are all-gathered and combined in rank order on the device
//   (deterministic).
// * The NCCL transport's cycle (pack kernels, grouped ncclSend / ncclRecv,
//   ncclBroadcast, ncclAllGather) is captured into one CUDA graph per context
//   and replayed; libnccl is resolved at run time (dlopen), so the library
//   has no link dependency on it.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <array>
#include <condition_variable>
#include <mutex>

namespace pmghost {

// ---------------------------------------------------------------- NCCL (run-time bound)
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
inline NcclApi& nccl_api() {
  static NcclApi a = [] {
    NcclApi x;
    // the process's NCCL if one is loaded (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.why = "libnccl.so.2 not found";
      return x;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    x.GetUniqueId = (decltype(x.GetUniqueId))sym("ncclGetUniqueId");
    x.CommInitRank = (decltype(x.CommInitRank))sym("ncclCommInitRank");
    x.CommDestroy = (decltype(x.CommDestroy))sym("ncclCommDestroy");
    x.Send = (decltype(x.Send))sym("ncclSend");
    x.Recv = (decltype(x.Recv))sym("ncclRecv");
    x.GroupStart = (decltype(x.GroupStart))sym("ncclGroupStart");
    x.GroupEnd = (decltype(x.GroupEnd))sym("ncclGroupEnd");
    x.Broadcast = (decltype(x.Broadcast))sym("ncclBroadcast");
    x.AllGather = (decltype(x.AllGather))sym("ncclAllGather");
    x.GetErrorString = (decltype(x.GetErrorString))sym("ncclGetErrorString");
    x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.Send && x.Recv && x.GroupStart && x.GroupEnd &&
           x.Broadcast && x.AllGather && x.GetErrorString;
    if (!x.ok) x.why = "libnccl.so.2 lacks a required symbol";
    return x;
  }();
  return a;
}
#define PMG_NCCL(x)                                                                              \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess)                                                                       \
      throw PmgError(PMG_ERR_CUDA, std::string("NCCL error: ") + nccl_api().GetErrorString(r_)); \
  } while (0)

// ---------------------------------------------------------------- kernels
static __global__ void __launch_bounds__(256) k_pack(const double* __restrict__ src, const int32_t* __restrict__ idx,
                                                     int n, double* __restrict__ buf) {
  pmgdev::pdl_begin();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = src[idx[i]];
}
static __global__ void __launch_bounds__(256) k_unpack(double* __restrict__ dst, const int32_t* __restrict__ idx,
                                                       int n, const double* __restrict__ buf) {
  pmgdev::pdl_begin();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[idx[i]] = buf[i];
}
// combine_records (multigrid.hpp:564-575) over levels, each level's record
// reduced over ranks in rank order: max, sum of squares, count
static __global__ void k_combine_ranks(const pmgdev::Rec* __restrict__ all, int world, int nlev, double* out) {
  pmgdev::pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double m = 0, s = 0;
  long long c = 0;
  for (int l = 0; l <= nlev; ++l) {
    double lm = 0, ls = 0;
    long long lc = 0;
    for (int r = 0; r < world; ++r) {
      const pmgdev::Rec& x = all[(size_t)r * (nlev + 1) + l];
      lm = fmax(lm, x.max);
      ls += x.sumsq;
      lc += x.count;
    }
    m = fmax(m, lm);
    s += ls;
    c += lc;
  }
  out[0] = m;
  out[1] = c > 0 ? sqrt(s / (double)c) : 0.0;
}

// ---------------------------------------------------------------- state
// One exchange pattern: concatenated per-peer cell lists (device), in peer order.
struct DistPlan {
  std::vector<int> peers;           // peer ranks with a non-empty send or receive list
  std::vector<int> scnt, rcnt;      // per listed peer
  std::vector<int> soff, roff;      // prefix offsets into the concatenated lists
  DevBuf<int32_t> sidx, ridx;
  int ns = 0, nr = 0;
  void finish(const std::vector<std::vector<int32_t>>& s, const std::vector<std::vector<int32_t>>& r,
              cudaStream_t st) {
    peers.clear(), scnt.clear(), rcnt.clear(), soff.assign(1, 0), roff.assign(1, 0);
    std::vector<int32_t> cs, cr;
    for (size_t p = 0; p < s.size(); ++p) {
      if (s[p].empty() && r[p].empty()) continue;
      peers.push_back((int)p);
      scnt.push_back((int)s[p].size());
      rcnt.push_back((int)r[p].size());
      cs.insert(cs.end(), s[p].begin(), s[p].end());
      cr.insert(cr.end(), r[p].begin(), r[p].end());
      soff.push_back((int)cs.size());
      roff.push_back((int)cr.size());
    }
    ns = (int)cs.size();
    nr = (int)cr.size();
    sidx.upload(cs, st);
    ridx.upload(cr, st);
  }
  // offset / count of the list sent to (received from) peer p, -1 if none
  int sent_to(int p, int& n) const {
    for (size_t q = 0; q < peers.size(); ++q)
      if (peers[q] == p) {
        n = scnt[q];
        return soff[q];
      }
    n = 0;
    return -1;
  }
};

struct LocalGroup;  // the in-process transport

enum Transport { TR_NONE = 0, TR_NCCL = 1, TR_LOCAL = 2 };

struct DistState {
  int world = 1, rank = 0, split = 1;
  int transport = TR_NONE;
  std::vector<int32_t> owner;                  // by block id
  std::vector<std::array<DistPlan, 3>> halo;   // [level][colour 0, colour 1, both]
  DistPlan gather;                             // level split-1 octant cells -> rank 0
  DevBuf<double> sbuf, rbuf;
  DevBuf<pmgdev::Rec> recs;                    // world x (L+1)
  ncclComm_t comm = nullptr;
  std::shared_ptr<LocalGroup> group;
  cudaEvent_t ev_packed = nullptr, ev_copied = nullptr;
  Graph g;
  bool graph_failed = false;
  ~DistState() {
    g.reset();
    if (comm) nccl_api().CommDestroy(comm);
    if (ev_packed) cudaEventDestroy(ev_packed);
    if (ev_copied) cudaEventDestroy(ev_copied);
  }
};

// Contexts of one process exchanging through device copies: each context is
// driven by its own host thread; a generation barrier orders the enqueues
// (an event is waited on only after its recorder passed the barrier).
struct LocalGroup {
  std::vector<Ctx*> ctx;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g0 = gen;
    if (++arrived == (int)ctx.size()) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g0; });
    }
  }
};

// ---------------------------------------------------------------- plans
// cells (i, j, k) of face d of a block, the lower transverse axis fastest
static void face_cells(int N, int D, int d, std::vector<std::array<int, 3>>& out) {
  out.clear();
  const int ax = d / 2, side = d & 1;
  if (D == 2) {
    for (int t = 0; t < N; ++t) {
      std::array<int, 3> q{0, 0, 0};
      q[(size_t)ax] = side ? N - 1 : 0;
      q[(size_t)(1 - ax)] = t;
      out.push_back(q);
    }
    return;
  }
  const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;
  for (int t1 = 0; t1 < N; ++t1)
    for (int t0 = 0; t0 < N; ++t0) {
      std::array<int, 3> q{0, 0, 0};
      q[(size_t)ax] = side ? N - 1 : 0;
      q[(size_t)o0] = t0;
      q[(size_t)o1] = t1;
      out.push_back(q);
    }
}

static int cell_addr(const Ctx& c, int slot, int i, int j, int k) {
  const int H = c.NI / 2;
  return slot * c.NI + ((i + j + k) & 1) * H + ((i + c.N * (j + c.N * k)) >> 1);
}

static int dist_owner_slot(const Ctx& c, int l, int s) {
  const DistState& ds = *c.dist;
  if (l < ds.split) return 0;
  return ds.owner[(size_t)c.mesh.slots[(size_t)l][(size_t)s]];
}

static void build_dist_plans(Ctx& c) {
  DistState& ds = *c.dist;
  const HostMesh& m = c.mesh;
  const int W = ds.world, R = ds.rank, D = c.dim, N = c.N;
  ds.halo.clear();
  ds.halo.resize((size_t)m.L + 1);
  size_t smax = 1, rmax = 1;
  std::vector<std::array<int, 3>> fc;
  for (int l = std::max(ds.split, 1); l <= m.L; ++l) {
    // [k][peer] cell lists, k = colour 0, colour 1, both
    std::vector<std::vector<int32_t>> snd[3], rcv[3];
    for (int k = 0; k < 3; ++k) snd[k].assign((size_t)W, {}), rcv[k].assign((size_t)W, {});
    const auto& sl = m.slots[(size_t)l];
    for (int s = 0; s < (int)sl.size(); ++s) {
      const int id = sl[(size_t)s];
      const int p = dist_owner_slot(c, l, s);
      for (int d = 0; d < c.F; ++d) {
        const int nid = m.nbr[(size_t)id * 6 + d];
        if (nid < 0) {
          const int cid = m.cnbr[(size_t)id * 6 + d];
          if (cid >= 0 && l - 1 >= ds.split && dist_owner_slot(c, l - 1, m.slot_of[(size_t)cid]) != p)
            throw PmgError(PMG_ERR_INVALID_ARG, "coarse-fine face across a partition boundary");
          continue;
        }
        const int q = dist_owner_slot(c, l, m.slot_of[(size_t)nid]);
        if (q == p || (p != R && q != R)) continue;
        // q's block nid reads this block's face layer on side d: p -> q
        face_cells(N, D, d, fc);
        for (const auto& x : fc) {
          const int a = cell_addr(c, s, x[0], x[1], x[2]);
          const int col = (x[0] + x[1] + x[2]) & 1;
          auto& L0 = p == R ? snd[col][(size_t)q] : rcv[col][(size_t)p];
          auto& L2 = p == R ? snd[2][(size_t)q] : rcv[2][(size_t)p];
          L0.push_back(a);
          L2.push_back(a);
        }
      }
    }
    for (int k = 0; k < 3; ++k) {
      ds.halo[(size_t)l][(size_t)k].finish(snd[k], rcv[k], c.stream);
      smax = std::max(smax, (size_t)ds.halo[(size_t)l][(size_t)k].ns);
      rmax = std::max(rmax, (size_t)ds.halo[(size_t)l][(size_t)k].nr);
    }
  }
  // gather: the octants of the split level's parents, from the children's ranks to rank 0
  if (ds.split >= 2) {
    const int g = ds.split, HN = N / 2;
    std::vector<std::vector<int32_t>> snd((size_t)W), rcv((size_t)W);
    const auto& sl = m.slots[(size_t)g];
    for (int s = 0; s < (int)sl.size(); ++s) {
      const int id = sl[(size_t)s];
      const int p = dist_owner_slot(c, g, s);
      if (p == 0 || (R != 0 && R != p)) continue;
      const int ps = m.slot_of[(size_t)m.parent[(size_t)id]];
      int o[3] = {0, 0, 0};
      for (int a = 0; a < D; ++a) o[a] = (m.coords[(size_t)id * 3 + a] & 1) * HN;
      auto& L = R == 0 ? rcv[(size_t)p] : snd[0];
      for (int kk = 0; kk < (D == 3 ? HN : 1); ++kk)
        for (int jj = 0; jj < HN; ++jj)
          for (int ii = 0; ii < HN; ++ii)
            L.push_back(cell_addr(c, ps, o[0] + ii, o[1] + jj, D == 3 ? o[2] + kk : 0));
    }
    ds.gather.finish(snd, rcv, c.stream);
    smax = std::max(smax, (size_t)ds.gather.ns);
    rmax = std::max(rmax, (size_t)ds.gather.nr);
  }
  ds.sbuf.alloc(smax);
  ds.rbuf.alloc(rmax);
  ds.recs.alloc((size_t)W * (size_t)(m.L + 1));
}

// ---------------------------------------------------------------- per-rank memory
#define PMG_CU(x)                                                                                 \
  do {                                                                                            \
    CUresult r_ = (x);                                                                            \
    if (r_ != CUDA_SUCCESS)                                                                       \
      throw PmgError(PMG_ERR_CUDA, "CUDA driver error " + std::to_string((int)r_) + " at " #x);   \
  } while (0)

// Replace `buf` (slot-major, slot_bytes per block) by a sparse copy that maps
// only the chunks holding the blocks flagged in `need`.
static void make_sparse(Ctx& c, DevBuf<double>& buf, const std::vector<uint8_t>& need, size_t slot_bytes) {
  VmmApi& v = vmm_api();
  if (!v.ok) throw PmgError(PMG_ERR_CUDA, "CUDA virtual memory management unavailable");
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c.device;
  size_t gran = 0;
  PMG_CU(v.Granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  const size_t total = buf.n * sizeof(double), size = (total + gran - 1) / gran * gran, nch = size / gran;
  std::vector<uint8_t> ch(nch, 0);
  for (size_t s = 0; s < need.size(); ++s)
    if (need[s])
      for (size_t q = s * slot_bytes / gran; q <= ((s + 1) * slot_bytes - 1) / gran; ++q) ch[q] = 1;
  auto sa = std::make_shared<SparseAlloc>();
  sa->size = size;
  PMG_CU(v.AddressReserve(&sa->base, size, gran, 0, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t q = 0; q < nch;) {
    if (!ch[q]) {
      ++q;
      continue;
    }
    size_t e = q;
    while (e < nch && ch[e]) ++e;
    const size_t off = q * gran, bytes = (e - q) * gran;
    CUmemGenericAllocationHandle hnd;
    PMG_CU(v.Create(&hnd, bytes, &prop, 0));
    sa->runs.emplace_back(off, bytes);
    sa->handles.push_back(hnd);
    PMG_CU(v.Map(sa->base + off, bytes, 0, hnd, 0));
    PMG_CU(v.SetAccess(sa->base + off, bytes, &acc, 1));
    sa->mapped += bytes;
    PMG_CUDA(cudaMemcpyAsync((char*)sa->base + off, (const char*)buf.p + off, std::min(bytes, total - off),
                             cudaMemcpyDeviceToDevice, c.stream));
    q = e;
  }
  PMG_CUDA(cudaStreamSynchronize(c.stream));
  const size_t n = buf.n;
  buf.release();
  buf.p = (double*)sa->base;
  buf.n = n;
  buf.sp = sa;
}

// Fields of the levels >= split with more than kSmallLevel blocks keep only
// this rank's blocks and their same-level face neighbours (the halo); the
// small levels and the coarse tail stay whole.
static void shrink_fields(Ctx& c) {
  DistState& ds = *c.dist;
  const HostMesh& m = c.mesh;
  for (int l = ds.split; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    if (d.nb <= kSmallLevel) continue;
    std::vector<uint8_t> need((size_t)d.nb, 0);
    for (int s = 0; s < d.nb; ++s) {
      if (dist_owner_slot(c, l, s) != ds.rank) continue;
      need[(size_t)s] = 1;
      const int id = m.slots[(size_t)l][(size_t)s];
      for (int f = 0; f < c.F; ++f) {
        const int nid = m.nbr[(size_t)id * 6 + f];
        if (nid >= 0) need[(size_t)m.slot_of[(size_t)nid]] = 1;
      }
    }
    const size_t sb = (size_t)c.NI * sizeof(double);
    make_sparse(c, d.phi, need, sb);
    make_sparse(c, d.rhs, need, sb);
    make_sparse(c, d.old, need, sb);
    make_sparse(c, d.res, need, sb);
  }
  c.staging.release();  // whole-mesh upload staging: allocated again on demand
}

// ---------------------------------------------------------------- transport
static double* level_var(Ctx& c, int var, int l) {
  LevelDev& d = *c.lev[(size_t)l];
  switch (var) {
    case PMG_VAR_PHI: return d.phi.p;
    case PMG_VAR_RHS: return d.rhs.p;
    case PMG_VAR_OLD: return d.old.p;
    default: return d.res.p;
  }
}

// the exchange pattern (level l, colour set k) or, for l < 0, the gather
static DistPlan& dist_plan(Ctx& c, int l, int k) {
  return l < 0 ? c.dist->gather : c.dist->halo[(size_t)l][(size_t)k];
}

// move the cells of pattern (l, k) of `field`: pack, transport, unpack
static void dist_move(Ctx& c, int l, int k, double* field) {
  DistState& ds = *c.dist;
  DistPlan& P = dist_plan(c, l, k);
  if (P.ns > 0)
    pdl_launch(k_pack, (unsigned)std::min((P.ns + 255) / 256, 4 * c.sms), 256, 0, c.stream, (const double*)field,
               (const int32_t*)P.sidx.p, P.ns, ds.sbuf.p);
  if (ds.transport == TR_NCCL) {
    if (!P.peers.empty()) {
      PMG_NCCL(nccl_api().GroupStart());
      for (size_t q = 0; q < P.peers.size(); ++q) {
        if (P.scnt[q])
          PMG_NCCL(nccl_api().Send(ds.sbuf.p + P.soff[q], (size_t)P.scnt[q], ncclFloat64, P.peers[q], ds.comm,
                                   c.stream));
        if (P.rcnt[q])
          PMG_NCCL(nccl_api().Recv(ds.rbuf.p + P.roff[q], (size_t)P.rcnt[q], ncclFloat64, P.peers[q], ds.comm,
                                   c.stream));
      }
      PMG_NCCL(nccl_api().GroupEnd());
    }
  } else if (ds.transport == TR_LOCAL) {
    LocalGroup& G = *ds.group;
    PMG_CUDA(cudaEventRecord(ds.ev_packed, c.stream));
    G.barrier();  // every peer's pack is enqueued and recorded
    for (size_t q = 0; q < P.peers.size(); ++q) {
      if (!P.rcnt[q]) continue;
      Ctx& pc = *G.ctx[(size_t)P.peers[q]];
      int n = 0;
      const int off = dist_plan(pc, l, k).sent_to(ds.rank, n);  // the peer's list for this rank
      if (off < 0 || n != P.rcnt[q]) throw PmgError(PMG_ERR_STATE, "halo plans of two ranks disagree");
      PMG_CUDA(cudaStreamWaitEvent(c.stream, pc.dist->ev_packed, 0));
      PMG_CUDA(cudaMemcpyAsync(ds.rbuf.p + P.roff[q], pc.dist->sbuf.p + off, (size_t)n * 8, cudaMemcpyDefault,
                               c.stream));
    }
    PMG_CUDA(cudaEventRecord(ds.ev_copied, c.stream));
    G.barrier();  // every peer's copies are enqueued and recorded
    for (Ctx* pc : G.ctx)  // our send buffer is reused only after every peer copied from it
      if (pc != &c) PMG_CUDA(cudaStreamWaitEvent(c.stream, pc->dist->ev_copied, 0));
  }
  if (P.nr > 0)
    pdl_launch(k_unpack, (unsigned)std::min((P.nr + 255) / 256, 4 * c.sms), 256, 0, c.stream, field,
               (const int32_t*)P.ridx.p, P.nr, (const double*)ds.rbuf.p);
  PMG_CUDA(cudaGetLastError());
}

static void dist_xchg(Ctx& c, int var, int l, int k) {
  DistState& ds = *c.dist;
  if (ds.world == 1 || l < ds.split) return;
  dist_move(c, l, k, level_var(c, var, l));
  phi_written(c, l);  // halo cells of level l changed (whatever `var`)
}

// whole level l of `var` from rank 0 to every rank
static void dist_bcast_level(Ctx& c, int var, int l) {
  DistState& ds = *c.dist;
  double* f = level_var(c, var, l);
  const size_t n = (size_t)c.lev[(size_t)l]->nb * c.NI;
  phi_written(c, l);
  if (ds.transport == TR_NCCL) {
    PMG_NCCL(nccl_api().Broadcast(f, f, n, ncclFloat64, 0, ds.comm, c.stream));
  } else if (ds.transport == TR_LOCAL) {
    LocalGroup& G = *ds.group;
    PMG_CUDA(cudaEventRecord(ds.ev_packed, c.stream));
    G.barrier();
    if (ds.rank != 0) {
      Ctx& r0 = *G.ctx[0];
      PMG_CUDA(cudaStreamWaitEvent(c.stream, r0.dist->ev_packed, 0));
      PMG_CUDA(cudaMemcpyAsync(f, level_var(r0, var, l), n * 8, cudaMemcpyDefault, c.stream));
    }
    PMG_CUDA(cudaEventRecord(ds.ev_copied, c.stream));
    G.barrier();
    if (ds.rank == 0)
      for (Ctx* pc : G.ctx)
        if (pc != &c) PMG_CUDA(cudaStreamWaitEvent(c.stream, pc->dist->ev_copied, 0));
  }
}

// every rank's per-level records, combined in rank order into c.stats
static void dist_records(Ctx& c) {
  DistState& ds = *c.dist;
  const size_t per = (size_t)c.mesh.L + 1;
  if (ds.transport == TR_NCCL) {
    PMG_NCCL(nccl_api().AllGather(c.rec.p, ds.recs.p, per * sizeof(pmgdev::Rec), ncclUint8, ds.comm, c.stream));
  } else if (ds.transport == TR_LOCAL) {
    LocalGroup& G = *ds.group;
    PMG_CUDA(cudaEventRecord(ds.ev_packed, c.stream));
    G.barrier();
    for (size_t r = 0; r < G.ctx.size(); ++r) {
      Ctx& pc = *G.ctx[r];
      if (&pc != &c) PMG_CUDA(cudaStreamWaitEvent(c.stream, pc.dist->ev_packed, 0));
      PMG_CUDA(cudaMemcpyAsync(ds.recs.p + r * per, pc.rec.p, per * sizeof(pmgdev::Rec), cudaMemcpyDefault,
                               c.stream));
    }
    PMG_CUDA(cudaEventRecord(ds.ev_copied, c.stream));
    G.barrier();
    for (Ctx* pc : G.ctx)
      if (pc != &c) PMG_CUDA(cudaStreamWaitEvent(c.stream, pc->dist->ev_copied, 0));
  } else {
    PMG_CUDA(cudaMemcpyAsync(ds.recs.p, c.rec.p, per * sizeof(pmgdev::Rec), cudaMemcpyDeviceToDevice, c.stream));
  }
  pdl_launch(k_combine_ranks, 1, 32, 0, c.stream, (const pmgdev::Rec*)ds.recs.p, ds.world, c.mesh.L, c.stats.p);
  PMG_CUDA(cudaGetLastError());
}

}  // namespace pmghost
