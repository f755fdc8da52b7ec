// ctx.h -- host-side state of one solver context (one mesh on one device).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <memory>
#include <unordered_set>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmg_b200.h"
#include "kernels.cuh"

namespace pmghost {

struct PmgError : std::runtime_error {
  int code;
  PmgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PMG_CUDA(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::pmghost::PmgError(PMG_ERR_CUDA, std::string("CUDA error: ") +            \
                                                  cudaGetErrorString(e_) + " at " #x); \
  } while (0)

// Kernel launch with programmatic stream serialization (programmatic
// dependent launch): the next kernel of the stream -- or of the captured
// graph -- is scheduled while this one drains; every kernel starts with
// pmgdev::pdl_begin() (griddepcontrol.wait), so correctness does not depend on
// it.  Off by default (measured no gain inside the captured cycle graphs;
// the streaming kernels occupy every SM); PMG_PDL=1 enables it.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PMG_PDL");
    return e && *e && *e != '0';
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PMG_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// the same, always with programmatic stream serialization (kernels that load
// their static data before griddepcontrol.wait)
template <typename... KArgs, typename... Args>
inline void pdl_launch_on(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PMG_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// Sparse device array (CUDA virtual memory management, driver entry points
// resolved at run time): the whole index range is reserved, physical memory
// is mapped only for the chunks a rank touches (its blocks and their halo
// blocks), so a partitioned rank holds its share of the mesh, not all of it.
struct VmmApi {
  bool ok = false;
  CUresult (*AddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*AddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*Create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*Release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*Map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*Unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*SetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*Granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
};
inline VmmApi& vmm_api() {
  static VmmApi a = [] {
    VmmApi x;
    auto get = [](const char* n) -> void* {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(n, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
      return f;
    };
    x.AddressReserve = (decltype(x.AddressReserve))get("cuMemAddressReserve");
    x.AddressFree = (decltype(x.AddressFree))get("cuMemAddressFree");
    x.Create = (decltype(x.Create))get("cuMemCreate");
    x.Release = (decltype(x.Release))get("cuMemRelease");
    x.Map = (decltype(x.Map))get("cuMemMap");
    x.Unmap = (decltype(x.Unmap))get("cuMemUnmap");
    x.SetAccess = (decltype(x.SetAccess))get("cuMemSetAccess");
    x.Granularity = (decltype(x.Granularity))get("cuMemGetAllocationGranularity");
    x.ok = x.AddressReserve && x.AddressFree && x.Create && x.Release && x.Map && x.Unmap && x.SetAccess &&
           x.Granularity;
    (void)cudaGetLastError();
    return x;
  }();
  return a;
}
struct SparseAlloc {
  CUdeviceptr base = 0;
  size_t size = 0;
  std::vector<std::pair<size_t, size_t>> runs;  // mapped (offset, bytes)
  std::vector<CUmemGenericAllocationHandle> handles;
  size_t mapped = 0;
  SparseAlloc() = default;
  SparseAlloc(const SparseAlloc&) = delete;
  SparseAlloc& operator=(const SparseAlloc&) = delete;
  ~SparseAlloc() {
    VmmApi& v = vmm_api();
    for (size_t i = 0; i < runs.size(); ++i) {
      v.Unmap(base + runs[i].first, runs[i].second);
      v.Release(handles[i]);
    }
    if (base) v.AddressFree(base, size);
  }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  std::shared_ptr<SparseAlloc> sp;  // set: p lies in a sparse (VMM) range
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), sp(std::move(o.sp)) { o.p = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n, sp = std::move(o.sp);
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (sp) sp.reset();
    else if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return sp ? sp->mapped : n * sizeof(T); }
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    PMG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size());
    if (!v.empty()) PMG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// levels with at most this many blocks run the per-cell (small-level) kernels:
// they are latency-bound, and a cell per thread gives the most loads in flight
constexpr int kSmallLevel = 64;

struct HostMesh {
  int nb = 0;
  int L = 0;
  std::vector<int32_t> level, coords, parent, children, nbr, cnbr;  // coords nb*3, children nb*8, nbr nb*6
  std::vector<double> origin, dx;
  std::vector<std::vector<int32_t>> slots;      // per level: block ids in device slot (Morton) order
  std::vector<std::vector<int32_t>> ref_order;  // per level: block ids in level_blocks (x-major) order
  std::vector<int32_t> slot_of;                 // block id -> slot within its level
};

struct HostStencils {
  bool valid = false;
  std::vector<int32_t> boundary, row_count, row_start;
  // row_of (StencilSet::row_of, one N^D page per block) kept for the boundary
  // blocks only: row_page[id] = page index or -1 (every entry -1)
  int NI = 0;
  std::vector<int32_t> row_page, row_pages;
  int32_t row_at(size_t id, size_t ii) const {
    const int32_t p = row_page[id];
    return p < 0 ? -1 : row_pages[(size_t)p * (size_t)NI + ii];
  }
  const int32_t* page(size_t id) const { return row_pages.data() + (size_t)row_page[id] * (size_t)NI; }
  std::vector<double> center, nb, bc, d;
  std::vector<int8_t> obj, pin;
  std::vector<uint8_t> mask;
  std::vector<int32_t> lin;
  std::vector<double> phi_b;
};

// the StencilSet's rows on the device (capi.cu ensure_devrows)
struct DevRows {
  DevBuf<double> center, nb, bc, d;
  DevBuf<int8_t> obj, pin;
  DevBuf<uint8_t> mask;
  DevBuf<int32_t> rowof;  // pages in HostStencils::row_page order
};

struct HostCoarse {
  int n = 0;
  std::vector<int32_t> rp, ci;
  std::vector<double> val, c0, cobj;  // cobj n_obj*n
  std::vector<int32_t> unk_block, unk_lin, uaddr;
  std::vector<double> dinv;
};

struct LevelDev {
  int nb = 0;
  int n_leaf = 0;  // leaf blocks (levels without leaves keep a zero record)
  DevBuf<uint8_t> own;  // multi-GPU ownership mask by slot (pmg_b200_set_owned)
  bool has_own = false;
  int n_own = 0;        // blocks this rank computes (nb unless set_owned restricted them)
  DevBuf<int32_t> nbr, cnbr, coords, parent, child, srow, bcoff, cfoff, row_of, slot_id;
  DevBuf<uint8_t> leaf, kind, r_mask;
  DevBuf<double> phi, rhs, old, res, bcval, cfold, r_center, r_nb, r_bc, r_d;
  DevBuf<double> r_coef;  // 16 per row (k_row_coef)
  size_t n_rows = 0;      // special rows of the level's interface blocks
  DevBuf<int8_t> r_obj, r_pin, skind;
  DevBuf<int32_t> ref_slot;  // level_blocks order position -> slot
  // block classes: "fast" = uniform stencil and all 2D faces same-level
  // (served by the lean kernels), "slow" = everything else
  DevBuf<int32_t> fast_list, slow_list;
  int n_fast = 0, n_slow = 0;
  // residual-family classes: lean = uniform stencil without coarse-fine faces
  DevBuf<int32_t> ufast_list, uslow_list;
  int n_ufast = 0, n_uslow = 0;
  // streaming GS (stream.cuh): lean blocks that are not entirely inside
  DevBuf<int32_t> gs_plan;  // 8 int32 per block (stream.cuh BlockPlan)
  int n_gs = 0;
  DevBuf<int32_t> rs_plan;  // every block without coarse-fine faces (incl. all-inside)
  int n_rs = 0;
  DevBuf<int32_t> ur_plan;  // uniform blocks without coarse-fine faces (= ufast_list)
  int n_ur = 0;
  DevBuf<int32_t> rfix_list;  // (slot, parent-local index) pairs for k_restrict_fix
  int n_rfix = 0;
  std::vector<int32_t> rfix_host;
  DevBuf<int32_t> rfix_tab;   // per listed parent: 2^D child gather entries (capi.cu cell_entry)
  DevBuf<double> rfix_gbc;
  DevBuf<int32_t> pin_list;   // (cell address, object) of this level's inside rows
  int n_pin = 0;
  DevBuf<int32_t> pp_plan;    // streaming prolongation plan (stream.cuh), -1: level not eligible
  int n_pp = -1;
  bool pp_cf = false;         // some parent-octant face in pp_plan is coarse-fine (CF kernel)
  DevBuf<int32_t> tab;        // small levels: per-cell row code + neighbour addresses (small.cuh)
  DevBuf<double> tgbc;
  bool has_tab = false;
  // k_gs_cut tables per colour: 8 int32 (cell, row, 6 neighbour addresses) + 6 ghost bc values
  DevBuf<int32_t> cut_ent[2];
  DevBuf<double> cut_gbc[2];
  DevBuf<double> cut_coef[2];  // 16 per cut row: center, nb[6], bc*phi_b[6], bc mask
  int n_cut[2] = {0, 0};
  DevBuf<int32_t> cut_off[2];  // nb + 1 per colour: cut rows of slot s (k_gs_coop)
  int coop = -1;               // k_gs_coop smooths this level (-1: not yet decided)
  DevBuf<int32_t> fix_list[2];  // (slot, entry) pairs of special rows in lean interface blocks
  int n_fix[2] = {0, 0};
  bool has_cf = false;       // some block has a coarse-fine face
  bool has_cfold = false;
  // coarse parts of the coarse-fine ghosts (LevelView::cfc): the level's
  // coarse-fine faces {slot, dir}, the table, and whether level l-1's PHI
  // changed since the table was built
  DevBuf<int32_t> cf_faces, cf_desc;  // cf_desc: 8 int32 per face for k_cfc_build (capi.cu set_mesh)
  int n_cf = 0;
  std::vector<int32_t> cfoff_host;  // cfoff as uploaded (the streaming plans carry the cfc page numbers)
  // streaming GS of blocks with coarse-fine faces (3D N = 8 / 16): they join
  // gs_plan with their faces' cfc pages (BlockPlan), their cut rows have
  // their own k_gs_cut tables, and only blocks with a cut row within two cells of a
  // coarse-fine face stay with k_gs_tile (gs_slow)
  bool gs_cf = false;
  DevBuf<int32_t> gs_slow;
  int n_gs_slow = 0;
  // streaming record (3D N = 8, or N = 16 with coarse-fine faces): the leaf
  // blocks the column kernel can take (BlockPlan entries with cfc pages), and
  // the leaf blocks with a cut row near a coarse-fine face (k_record_tile)
  DevBuf<int32_t> rc_plan, rc_slow;
  int n_rc = 0, n_rc_slow = 0;
  // streaming residual + restriction on the same levels: every block whose
  // parents with a cut child keep clear of the coarse-fine faces (k_restrict_fix
  // gathers cannot express those ghosts); the others by k_restrict_tile
  DevBuf<int32_t> rr_plan, rr_slow;
  int n_rr = 0, n_rr_slow = 0;
  DevBuf<int32_t> cutcf_ent[2];
  DevBuf<double> cutcf_gbc[2], cutcf_coef[2];
  int n_cutcf[2] = {0, 0};
  DevBuf<double> cfc;
  bool cfc_dirty = true;
  bool dense = false;   // all blocks present, slot == Morton code
  bool bczero = true;   // no Dirichlet face values (all zero)
  pmgdev::LevelView view{};
};

struct Ctx;
struct DistState;  // dist.h: the Morton-partitioned cycle

// Launchers, templated on (Dim, N) inside ops.cu.
struct Ops {
  virtual ~Ops() = default;
  virtual void gs(Ctx& c, int l, int parity) = 0;
  // smooth(l, steps) as one cooperative launch; false: not eligible (use gs)
  virtual bool smooth(Ctx& c, int l, int steps) = 0;
  virtual void residual(Ctx& c, int l) = 0;
  virtual void restrict_(Ctx& c, int l, int mode) = 0;
  virtual void fas(Ctx& c, int lc, bool fas) = 0;
  virtual void cfold(Ctx& c, int lc) = 0;
  // FAS right-hand side / OLD of level lc and, beside it on the forked stream,
  // the OLD ghost snapshot of its coarse-fine faces (both only read PHI)
  virtual void fas_cfold(Ctx& c, int lc, bool fas) = 0;
  virtual void cfc_build(Ctx& c, int l) = 0;
  // the block-per-CTA kernels read coarse-fine ghosts from the cfc table, so
  // residual + restriction of a level with coarse-fine faces is one pass
  virtual bool cf_table() const = 0;
  virtual void prolong(Ctx& c, int l, bool full) = 0;
  virtual void record(Ctx& c, int l) = 0;
  virtual void pins(Ctx& c, int l) = 0;
  virtual void coarse(Ctx& c) = 0;
  // face_gradient (fields.hpp:149-232) of PHI over the leaves: faces[n_leaves][D][(N+1) N^(D-1)],
  // optionally the cell-centred magnitude mag[n_leaves][N^D]
  virtual void face_gradient(Ctx& c, int n_leaves, double* faces, double* mag) = 0;
  // error_norms against the analytic sphere solution (fields.hpp:35-69): fills
  // `part` with 3 doubles per CTA (max |d|, sum w d^2, sum w), returns the CTA count
  virtual int error_norms(Ctx& c, int n_leaves, const double* origin, int tag, double phi_b, double a,
                          double R, int vw, double* part, int* err) = 0;
  virtual void scatter(Ctx& c, int l, double* dst, const double* staging, const int32_t* slot_id,
                       int layout) = 0;
  virtual void gather(Ctx& c, int l, int var, double* staging, const int32_t* slot_id,
                      int layout) = 0;
  virtual void build_stencils(Ctx& c, const pmg_lsf_t* lsf, int n_lsf,
                              const pmg_stencil_cfg_t* cfg) = 0;
};
std::unique_ptr<Ops> make_ops(int dim, int N);

struct Graph {
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    kernels = 0;
  }
  ~Graph() { reset(); }
};

struct Ctx {
  int dim = 3, N = 16, F = 6, NI = 0, S = 0, NT = 0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  int device = 0;
  std::vector<std::vector<uint8_t>> owned;  // per level, by slot (empty: every block)
  int sms = 148;  // multiprocessors of `device`
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // forked branch for concurrent block classes
  // double-buffered field upload (pmg_b200_stage_field_async / commit_staged_field)
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_consumed = nullptr;
  DevBuf<double> stage2;
  int staged_var = -1, staged_level = 0, staged_layout = 0;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string err;

  HostMesh mesh;
  bool have_mesh = false;
  int bctype[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> face_vals[6];  // per dir, concatenated over physical-face blocks in id order
  std::vector<int32_t> face_off[6];  // per dir, per block: offset into face_vals[dir] or -1

  HostStencils st;
  std::unique_ptr<DevRows> devrows;
  HostCoarse coarse;
  std::vector<std::unique_ptr<LevelDev>> lev;  // index 0 unused
  DevBuf<double> phi_b;
  // outbuf: stats[2], diag[2], status (int32 in one double), then the level
  // records -- one D2H copy and one memset per cycle instead of three and two
  DevBuf<double> outbuf;
  template <typename T>
  struct View {
    T* p = nullptr;
    size_t n = 0;
  };
  View<pmgdev::Rec> rec;
  DevBuf<pmgdev::Rec> partial;
  DevBuf<int2> leaf_tab;            // (level, slot) of every leaf in dump order (io.hpp:17-21)
  DevBuf<double> ff_faces, ff_mag;  // face_gradient scratch
  DevBuf<unsigned int> counter;
  View<double> stats, diag;
  View<int> status;
  DevBuf<double> staging;
  // coarse system on device
  DevBuf<int32_t> c_rp, c_ci, c_uaddr;
  DevBuf<double> c_val, c_dinv, c_c0, c_cobj, c_scratch;
  // cell-indexed level-1 operator for the on-chip BiCGStab (coarse.cuh)
  DevBuf<uint8_t> cf_flags;
  DevBuf<double> cf_diag, cf_spec_c, cf_c0, cf_ob_val;
  DevBuf<int16_t> cf_spec;
  DevBuf<int32_t> cf_ob_start;
  DevBuf<int8_t> cf_ob_obj;
  double cf_w = 0;

  double* h_out = nullptr;  // pinned image of outbuf's first 5 doubles: stats[2], diag[2], status
  void* h_buf = nullptr;    // pinned transfer buffer (pmg_b200_host_buffer)
  size_t h_buf_bytes = 0;
  int* h_status = nullptr;  // = (int*)(h_out + 4)
  double* h_out_dev = nullptr;  // device address of h_out (mapped pinned memory)
  // the cycle's last record (level finish_level) writes the CycleStats and
  // the host copy itself (k_record_fold's FinishArgs); `finished` tells
  // enq_finish that it did
  int finish_level = 0;
  bool finished = false;

  pmg_mg_cfg_t cfg{2, 2, 1e-6, 2000, 1};
  bool solver = false;
  bool have_guess = false;
  // colour whose prolonged values the caller overwrites next (the V-cycle's
  // first post-smoothing half-sweep), -1: every cell (the op-level API)
  int prolong_dead = -1;
  std::unique_ptr<Ops> ops;
  Graph g_v, g_fmg[2], g_measure;
  bool graphs_dirty = true;

  // kernels whose >48 KB dynamic shared memory / non-portable cluster
  // attribute is set: cudaFuncSetAttribute is per device, a context is one device
  std::unordered_set<const void*> attr_done;
  DevBuf<unsigned> gbar;  // k_gs_coop grid barrier {count, generation}
  int cluster16 = -1;  // 16-CTA coarse-solve cluster schedulable (-1: not yet queried)
  std::unique_ptr<DistState> dist;  // pmg_b200_set_partition (nullptr: one context, whole mesh)

  ~Ctx();
};

// PHI of level l was (or may have been) written: the cfc table of level l+1 is stale
inline void phi_written(Ctx& c, int l) {
  if (l >= 1 && l + 1 < (int)c.lev.size() && c.lev[(size_t)l + 1]) c.lev[(size_t)l + 1]->cfc_dirty = true;
}
inline void cfc_all_dirty(Ctx& c) {
  for (auto& d : c.lev)
    if (d) d->cfc_dirty = true;
}
inline void ensure_cfc(Ctx& c, int l) {
  LevelDev& d = *c.lev[(size_t)l];
  if (d.n_cf == 0 || !d.cfc_dirty) return;
  c.ops->cfc_build(c, l);
  d.cfc_dirty = false;
}

inline void set_smem_attr(Ctx& c, const void* fn, size_t smem) {
  if (!c.attr_done.insert(fn).second) return;
  PMG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}
inline void set_cluster_attr(Ctx& c, const void* fn) {
  if (!c.attr_done.insert(fn).second) return;
  PMG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

}  // namespace pmghost
