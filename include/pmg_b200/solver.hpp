// pmg_b200/solver.hpp -- header-only C++ drop-in for the reference solver API.
//
//   #include "pmg/multigrid.hpp"          // the reference (mesh, stencils, config)
//   #include "pmg_b200/solver.hpp"        // this header; link libpmg_b200.so
//
//   pmg::b200::MgSolver<3> solver(mesh, stencils, cfg);   // was pmg::MgSolver<3>
//   pmg::CycleStats s = solver.v_cycle();
//
// pmg::b200::MgSolver<Dim> has the public surface of pmg::MgSolver<Dim>
// (proj/include/pmg/multigrid.hpp:292-480): same constructor arguments, same
// methods, same CycleStats, same exception types and messages.  The mesh and
// stencils are the reference's own pmg::TreeMesh<Dim> / pmg::StencilSet<Dim>;
// they are uploaded once (topology, face BCs evaluated at the face centres,
// stencil rows, PHI and RHS) and every cycle runs on the GPU through the C-ABI
// of include/pmg_b200.h.  Like the reference, the solver holds non-owning
// references: after each cycle PHI is copied back into mesh.field(id, VAR_PHI)
// (ghosts included) unless set_sync_to_host(false) -- then call sync_to_host()
// when the host copy is needed.  pmg::b200::build_stencils replaces
// pmg::build_stencils (stencil.hpp:207-222) with the GPU build and returns an
// identical StencilSet.
#ifndef PMG_B200_SOLVER_HPP
#define PMG_B200_SOLVER_HPP

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pmg/fields.hpp"
#include "pmg/multigrid.hpp"
#include "pmg_b200.h"

namespace pmg {
namespace b200 {

namespace detail {

inline void check(pmg_b200_ctx* h, int rc) {
  if (rc == PMG_OK) return;
  const std::string msg = pmg_b200_last_error(h);
  if (rc == PMG_ERR_TOPOLOGY) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

template <int Dim>
void upload_mesh(pmg_b200_ctx* h, const TreeMesh<Dim>& mesh);

template <int Dim>
pmg_b200_ctx* make_context(const TreeMesh<Dim>& mesh, int device) {
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int k = 0; k < Dim; ++k) {
    lo[k] = mesh.domain_lo()[k];
    hi[k] = mesh.domain_hi()[k];
  }
  pmg_b200_ctx* h = pmg_b200_create(Dim, mesh.block_size(), lo, hi, device);
  if (!h) throw std::runtime_error("pmg_b200_create: out of memory");
  try {  // the context is destroyed on any failure below
    if (*pmg_b200_last_error(h)) throw std::runtime_error(pmg_b200_last_error(h));
    upload_mesh<Dim>(h, mesh);
  } catch (...) {
    pmg_b200_destroy(h);
    throw;
  }
  return h;
}

// topology and physical face values of the reference's mesh
template <int Dim>
void upload_mesh(pmg_b200_ctx* h, const TreeMesh<Dim>& mesh) {
  const int nb = mesh.n_blocks();
  std::vector<int32_t> level(nb), coords(nb * 3, 0), parent(nb), children(nb * 8, -1),
      nbr(nb * 6, -1), cnbr(nb * 6, -1);
  std::vector<double> origin(nb * 3, 0.0), dx(nb);
  for (int id = 0; id < nb; ++id) {
    const Block<Dim>& b = mesh.block(id);
    level[id] = b.level;
    dx[id] = b.dx;
    parent[id] = b.parent;
    for (int k = 0; k < Dim; ++k) {
      coords[id * 3 + k] = b.coords[k];
      origin[id * 3 + k] = b.origin[k];
    }
    for (int c = 0; c < (1 << Dim); ++c) children[id * 8 + c] = b.children[c];
    for (int f = 0; f < 2 * Dim; ++f) {
      nbr[id * 6 + f] = b.nbr[f];
      cnbr[id * 6 + f] = b.coarse_nbr[f];
    }
  }
  check(h, pmg_b200_set_mesh(h, nb, level.data(), coords.data(), origin.data(), dx.data(),
                             parent.data(), children.data(), nbr.data(), cnbr.data()));
  // face BCs: the std::function evaluated at every physical ghost-face centre
  // (mesh.hpp:538-552), in block-id order
  const int N = mesh.block_size();
  for (int dir = 0; dir < 2 * Dim; ++dir) {
    const FaceBc<Dim>& fb = mesh.face_bc[dir];
    std::vector<double> vals;
    if (fb.type == FaceBcType::dirichlet && fb.value) {
      const int axis = dir / 2, side = dir & 1;
      for (int id = 0; id < nb; ++id) {
        const Block<Dim>& b = mesh.block(id);
        if (b.nbr[dir] >= 0 || b.coarse_nbr[dir] >= 0) continue;
        const int nt = Dim == 2 ? N : N * N;
        for (int t = 0; t < nt; ++t) {
          IVec<Dim> i1{};
          int u = t;
          for (int k = 0; k < Dim; ++k) {
            if (k == axis) continue;
            i1[k] = u % N;
            u /= N;
          }
          i1[axis] = side ? N - 1 : 0;
          Vec<Dim> xf = mesh.cell_center(b, i1);
          xf[axis] += 0.5 * b.dx * dir_sign(dir);
          vals.push_back(fb.eval(xf));
        }
      }
    }
    check(h, pmg_b200_set_face_bc(h, dir,
                                  fb.type == FaceBcType::neumann_zero ? PMG_BC_NEUMANN_ZERO
                                                                      : PMG_BC_DIRICHLET,
                                  vals.empty() ? nullptr : vals.data()));
  }
}

template <int Dim>
void upload_stencils(pmg_b200_ctx* h, const TreeMesh<Dim>& mesh, const StencilSet<Dim>& set) {
  const int nb = mesh.n_blocks();
  size_t ni = 1;
  for (int k = 0; k < Dim; ++k) ni *= (size_t)mesh.block_size();
  constexpr int F = 2 * Dim;
  std::vector<int32_t> boundary(nb, 0), rc(nb, 0), row_of((size_t)nb * ni, -1), lin;
  std::vector<double> center, nbv, bcv, dv;
  std::vector<int8_t> obj, pin;
  std::vector<uint8_t> mask;
  for (int id = 0; id < nb; ++id) {
    const BlockStencil<Dim>& st = set.by_block[(size_t)id];
    boundary[id] = st.boundary ? 1 : 0;
    if (!st.boundary) continue;
    std::copy(st.row_of.begin(), st.row_of.end(), row_of.begin() + (long)id * (long)ni);
    rc[id] = (int32_t)st.rows.size();
    for (const auto& c : st.rows) {
      center.push_back(c.center);
      for (int f = 0; f < F; ++f) {
        nbv.push_back(c.nb[f]);
        bcv.push_back(c.bc[f]);
        dv.push_back(c.d[f]);
        obj.push_back(c.obj[f]);
      }
      mask.push_back(c.mask);
      pin.push_back(c.pin_obj);
      lin.push_back(c.lin);
    }
  }
  std::vector<double> phib = set.bv.phi_b;
  if (center.empty()) {  // keep pointers valid
    center.push_back(0);
    nbv.assign(F, 0);
    bcv.assign(F, 0);
    dv.assign(F, 0);
    obj.assign(F, 0);
    mask.push_back(0);
    pin.push_back(0);
    lin.push_back(0);
  }
  if (phib.empty()) phib.push_back(0.0);
  check(h, pmg_b200_set_stencils(h, boundary.data(), rc.data(), row_of.data(), center.data(),
                                 nbv.data(), bcv.data(), dv.data(), obj.data(), mask.data(),
                                 pin.data(), lin.data(), (int)set.bv.phi_b.size(), phib.data()));
}

}  // namespace detail

/// GPU replacement of pmg::build_stencils (stencil.hpp:207-222): same inputs,
/// an identical StencilSet (bit-exact rows; see tests/test_gpu_stencils.py).
template <int Dim>
StencilSet<Dim> build_stencils(const TreeMesh<Dim>& mesh, const LevelSetSpec<Dim>& lsf,
                               const StencilBuildConfig& cfg, int device = 0) {
  pmg_b200_ctx* h = detail::make_context(mesh, device);
  std::vector<pmg_lsf_t> d;
  auto one = [&](const LevelSetSpec<Dim>& s) {
    pmg_lsf_t x{};
    x.shape = (int32_t)s.shape;
    x.cylindrical = s.cylindrical ? 1 : 0;
    for (int k = 0; k < Dim; ++k) {
      x.center[k] = s.center[k];
      x.seg_a[k] = s.seg_a[k];
      x.seg_b[k] = s.seg_b[k];
    }
    x.radius = s.radius;
    x.boundary_value = s.boundary_value;
    x.shift_p = s.shift_p;
    x.shift_q = s.shift_q;
    x.scale = s.scale;
    d.push_back(x);
  };
  one(lsf);
  if (lsf.shape == Shape::composite_min)
    for (const auto& c : lsf.children) one(c);
  pmg_stencil_cfg_t c{cfg.root.eps_tol, cfg.root.max_bracket_iters, cfg.root.d_min,
                      cfg.w_min, cfg.boundary_safety, cfg.thin_rescue ? 1 : 0};
  try {
    detail::check(h, pmg_b200_build_stencils(h, d.data(), (int)d.size(), &c));
    const int nb = mesh.n_blocks();
    std::vector<int32_t> boundary(nb), rc(nb);
    const int R = pmg_b200_stencil_summary(h, boundary.data(), rc.data());
    if (R < 0) detail::check(h, -R);
    constexpr int F = 2 * Dim;
    size_t ni = 1;
    for (int k = 0; k < Dim; ++k) ni *= (size_t)mesh.block_size();
    const size_t R1 = R > 0 ? (size_t)R : 1;
    std::vector<int32_t> row_of((size_t)nb * ni), lin(R1);
    std::vector<double> center(R1), nbv(R1 * F), bcv(R1 * F), dv(R1 * F);
    std::vector<int8_t> obj(R1 * F), pin(R1);
    std::vector<uint8_t> mask(R1);
    detail::check(h, pmg_b200_get_stencils(h, row_of.data(), center.data(), nbv.data(), bcv.data(),
                                           dv.data(), obj.data(), mask.data(), pin.data(),
                                           lin.data()));
    StencilSet<Dim> set;
    set.by_block.resize((size_t)nb);
    set.bv.phi_b.resize((size_t)lsf.n_objects());
    for (int i = 0; i < lsf.n_objects(); ++i) set.bv.phi_b[(size_t)i] = lsf.object(i).boundary_value;
    size_t r = 0;
    for (int id = 0; id < nb; ++id) {
      BlockStencil<Dim>& st = set.by_block[(size_t)id];
      st.dx = mesh.block(id).dx;
      st.boundary = boundary[id] != 0;
      if (!st.boundary) continue;
      st.row_of.assign(row_of.begin() + (long)id * (long)ni, row_of.begin() + (long)(id + 1) * (long)ni);
      for (int q = 0; q < rc[id]; ++q, ++r) {
        StencilCell<Dim> cell;
        cell.center = center[r];
        for (int f = 0; f < F; ++f) {
          cell.nb[f] = nbv[r * F + f];
          cell.bc[f] = bcv[r * F + f];
          cell.d[f] = dv[r * F + f];
          cell.obj[f] = obj[r * F + f];
        }
        cell.mask = mask[r];
        cell.pin_obj = pin[r];
        cell.lin = lin[r];
        st.rows.push_back(cell);
      }
    }
    pmg_b200_destroy(h);
    return set;
  } catch (...) {
    pmg_b200_destroy(h);
    throw;
  }
}

template <int Dim>
class MgSolver {
 public:
  MgSolver(TreeMesh<Dim>& mesh, StencilSet<Dim>& stencils, const MgConfig& cfg, int device = 0)
      : mesh_(mesh), set_(stencils), cfg_(cfg), pool_(cfg.threads) {
    cfg_.validate();
    h_ = detail::make_context(mesh_, device);
    try {
      detail::upload_stencils(h_, mesh_, set_);
      upload(VAR_RHS);
      upload(VAR_PHI);
      pmg_mg_cfg_t c{cfg_.n_down, cfg_.n_up, cfg_.coarse_rel_tol, cfg_.coarse_max_iters,
                     cfg_.threads};
      detail::check(h_, pmg_b200_solver_create(h_, &c));  // includes init()
      if (sync_) sync_to_host();
    } catch (...) {
      pmg_b200_destroy(h_);
      throw;
    }
  }
  ~MgSolver() { pmg_b200_destroy(h_); }
  MgSolver(const MgSolver&) = delete;
  MgSolver& operator=(const MgSolver&) = delete;

  /// init() re-reads PHI, RHS and the boundary values from the host objects.
  void init() {
    upload(VAR_RHS);
    upload(VAR_PHI);
    for (size_t o = 0; o < set_.bv.phi_b.size(); ++o)
      detail::check(h_, pmg_b200_set_boundary_value(h_, (int)o, set_.bv.phi_b[o]));
    detail::check(h_, pmg_b200_init(h_));
    if (sync_) sync_to_host();
  }
  CycleStats run_cycle() { return cfg_.cycle == CycleType::fmg ? fmg_cycle() : v_cycle(); }
  CycleStats v_cycle() { return stats(pmg_b200_v_cycle); }
  CycleStats fmg_cycle() { return stats(pmg_b200_fmg_cycle); }
  CycleStats measure_residual() { return stats(pmg_b200_measure_residual); }
  void gsrb_sweep(int level, int parity) { op(pmg_b200_gsrb_sweep(h_, level, parity)); }
  void restrict_level(int level) { op(pmg_b200_restrict_level(h_, level)); }
  void restrict_level_no_guess(int level) { op(pmg_b200_restrict_level_no_guess(h_, level)); }
  void prolong_correction(int level) { op(pmg_b200_prolong_correction(h_, level)); }
  void prolong_full(int level) { op(pmg_b200_prolong_full(h_, level)); }
  void coarse_solve() { op(pmg_b200_coarse_solve(h_)); }
  void set_have_guess(bool v) { detail::check(h_, pmg_b200_set_have_guess(h_, v ? 1 : 0)); }
  /// The host thread pool (MgSolver::pool, multigrid.hpp:475): the cycles
  /// run on the GPU; host-side helpers a caller runs over the mesh use it.
  ThreadPool& pool() { return pool_; }
  const CoarseSystem& coarse_system() const {
    int32_t n, nnz, no;
    detail::check(h_, pmg_b200_coarse_sizes(h_, &n, &nnz, &no));
    cs_.n = n;
    cs_.rp.assign((size_t)n + 1, 0);
    cs_.ci.assign((size_t)nnz, 0);
    cs_.val.assign((size_t)nnz, 0.0);
    cs_.c0.assign((size_t)n, 0.0);
    std::vector<double> cobj((size_t)no * (size_t)n + 1);
    std::vector<int32_t> ub((size_t)n + 1), ul((size_t)n + 1);
    detail::check(h_, pmg_b200_coarse_get(h_, cs_.rp.data(), cs_.ci.data(), cs_.val.data(),
                                          cs_.c0.data(), cobj.data(), ub.data(), ul.data()));
    cs_.cobj.assign((size_t)no, std::vector<double>((size_t)n));
    for (int o = 0; o < no; ++o)
      std::copy(cobj.begin() + (long)o * n, cobj.begin() + (long)(o + 1) * n, cs_.cobj[(size_t)o].begin());
    cs_.unknown_cell.clear();
    for (int u = 0; u < n; ++u) cs_.unknown_cell.emplace_back(ub[(size_t)u], ul[(size_t)u]);
    return cs_;
  }

  /// pmg::error_norms (fields.hpp:35-69) of PHI against an AnalyticSolution,
  /// evaluated on the device: no copy of PHI to the host.
  ErrorNorms error_norms(const AnalyticSolution& sol, bool volume_weighted = false) const {
    ErrorNorms e;
    const int tag = sol.tag == AnalyticSolution::Case::sphere3d ? 1 : 0;
    detail::check(h_, pmg_b200_error_norms(h_, VAR_PHI, tag, sol.phi_b, sol.a, sol.R, volume_weighted ? 1 : 0,
                                           &e.linf, &e.l2));
    return e;
  }
  /// pmg::face_gradient (fields.hpp:149-232) of PHI on the device; the
  /// cell-centred magnitude goes to mesh.field(id, var_out) of every leaf when
  /// var_out >= 0, as the reference writes it.
  FaceField<Dim> face_gradient(int var_out = -1) {
    const int nl = pmg_b200_n_leaves(h_);
    if (nl < 0) detail::check(h_, -nl);
    const int N = mesh_.block_size();
    size_t ni = 1, per_axis = (size_t)N + 1;
    for (int k = 0; k < Dim; ++k) ni *= (size_t)N;
    for (int k = 1; k < Dim; ++k) per_axis *= (size_t)N;
    std::vector<double> faces((size_t)nl * Dim * per_axis), mag(var_out >= 0 ? (size_t)nl * ni : 1);
    std::vector<int32_t> ids((size_t)nl);
    detail::check(h_, pmg_b200_face_gradient(h_, VAR_PHI, faces.data(), var_out >= 0 ? mag.data() : nullptr,
                                             ids.data()));
    FaceField<Dim> ff;
    ff.block_ids.assign(ids.begin(), ids.end());
    ff.faces.resize((size_t)nl);
    for (int q = 0; q < nl; ++q)
      for (int a = 0; a < Dim; ++a)
        ff.faces[(size_t)q][(size_t)a].assign(faces.begin() + (long)((size_t)q * Dim + a) * (long)per_axis,
                                              faces.begin() + (long)((size_t)q * Dim + a + 1) * (long)per_axis);
    if (var_out >= 0) {
      IVec<Dim> zero{}, nn;
      nn.fill(N);
      for (int q = 0; q < nl; ++q) {
        double* out = mesh_.field(ids[(size_t)q], var_out);
        size_t c = 0;
        for_box<Dim>(zero, nn, [&](const IVec<Dim>& i) { out[mesh_.lin(i)] = mag[(size_t)q * ni + c++]; });
      }
    }
    return ff;
  }
  /// pmg::write_dump (io.hpp:23-71) of PHI streamed from the device.
  void write_dump(const std::string& path, const std::string& field_name) {
    detail::check(h_, pmg_b200_write_dump(h_, VAR_PHI, path.c_str(), field_name.c_str()));
  }

  /// Copy PHI (ghost layers included) from the GPU into mesh.field(id, VAR_PHI).
  /// The copy goes through the context's page-locked buffer and is scattered
  /// into the blocks by the solver's thread pool.
  void sync_to_host() {
    const size_t S = mesh_.var_stride();
    const size_t bytes = (size_t)mesh_.n_blocks() * S * sizeof(double);
    double* buf = static_cast<double*>(pmg_b200_host_buffer(h_, bytes));
    if (!buf) detail::check(h_, PMG_ERR_CUDA);
    detail::check(h_, pmg_b200_download_field(h_, VAR_PHI, buf, PMG_LAYOUT_PADDED));
    parallel_for(&pool_, mesh_.n_blocks(), [&](int id) {
      std::memcpy(mesh_.field(id, VAR_PHI), buf + (size_t)id * S, S * sizeof(double));
    });
  }
  /// Drop-in default true: PHI is copied back after every cycle/operation.
  void set_sync_to_host(bool v) { sync_ = v; }
  pmg_b200_ctx* context() { return h_; }

 private:
  void upload(int var) {
    const size_t S = mesh_.var_stride();
    std::vector<double> buf((size_t)mesh_.n_blocks() * S);
    for (int id = 0; id < mesh_.n_blocks(); ++id)
      std::memcpy(buf.data() + (size_t)id * S, mesh_.field(id, var), S * sizeof(double));
    detail::check(h_, pmg_b200_upload_field(h_, var, buf.data(), PMG_LAYOUT_PADDED));
  }
  void op(int rc) {
    detail::check(h_, rc);
    if (sync_) sync_to_host();
  }
  CycleStats stats(int (*fn)(pmg_b200_ctx*, pmg_cycle_stats_t*)) {
    pmg_cycle_stats_t s{};
    detail::check(h_, fn(h_, &s));
    if (sync_) sync_to_host();
    CycleStats out;
    out.max_resid = s.max_resid;
    out.l2_resid = s.l2_resid;
    return out;
  }

  TreeMesh<Dim>& mesh_;
  StencilSet<Dim>& set_;
  MgConfig cfg_;
  ThreadPool pool_;
  pmg_b200_ctx* h_ = nullptr;
  bool sync_ = true;
  mutable CoarseSystem cs_;
};

}  // namespace b200
}  // namespace pmg

#endif  // PMG_B200_SOLVER_HPP
