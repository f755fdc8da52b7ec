// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/oc_api.h).
//
// Thin C shim that drives the UNMODIFIED reference implementation
// (/root/reference/proj/include/pmg/*.hpp, header-only C++20) through its own
// public API so that tests and the CPU baseline can call it via ctypes.  No
// reference source is copied here: the headers are #included read-only from
// the reference tree by oracle/Makefile and the result goes to oracle/_ref/.
//
// Forwarding map (reference file:line):
//   oc_build_uniform       -> pmg::build_uniform            mesh.hpp:565-572
//   oc_refine_band         -> pmg::detail::refine_by_criterion harness.hpp:295-321
//   oc_refine_crit         -> the same with build_case's criteria  harness.hpp:351-355, 413-418
//   oc_adapt               -> TreeMesh::adapt                mesh.hpp:157-204
//   oc_fill_ghosts         -> TreeMesh::fill_ghosts          mesh.hpp:217-221
//   oc_build_stencils      -> pmg::build_stencils            stencil.hpp:207-222
//   oc_apply_pins          -> pmg::apply_pins                stencil.hpp:225-237
//   oc_residual_level      -> pmg::residual_block per block  stencil.hpp:325-359
//   oc_solver_create/...   -> pmg::MgSolver<D>               multigrid.hpp:292-792
//   oc_coarse_*            -> MgSolver::coarse_system        multigrid.hpp:474
//   oc_face_gradient       -> pmg::face_gradient             fields.hpp:149-232
//   oc_error_norms         -> pmg::error_norms               fields.hpp:35-69
#include <limits>  // levelset.hpp uses numeric_limits without including it
#include <memory>
#include <string>
#include <vector>

#include "pmg/harness.hpp"
#include "oc_api.h"

namespace {

using namespace pmg;

struct Base {
  virtual ~Base() = default;
  std::string err;
  virtual int build_uniform(int levels) = 0;
  virtual int refine_band(const pmg_lsf_t* l, int n, double band, int max_level) = 0;
  virtual int refine_crit(int kind, double p0, double p1, const double* centre, int max_level) = 0;
  virtual int adapt(const uint8_t* flags, int n, int max_level) = 0;
  virtual int n_blocks() = 0;
  virtual int n_levels() = 0;
  virtual int topology(int32_t*, int32_t*, double*, double*, int32_t*, int32_t*, int32_t*,
                       int32_t*) = 0;
  virtual int level_blocks(int level, int32_t* ids) = 0;
  virtual int set_face_bc(int dir, int type, double c, const double* g) = 0;
  virtual int set_field(int var, const double* buf) = 0;
  virtual int get_field(int var, double* buf) = 0;
  virtual int build_stencils(const pmg_lsf_t* l, int n, const pmg_stencil_cfg_t* cfg) = 0;
  virtual int summary(int32_t* boundary, int32_t* rc) = 0;
  virtual int get_stencils(int32_t*, double*, double*, double*, double*, int8_t*, uint8_t*,
                           int8_t*, int32_t*) = 0;
  virtual int set_stencils(const int32_t*, const int32_t*, const int32_t*, const double*,
                           const double*, const double*, const double*, const int8_t*,
                           const uint8_t*, const int8_t*, const int32_t*, int,
                           const double*) = 0;
  virtual int set_bv(int obj, double v) = 0;
  virtual int solver_create(const pmg_mg_cfg_t* cfg) = 0;
  virtual int op(int which, int a, int b, pmg_cycle_stats_t* out) = 0;
  virtual int coarse_sizes(int32_t*, int32_t*, int32_t*) = 0;
  virtual int coarse_get(int32_t*, int32_t*, double*, double*, double*, int32_t*, int32_t*) = 0;
  virtual int probe(int32_t*, int32_t*, double*) = 0;
  virtual int face_grad(int var, int var_out, double* faces, int32_t* ids) = 0;
  virtual int err_norms(int var, int tag, double phi_b, double a, double R, int vw, double* out) = 0;
};

enum Op {
  OP_INIT, OP_V, OP_FMG, OP_MEASURE, OP_GSRB, OP_FILL, OP_PINS, OP_RESID, OP_RESTRICT,
  OP_RESTRICT_NG, OP_PROLONG, OP_PROLONG_FULL, OP_COARSE, OP_HAVE_GUESS
};

template <int D>
LevelSetSpec<D> to_spec1(const pmg_lsf_t& s) {
  LevelSetSpec<D> r;
  r.shape = static_cast<Shape>(s.shape);
  for (int k = 0; k < D; ++k) {
    r.center[k] = s.center[k];
    r.seg_a[k] = s.seg_a[k];
    r.seg_b[k] = s.seg_b[k];
  }
  r.radius = s.radius;
  r.boundary_value = s.boundary_value;
  r.shift_p = s.shift_p;
  r.shift_q = s.shift_q;
  r.scale = s.scale;
  r.cylindrical = s.cylindrical != 0;
  return r;
}

template <int D>
LevelSetSpec<D> to_spec(const pmg_lsf_t* l, int n) {
  LevelSetSpec<D> r = to_spec1<D>(l[0]);
  if (r.shape == Shape::composite_min)
    for (int i = 1; i < n; ++i) r.children.push_back(to_spec1<D>(l[i]));
  return r;
}

template <int D>
struct Impl final : Base {
  static constexpr int F = 2 * D;
  TreeMesh<D> mesh;
  StencilSet<D> set;
  std::unique_ptr<MgSolver<D>> solver;
  int N;

  Impl(int n, const double* lo, const double* hi) : mesh(vec(lo), vec(hi), n), N(n) {}

  static Vec<D> vec(const double* p) {
    Vec<D> v;
    for (int k = 0; k < D; ++k) v[k] = p[k];
    return v;
  }
  size_t n_int() const {
    size_t s = 1;
    for (int k = 0; k < D; ++k) s *= static_cast<size_t>(N);
    return s;
  }

  int build_uniform(int levels) override {
    Vec<D> lo = mesh.domain_lo(), hi = mesh.domain_hi();
    auto bc = mesh.face_bc;
    mesh = pmg::build_uniform<D>(lo, hi, N, levels);
    mesh.face_bc = bc;
    solver.reset();
    return 0;
  }
  int refine_band(const pmg_lsf_t* l, int n, double band, int max_level) override {
    LevelSetSpec<D> s = to_spec<D>(l, n);
    detail::refine_by_criterion<D>(mesh, max_level,
                                   [&](const Block<D>& b, const Vec<D>& x) {
                                     return std::abs(lsf_eval(s, x)) < band * b.dx;
                                   });
    solver.reset();
    return 0;
  }
  int refine_crit(int kind, double p0, double p1, const double* centre, int max_level) override {
    Vec<D> c;
    for (int k = 0; k < D; ++k) c[k] = centre[k];
    if (kind == 1)
      detail::refine_by_criterion<D>(mesh, max_level, [=](const Block<D>& b, const Vec<D>& x) {
        return b.dx > p0 * std::max(1.0, norm(x - c) / p1);
      });
    else
      detail::refine_by_criterion<D>(mesh, max_level, [=](const Block<D>& b, const Vec<D>& x) {
        return b.dx > p0 && norm(x - c) < p1;
      });
    solver.reset();
    return 0;
  }
  int adapt(const uint8_t* flags, int n, int max_level) override {
    std::vector<RefineFlag> f(static_cast<size_t>(mesh.n_blocks()), RefineFlag::keep);
    for (int id = 0; id < mesh.n_blocks() && id < n; ++id)
      if (flags[id] == 1) f[static_cast<size_t>(id)] = RefineFlag::refine;
    mesh.adapt(f, max_level);
    solver.reset();
    return 0;
  }
  int n_blocks() override { return mesh.n_blocks(); }
  int n_levels() override { return mesh.n_levels(); }
  int topology(int32_t* level, int32_t* coords, double* origin, double* dx, int32_t* parent,
               int32_t* children, int32_t* nbr, int32_t* cnbr) override {
    for (int id = 0; id < mesh.n_blocks(); ++id) {
      const Block<D>& b = mesh.block(id);
      level[id] = b.level;
      dx[id] = b.dx;
      parent[id] = b.parent;
      for (int k = 0; k < 3; ++k) {
        coords[3 * id + k] = k < D ? b.coords[k] : 0;
        origin[3 * id + k] = k < D ? b.origin[k] : 0.0;
      }
      for (int c = 0; c < 8; ++c) children[8 * id + c] = c < (1 << D) ? b.children[c] : -1;
      for (int f = 0; f < 6; ++f) {
        nbr[6 * id + f] = f < F ? b.nbr[f] : -1;
        cnbr[6 * id + f] = f < F ? b.coarse_nbr[f] : -1;
      }
    }
    return 0;
  }
  int level_blocks(int level, int32_t* ids) override {
    if (level < 1 || level > mesh.n_levels()) return 0;
    const auto& v = mesh.level_blocks(level);
    for (size_t i = 0; i < v.size(); ++i) ids[i] = v[i];
    return static_cast<int>(v.size());
  }
  int set_face_bc(int dir, int type, double c, const double* g) override {
    FaceBc<D> fb;
    fb.type = type == PMG_BC_NEUMANN_ZERO ? FaceBcType::neumann_zero : FaceBcType::dirichlet;
    std::array<double, D> gg{};
    for (int k = 0; k < D; ++k) gg[k] = g ? g[k] : 0.0;
    bool nonzero = c != 0.0;
    for (int k = 0; k < D; ++k) nonzero = nonzero || gg[k] != 0.0;
    if (nonzero)
      fb.value = [c, gg](const Vec<D>& x) {
        double v = c;
        for (int k = 0; k < D; ++k) v += gg[k] * x[k];
        return v;
      };
    mesh.face_bc[static_cast<size_t>(dir)] = fb;
    return 0;
  }
  int set_field(int var, const double* buf) override {
    const size_t s = mesh.var_stride();
    for (int id = 0; id < mesh.n_blocks(); ++id)
      std::copy(buf + id * s, buf + (id + 1) * s, mesh.field(id, var));
    return 0;
  }
  int get_field(int var, double* buf) override {
    const size_t s = mesh.var_stride();
    for (int id = 0; id < mesh.n_blocks(); ++id)
      std::copy(mesh.field(id, var), mesh.field(id, var) + s, buf + id * s);
    return 0;
  }
  int build_stencils(const pmg_lsf_t* l, int n, const pmg_stencil_cfg_t* c) override {
    StencilBuildConfig sc;
    sc.root.eps_tol = c->eps_tol;
    sc.root.max_bracket_iters = c->max_bracket_iters;
    sc.root.d_min = c->d_min;
    sc.w_min = c->w_min;
    sc.boundary_safety = c->boundary_safety;
    sc.thin_rescue = c->thin_rescue != 0;
    // the reference's own block-parallel pool; results are thread-count independent
    ThreadPool pool(static_cast<int>(std::max(1u, std::thread::hardware_concurrency())));
    set = pmg::build_stencils<D>(mesh, to_spec<D>(l, n), sc, &pool);
    solver.reset();
    return 0;
  }
  int summary(int32_t* boundary, int32_t* rc) override {
    int tot = 0;
    for (int id = 0; id < mesh.n_blocks(); ++id) {
      const auto& st = set.by_block[static_cast<size_t>(id)];
      if (boundary) boundary[id] = st.boundary ? 1 : 0;
      if (rc) rc[id] = static_cast<int32_t>(st.rows.size());
      tot += static_cast<int>(st.rows.size());
    }
    return tot;
  }
  int get_stencils(int32_t* row_of, double* center, double* nb, double* bc, double* d,
                   int8_t* obj, uint8_t* mask, int8_t* pin, int32_t* lin) override {
    size_t r = 0;
    const size_t ni = n_int();
    for (int id = 0; id < mesh.n_blocks(); ++id) {
      const auto& st = set.by_block[static_cast<size_t>(id)];
      for (size_t c = 0; c < ni; ++c)
        row_of[id * ni + c] = st.boundary ? st.row_of[c] : -1;
      for (const auto& cell : st.rows) {
        center[r] = cell.center;
        for (int f = 0; f < F; ++f) {
          nb[r * F + f] = cell.nb[f];
          bc[r * F + f] = cell.bc[f];
          d[r * F + f] = cell.d[f];
          obj[r * F + f] = cell.obj[f];
        }
        mask[r] = cell.mask;
        pin[r] = cell.pin_obj;
        lin[r] = cell.lin;
        ++r;
      }
    }
    return 0;
  }
  int set_stencils(const int32_t* boundary, const int32_t* rc, const int32_t* row_of,
                   const double* center, const double* nb, const double* bc, const double* d,
                   const int8_t* obj, const uint8_t* mask, const int8_t* pin,
                   const int32_t* lin, int n_obj, const double* phi_b) override {
    set = StencilSet<D>{};
    set.by_block.resize(static_cast<size_t>(mesh.n_blocks()));
    set.bv.phi_b.assign(phi_b, phi_b + n_obj);
    size_t r = 0;
    const size_t ni = n_int();
    for (int id = 0; id < mesh.n_blocks(); ++id) {
      auto& st = set.by_block[static_cast<size_t>(id)];
      st.dx = mesh.block(id).dx;
      st.boundary = boundary[id] != 0;
      if (st.boundary) st.row_of.assign(row_of + id * ni, row_of + (id + 1) * ni);
      for (int k = 0; k < rc[id]; ++k, ++r) {
        StencilCell<D> cell;
        cell.center = center[r];
        for (int f = 0; f < F; ++f) {
          cell.nb[f] = nb[r * F + f];
          cell.bc[f] = bc[r * F + f];
          cell.d[f] = d[r * F + f];
          cell.obj[f] = obj[r * F + f];
        }
        cell.mask = mask[r];
        cell.pin_obj = pin[r];
        cell.lin = lin[r];
        st.rows.push_back(cell);
      }
    }
    solver.reset();
    return 0;
  }
  int set_bv(int obj, double v) override {
    set.set_boundary_value(obj, v);
    return 0;
  }
  int solver_create(const pmg_mg_cfg_t* c) override {
    MgConfig mg;
    mg.n_down = c->n_down;
    mg.n_up = c->n_up;
    mg.coarse_rel_tol = c->coarse_rel_tol;
    mg.coarse_max_iters = c->coarse_max_iters;
    mg.threads = c->threads;
    tol = c->coarse_rel_tol;
    max_iters = c->coarse_max_iters;
    solver.reset();
    solver = std::make_unique<MgSolver<D>>(mesh, set, mg);
    return 0;
  }
  int op(int which, int a, int b, pmg_cycle_stats_t* out) override {
    CycleStats s;
    if (!solver && which != OP_FILL && which != OP_PINS && which != OP_RESID) {
      err = "solver not created";
      return PMG_ERR_STATE;
    }
    switch (which) {
      case OP_INIT: solver->init(); break;
      case OP_V: s = solver->v_cycle(); break;
      case OP_FMG: s = solver->fmg_cycle(); break;
      case OP_MEASURE: s = solver->measure_residual(); break;
      case OP_GSRB: solver->gsrb_sweep(a, b); break;
      case OP_FILL: mesh.fill_ghosts(a, b); break;
      case OP_PINS: apply_pins(mesh, set, a); break;
      case OP_RESID:
        for (int id : mesh.level_blocks(a))
          residual_block(mesh, id, set.by_block[static_cast<size_t>(id)], set.bv, VAR_PHI,
                         VAR_RHS, VAR_RES);
        break;
      case OP_RESTRICT: solver->restrict_level(a); break;
      case OP_RESTRICT_NG: solver->restrict_level_no_guess(a); break;
      case OP_PROLONG: solver->prolong_correction(a); break;
      case OP_PROLONG_FULL: solver->prolong_full(a); break;
      case OP_COARSE: solver->coarse_solve(); break;
      case OP_HAVE_GUESS: solver->set_have_guess(a != 0); break;
      default: err = "bad op"; return PMG_ERR_INVALID_ARG;
    }
    if (out) {
      out->max_resid = s.max_resid;
      out->l2_resid = s.l2_resid;
    }
    return 0;
  }
  int coarse_sizes(int32_t* n, int32_t* nnz, int32_t* nobj) override {
    if (!solver) return PMG_ERR_STATE;
    const CoarseSystem& cs = solver->coarse_system();
    *n = cs.n;
    *nnz = static_cast<int32_t>(cs.val.size());
    *nobj = static_cast<int32_t>(cs.cobj.size());
    return 0;
  }
  int coarse_get(int32_t* rp, int32_t* ci, double* val, double* c0, double* cobj,
                 int32_t* ub, int32_t* ul) override {
    if (!solver) return PMG_ERR_STATE;
    const CoarseSystem& cs = solver->coarse_system();
    std::copy(cs.rp.begin(), cs.rp.end(), rp);
    std::copy(cs.ci.begin(), cs.ci.end(), ci);
    std::copy(cs.val.begin(), cs.val.end(), val);
    std::copy(cs.c0.begin(), cs.c0.end(), c0);
    for (size_t o = 0; o < cs.cobj.size(); ++o)
      std::copy(cs.cobj[o].begin(), cs.cobj[o].end(), cobj + o * static_cast<size_t>(cs.n));
    for (int u = 0; u < cs.n; ++u) {
      ub[u] = cs.unknown_cell[static_cast<size_t>(u)].first;
      ul[u] = cs.unknown_cell[static_cast<size_t>(u)].second;
    }
    return 0;
  }
  int probe(int32_t* conv, int32_t* iters, double* rel) override {
    if (!solver) return PMG_ERR_STATE;
    const CoarseSystem& cs = solver->coarse_system();
    const size_t n = static_cast<size_t>(cs.n);
    std::vector<double> b(n), x(n);
    for (size_t u = 0; u < n; ++u) {
      const auto& [id, lin] = cs.unknown_cell[u];
      b[u] = mesh.field(id, VAR_RHS)[lin] + cs.c0[u];
      x[u] = mesh.field(id, VAR_PHI)[lin];
    }
    for (size_t o = 0; o < set.bv.phi_b.size(); ++o)
      for (size_t u = 0; u < n; ++u) b[u] += cs.cobj[o][u] * set.bv.phi_b[o];
    auto res = detail::bicgstab(cs, b, x, tol, max_iters);
    *conv = res.converged ? 1 : 0;
    *iters = res.iters;
    *rel = res.rel;
    return 0;
  }  // pmg::error_norms with pmg::AnalyticSolution (fields.hpp:35-69)
  int err_norms(int var, int tag, double phi_b, double a, double R, int vw, double* out) override {
    AnalyticSolution sol;
    sol.tag = tag == 0 ? AnalyticSolution::Case::sphere2d : AnalyticSolution::Case::sphere3d;
    sol.phi_b = phi_b;
    sol.a = a;
    sol.R = R;
    const ErrorNorms e = pmg::error_norms<D>(mesh, set, var, sol, vw != 0);
    out[0] = e.linf;
    out[1] = e.l2;
    return 0;
  }
  // pmg::face_gradient (fields.hpp:149-232): faces flattened per leaf, axis
  int face_grad(int var, int var_out, double* faces, int32_t* ids) override {
    const FaceField<D> ff = pmg::face_gradient<D>(mesh, set, var, var_out);
    size_t k = 0;
    for (size_t b = 0; b < ff.block_ids.size(); ++b) {
      if (ids) ids[b] = ff.block_ids[b];
      for (int a = 0; a < D; ++a)
        for (double v : ff.faces[b][static_cast<size_t>(a)]) {
          if (faces) faces[k] = v;
          ++k;
        }
    }
    return static_cast<int>(ff.block_ids.size());
  }

  double tol = 1e-6;
  int max_iters = 2000;
};

template <typename Fn>
int guard(oc_ctx* h, Fn&& fn);

}  // namespace

struct oc_ctx {
  std::unique_ptr<Base> impl;
  std::string err;
};

namespace {
template <typename Fn>
int guard(oc_ctx* h, Fn&& fn) {
  if (!h || !h->impl) return PMG_ERR_STATE;
  try {
    h->err.clear();
    int rc = fn(*h->impl);
    if (rc != 0 && h->err.empty()) h->err = h->impl->err;
    return rc;
  } catch (const std::logic_error& e) {
    h->err = e.what();
    return PMG_ERR_TOPOLOGY;
  } catch (const std::runtime_error& e) {
    h->err = e.what();
    std::string m = e.what();
    return m.rfind("coarse solve failed", 0) == 0 ? PMG_ERR_COARSE_STALL : PMG_ERR_INVALID_ARG;
  } catch (const std::exception& e) {
    h->err = e.what();
    return PMG_ERR_INVALID_ARG;
  }
}
}  // namespace

extern "C" {

oc_ctx* oc_create(int dim, int N, const double* lo, const double* hi) {
  auto* h = new oc_ctx;
  try {
    if (dim == 2)
      h->impl = std::make_unique<Impl<2>>(N, lo, hi);
    else if (dim == 3)
      h->impl = std::make_unique<Impl<3>>(N, lo, hi);
    else
      throw std::runtime_error("dim must be 2 or 3");
  } catch (const std::exception& e) {
    h->err = e.what();
  }
  return h;
}
void oc_destroy(oc_ctx* h) { delete h; }
const char* oc_last_error(oc_ctx* h) { return h ? h->err.c_str() : "null handle"; }

int oc_build_uniform(oc_ctx* h, int levels) {
  return guard(h, [&](Base& b) { return b.build_uniform(levels); });
}
int oc_refine_band(oc_ctx* h, const pmg_lsf_t* l, int n, double band, int max_level) {
  return guard(h, [&](Base& b) { return b.refine_band(l, n, band, max_level); });
}
int oc_refine_crit(oc_ctx* h, int kind, double p0, double p1, const double* centre, int max_level) {
  return guard(h, [&](Base& b) { return b.refine_crit(kind, p0, p1, centre, max_level); });
}
int oc_adapt(oc_ctx* h, const uint8_t* flags, int n, int max_level) {
  return guard(h, [&](Base& b) { return b.adapt(flags, n, max_level); });
}
int oc_n_blocks(oc_ctx* h) { return h && h->impl ? h->impl->n_blocks() : -1; }
int oc_n_levels(oc_ctx* h) { return h && h->impl ? h->impl->n_levels() : -1; }
int oc_get_topology(oc_ctx* h, int32_t* level, int32_t* coords, double* origin, double* dx,
                    int32_t* parent, int32_t* children, int32_t* nbr, int32_t* cnbr) {
  return guard(h, [&](Base& b) {
    return b.topology(level, coords, origin, dx, parent, children, nbr, cnbr);
  });
}
int oc_level_blocks(oc_ctx* h, int level, int32_t* ids) {
  return h && h->impl ? h->impl->level_blocks(level, ids) : -1;
}
int oc_set_face_bc(oc_ctx* h, int dir, int type, double c, const double* g) {
  return guard(h, [&](Base& b) { return b.set_face_bc(dir, type, c, g); });
}
int oc_set_field(oc_ctx* h, int var, const double* buf) {
  return guard(h, [&](Base& b) { return b.set_field(var, buf); });
}
int oc_get_field(oc_ctx* h, int var, double* buf) {
  return guard(h, [&](Base& b) { return b.get_field(var, buf); });
}
int oc_build_stencils(oc_ctx* h, const pmg_lsf_t* l, int n, const pmg_stencil_cfg_t* cfg) {
  return guard(h, [&](Base& b) { return b.build_stencils(l, n, cfg); });
}
int oc_stencil_summary(oc_ctx* h, int32_t* boundary, int32_t* rc) {
  int tot = -1;
  int st = guard(h, [&](Base& b) {
    tot = b.summary(boundary, rc);
    return 0;
  });
  return st == 0 ? tot : -st;
}
int oc_get_stencils(oc_ctx* h, int32_t* row_of, double* center, double* nb, double* bc,
                    double* d, int8_t* obj, uint8_t* mask, int8_t* pin, int32_t* lin) {
  return guard(h, [&](Base& b) {
    return b.get_stencils(row_of, center, nb, bc, d, obj, mask, pin, lin);
  });
}
int oc_set_stencils(oc_ctx* h, const int32_t* boundary, const int32_t* rc,
                    const int32_t* row_of, const double* center, const double* nb,
                    const double* bc, const double* d, const int8_t* obj, const uint8_t* mask,
                    const int8_t* pin, const int32_t* lin, int n_obj, const double* phi_b) {
  return guard(h, [&](Base& b) {
    return b.set_stencils(boundary, rc, row_of, center, nb, bc, d, obj, mask, pin, lin, n_obj,
                          phi_b);
  });
}
int oc_set_boundary_value(oc_ctx* h, int obj, double v) {
  return guard(h, [&](Base& b) { return b.set_bv(obj, v); });
}
int oc_solver_create(oc_ctx* h, const pmg_mg_cfg_t* cfg) {
  return guard(h, [&](Base& b) { return b.solver_create(cfg); });
}
#define OC_OP(name, code, A, B, OUT) \
  int name { return guard(h, [&](Base& b) { return b.op(code, A, B, OUT); }); }
OC_OP(oc_init(oc_ctx* h), OP_INIT, 0, 0, nullptr)
OC_OP(oc_v_cycle(oc_ctx* h, pmg_cycle_stats_t* out), OP_V, 0, 0, out)
OC_OP(oc_fmg_cycle(oc_ctx* h, pmg_cycle_stats_t* out), OP_FMG, 0, 0, out)
OC_OP(oc_measure_residual(oc_ctx* h, pmg_cycle_stats_t* out), OP_MEASURE, 0, 0, out)
OC_OP(oc_gsrb_sweep(oc_ctx* h, int level, int parity), OP_GSRB, level, parity, nullptr)
OC_OP(oc_fill_ghosts(oc_ctx* h, int level, int var), OP_FILL, level, var, nullptr)
OC_OP(oc_apply_pins(oc_ctx* h, int level), OP_PINS, level, 0, nullptr)
OC_OP(oc_residual_level(oc_ctx* h, int level), OP_RESID, level, 0, nullptr)
OC_OP(oc_restrict_level(oc_ctx* h, int level), OP_RESTRICT, level, 0, nullptr)
OC_OP(oc_restrict_level_no_guess(oc_ctx* h, int level), OP_RESTRICT_NG, level, 0, nullptr)
OC_OP(oc_prolong_correction(oc_ctx* h, int level), OP_PROLONG, level, 0, nullptr)
OC_OP(oc_prolong_full(oc_ctx* h, int level), OP_PROLONG_FULL, level, 0, nullptr)
OC_OP(oc_coarse_solve(oc_ctx* h), OP_COARSE, 0, 0, nullptr)
OC_OP(oc_set_have_guess(oc_ctx* h, int v), OP_HAVE_GUESS, v, 0, nullptr)
#undef OC_OP
int oc_coarse_sizes(oc_ctx* h, int32_t* n, int32_t* nnz, int32_t* nobj) {
  return guard(h, [&](Base& b) { return b.coarse_sizes(n, nnz, nobj); });
}
int oc_coarse_get(oc_ctx* h, int32_t* rp, int32_t* ci, double* val, double* c0, double* cobj,
                  int32_t* ub, int32_t* ul) {
  return guard(h, [&](Base& b) { return b.coarse_get(rp, ci, val, c0, cobj, ub, ul); });
}

int oc_bicgstab_probe(oc_ctx* h, int32_t* conv, int32_t* iters, double* rel) {
  return guard(h, [&](Base& b) { return b.probe(conv, iters, rel); });
}

/* reference build only: pmg::error_norms(AnalyticSolution); out = {linf, l2} */
int oc_error_norms(oc_ctx* h, int var, int tag, double phi_b, double a, double R, int vw, double* out) {
  if (!h || !h->impl) return -1;
  try {
    h->err.clear();
    return h->impl->err_norms(var, tag, phi_b, a, R, vw, out);
  } catch (const std::exception& e) {
    h->err = e.what();
    return -1;
  }
}
/* reference build only: pmg::face_gradient; returns the number of leaves (or < 0) */
int oc_face_gradient(oc_ctx* h, int var, int var_out, double* faces, int32_t* leaf_ids) {
  if (!h || !h->impl) return -1;
  try {
    h->err.clear();
    return h->impl->face_grad(var, var_out, faces, leaf_ids);
  } catch (const std::exception& e) {
    h->err = e.what();
    return -1;
  }
}
}  // extern "C"
