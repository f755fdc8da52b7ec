// pmg_oracle.cpp -- TEST INFRASTRUCTURE ONLY: CPU restatement of the
// reference's V-cycle / FMG hot path (oracle/oc_api.h).  Built to
// oracle/_ref/libpmgport.so.  Loaded only by tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline leg; the product never links it.
//
// A from-scratch, single-threaded restatement of the algorithm of the
// reference C++ implementation (/root/reference/proj/include/pmg/*.hpp), in
// plain flat-array C++.  Each function cites what it restates; arithmetic is
// written in the reference's operation order and the file is compiled with
// -ffp-contract=off, so results are bit-identical to the reference build
// (checked by tests/test_oracle.py against oracle/_ref/libpmgref.so and the
// committed golden fixtures).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "oc_api.h"

namespace {

constexpr int NV = 5;  // PHI RHS RES OLD AUX (mesh.hpp:13-20)
constexpr double INF = std::numeric_limits<double>::infinity();

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void need(bool c, const std::string& m) {
  if (!c) throw Err(PMG_ERR_INVALID_ARG, m);
}

// ------------------------------------------------------------------ level set
// levelset.hpp:80-148
struct Lsf {
  std::vector<pmg_lsf_t> d;  // [0] root, children after for composite
  bool composite() const { return d[0].shape == PMG_SHAPE_COMPOSITE_MIN; }
  int n_obj() const { return composite() ? (int)d.size() - 1 : 1; }
};

double nrm(const double* a, int D) {
  double s = 0;
  for (int k = 0; k < D; ++k) s += a[k] * a[k];
  return std::sqrt(s);
}

double eval1(const pmg_lsf_t& s, const double* x, int D) {
  if (s.shape == PMG_SHAPE_NONE) return 1.0;
  if (s.shape == PMG_SHAPE_SPHERE) {
    double a[3];
    for (int k = 0; k < D; ++k) a[k] = x[k] - s.center[k];
    return nrm(a, D) - s.radius;
  }
  if (s.shape == PMG_SHAPE_ROD) {  // distance to a segment (levelset.hpp:56-70)
    double ab2 = 0, t = 0;
    for (int k = 0; k < D; ++k) {
      ab2 += (s.seg_b[k] - s.seg_a[k]) * (s.seg_b[k] - s.seg_a[k]);
      t += (x[k] - s.seg_a[k]) * (s.seg_b[k] - s.seg_a[k]);
    }
    t = ab2 > 0 ? std::clamp(t / ab2, 0.0, 1.0) : 0.0;
    double d2 = 0;
    for (int k = 0; k < D; ++k) {
      const double p = s.seg_a[k] + t * (s.seg_b[k] - s.seg_a[k]);
      d2 += (x[k] - p) * (x[k] - p);
    }
    return std::sqrt(d2) - s.radius;
  }
  double p, q;
  if (D == 3 && s.cylindrical) {
    p = s.scale * (std::sqrt(x[0] * x[0] + x[1] * x[1]) - s.shift_p);
    q = s.scale * (x[2] - s.shift_q);
  } else {
    p = s.scale * (x[0] - s.shift_p);
    q = s.scale * (x[1] - s.shift_q);
  }
  switch (s.shape) {
    case PMG_SHAPE_SPHEROID: return std::sqrt(8 * p * p + q * q) - 1.0;
    case PMG_SHAPE_RHOMBUS: return 8 * std::abs(p) + std::abs(q) - 1.5;
    case PMG_SHAPE_HEART: {
      const double u = q - std::cbrt(p * p);
      return p * p + u * u - 1.0;
    }
    case PMG_SHAPE_ASTROID: return std::cbrt(p * p) / 0.8 + std::cbrt(q * q) / 1.5 - 0.8;
    default: return 0.0;
  }
}

double lsf(const Lsf& L, const double* x, int D) {
  if (!L.composite()) return eval1(L.d[0], x, D);
  double f = INF;
  for (size_t i = 1; i < L.d.size(); ++i) f = std::min(f, eval1(L.d[i], x, D));
  return f;
}

int attaining(const Lsf& L, const double* x, int D) {
  if (!L.composite()) return 0;
  int best = 0;
  double fb = INF;
  for (size_t i = 1; i < L.d.size(); ++i) {
    const double f = eval1(L.d[i], x, D);
    if (f < fb) {
      fb = f;
      best = (int)i - 1;
    }
  }
  return best;
}

void grad(const Lsf& L, const double* x, double h, int D, double* g) {  // levelset.hpp:151-168
  for (int k = 0; k < D; ++k) {
    double xp[3], xm[3];
    for (int a = 0; a < D; ++a) xp[a] = xm[a] = x[a];
    xp[k] += h;
    xm[k] -= h;
    g[k] = (lsf(L, xp, D) - lsf(L, xm, D)) / (2 * h);
  }
}

bool candidate(const Lsf& L, const double* x, double h, double safety, int D) {  // :277-289
  const double len = safety * std::sqrt((double)D) * h;
  double g[3];
  grad(L, x, h, D, g);
  return std::abs(lsf(L, x, D)) < len * nrm(g, D);
}

void lerp(const double* a, const double* b, double t, double* p, int D) {
  for (int k = 0; k < D; ++k) p[k] = a[k] + (b[k] - a[k]) * t;
}

double bisect(const Lsf& L, const double* a, const double* b, double lo, double hi, double eps,
              int D) {  // levelset.hpp:198-209
  while (hi - lo > eps) {
    const double mid = 0.5 * (lo + hi);
    double p[3];
    lerp(a, b, mid, p, D);
    if (lsf(L, p, D) > 0)
      lo = mid;
    else
      hi = mid;
  }
  return 0.5 * (lo + hi);
}

double root_position(const Lsf& L, const double* a, const double* b, const pmg_stencil_cfg_t& c,
                     int D) {  // levelset.hpp:223-257
  const double fa = lsf(L, a, D);
  if (fa * lsf(L, b, D) <= 0) return bisect(L, a, b, 0.0, 1.0, c.eps_tol, D);
  const double ip = 0.6180339887498949;
  double lo = 0.0, hi = 1.0;
  double t1 = hi - ip * (hi - lo), t2 = lo + ip * (hi - lo);
  double p[3];
  lerp(a, b, t1, p, D);
  double g1 = fa * lsf(L, p, D);
  lerp(a, b, t2, p, D);
  double g2 = fa * lsf(L, p, D);
  if (g1 <= 0) return bisect(L, a, b, 0.0, t1, c.eps_tol, D);
  if (g2 <= 0) return bisect(L, a, b, 0.0, t2, c.eps_tol, D);
  for (int it = 0; it < c.max_bracket_iters && hi - lo > c.eps_tol; ++it) {
    if (g1 <= g2) {
      hi = t2;
      t2 = t1;
      g2 = g1;
      t1 = hi - ip * (hi - lo);
      lerp(a, b, t1, p, D);
      g1 = fa * lsf(L, p, D);
      if (g1 <= 0) return bisect(L, a, b, 0.0, t1, c.eps_tol, D);
    } else {
      lo = t1;
      t1 = t2;
      g1 = g2;
      t2 = lo + ip * (hi - lo);
      lerp(a, b, t2, p, D);
      g2 = fa * lsf(L, p, D);
      if (g2 <= 0) return bisect(L, a, b, 0.0, t2, c.eps_tol, D);
    }
  }
  return -1.0;
}

// ------------------------------------------------------------------ data model
struct Row {  // StencilCell (stencil.hpp:27-49)
  double center = 0;
  double nb[6] = {0, 0, 0, 0, 0, 0}, bc[6] = {0, 0, 0, 0, 0, 0}, d[6] = {1, 1, 1, 1, 1, 1};
  int8_t obj[6] = {-1, -1, -1, -1, -1, -1};
  uint8_t mask = PMG_SOLVED;
  int8_t pin = -1;
  int32_t lin = -1;
};

struct BlockSt {  // BlockStencil (stencil.hpp:57-80)
  bool boundary = false;
  std::vector<int32_t> row_of;
  std::vector<Row> rows;
};

struct Coarse {  // CoarseSystem (multigrid.hpp:41-57)
  int n = 0;
  std::vector<int> rp, ci;
  std::vector<double> val, c0;
  std::vector<std::vector<double>> cobj;
  std::vector<std::pair<int, int>> cell;
};

struct Rec {
  double max = 0, sumsq = 0;
  long count = 0;
};

struct Ctx {
  int D, N, F, S, NI, s1, s2;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  // blocks
  std::vector<int> lvl, par;
  std::vector<std::array<int, 3>> crd;
  std::vector<std::array<double, 3>> org;
  std::vector<double> bdx;
  std::vector<std::array<int, 8>> kids;
  std::vector<std::array<int, 6>> nb, cnb;
  std::vector<std::vector<int>> levels;
  std::vector<std::map<std::array<int, 3>, int>> maps;
  std::vector<double> data;
  // boundary conditions: type, affine value c + g.x
  int bct[6] = {0, 0, 0, 0, 0, 0};
  double bcc[6] = {0, 0, 0, 0, 0, 0}, bcg[6][3] = {};
  // stencils
  std::vector<BlockSt> st;
  std::vector<double> phib;
  // solver
  bool have_solver = false, have_guess = false;
  pmg_mg_cfg_t cfg{2, 2, 1e-6, 2000, 1};
  Coarse cs;
  std::vector<Rec> recs;
  std::string err;

  int nblocks() const { return (int)lvl.size(); }
  int nlevels() const { return (int)levels.size() - 1; }
  double* f(int id, int var) { return data.data() + ((size_t)id * NV + var) * S; }
  int lin(int i, int j, int k) const { return (i + 1) + (j + 1) * s1 + (D == 3 ? (k + 1) * s2 : 0); }
  void center(int id, int i, int j, int k, double* x) const {  // mesh.hpp:139-143
    const int ii[3] = {i, j, k};
    for (int a = 0; a < D; ++a) x[a] = org[id][a] + (ii[a] + 0.5) * bdx[id];
  }
  double bcval(int dir, const double* x) const {
    double v = bcc[dir];
    for (int k = 0; k < D; ++k) v += bcg[dir][k] * x[k];
    return v;
  }
  bool bc_null(int dir) const {
    bool z = bcc[dir] == 0.0;
    for (int k = 0; k < D; ++k) z = z && bcg[dir][k] == 0.0;
    return z;
  }
  // interior iteration in for_box order (core.hpp:85-97)
  template <class Fn>
  void each(Fn&& fn) const {
    for (int k = 0; k < (D == 3 ? N : 1); ++k)
      for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i) fn(i, j, k, i + N * (j + N * k));
  }
  const Row* row(int id, int ii) const {
    const BlockSt& b = st[(size_t)id];
    if (!b.boundary) return nullptr;
    const int r = b.row_of[(size_t)ii];
    return r < 0 ? nullptr : &b.rows[(size_t)r];
  }
  bool inside(int id, int ii) const {
    const Row* r = row(id, ii);
    return r && r->mask == PMG_INSIDE;
  }
};

// ------------------------------------------------------------------ mesh (mesh.hpp)
void new_block(Ctx& c, int level, std::array<int, 3> co, std::array<double, 3> o, double dx,
               int parent) {
  c.lvl.push_back(level);
  c.crd.push_back(co);
  c.org.push_back(o);
  c.bdx.push_back(dx);
  c.par.push_back(parent);
  std::array<int, 8> k;
  k.fill(-1);
  c.kids.push_back(k);
  std::array<int, 6> n6;
  n6.fill(-1);
  c.nb.push_back(n6);
  c.cnb.push_back(n6);
  c.data.resize((size_t)c.nblocks() * NV * c.S, 0.0);
  if ((int)c.maps.size() <= level) c.maps.resize((size_t)level + 1);
  c.maps[(size_t)level][co] = c.nblocks() - 1;
}

int find(const Ctx& c, int level, const std::array<int, 3>& co) {
  if (level < 1 || level >= (int)c.maps.size()) return -1;
  auto it = c.maps[(size_t)level].find(co);
  return it == c.maps[(size_t)level].end() ? -1 : it->second;
}

bool inb(const Ctx& c, int level, const std::array<int, 3>& co) {
  const int n = 1 << (level - 1);
  for (int k = 0; k < c.D; ++k)
    if (co[(size_t)k] < 0 || co[(size_t)k] >= n) return false;
  return true;
}

void topology(Ctx& c) {  // rebuild_topology (mesh.hpp:429-469)
  int L = 1;
  for (int l : c.lvl) L = std::max(L, l);
  c.levels.assign((size_t)L + 1, {});
  c.maps.assign((size_t)L + 1, {});
  for (int id = 0; id < c.nblocks(); ++id) {
    c.levels[(size_t)c.lvl[(size_t)id]].push_back(id);
    c.maps[(size_t)c.lvl[(size_t)id]][c.crd[(size_t)id]] = id;
  }
  for (auto& v : c.levels)
    std::sort(v.begin(), v.end(), [&](int a, int b) {
      for (int k = 0; k < c.D; ++k)
        if (c.crd[(size_t)a][(size_t)k] != c.crd[(size_t)b][(size_t)k])
          return c.crd[(size_t)a][(size_t)k] < c.crd[(size_t)b][(size_t)k];
      return false;
    });
  for (int id = 0; id < c.nblocks(); ++id)
    for (int dir = 0; dir < c.F; ++dir) {
      auto nc = c.crd[(size_t)id];
      nc[(size_t)(dir / 2)] += (dir & 1) ? 1 : -1;
      c.nb[(size_t)id][(size_t)dir] = -1;
      c.cnb[(size_t)id][(size_t)dir] = -1;
      if (!inb(c, c.lvl[(size_t)id], nc)) continue;
      const int n = find(c, c.lvl[(size_t)id], nc);
      if (n >= 0) {
        c.nb[(size_t)id][(size_t)dir] = n;
      } else {
        std::array<int, 3> pc = {nc[0] >> 1, nc[1] >> 1, nc[2] >> 1};
        const int p = find(c, c.lvl[(size_t)id] - 1, pc);
        if (p < 0) throw Err(PMG_ERR_TOPOLOGY, "ghost region has no covering block");
        c.cnb[(size_t)id][(size_t)dir] = p;
      }
    }
}

void refine_one(Ctx& c, int id) {  // do_refine (mesh.hpp:292-320), fields left zero
  const int nc = 1 << c.D;
  for (int ch = 0; ch < nc; ++ch) {
    std::array<int, 3> co = {0, 0, 0};
    std::array<double, 3> o = {0, 0, 0};
    for (int k = 0; k < c.D; ++k) {
      const int bit = (ch >> k) & 1;
      co[(size_t)k] = 2 * c.crd[(size_t)id][(size_t)k] + bit;
      o[(size_t)k] = c.org[(size_t)id][(size_t)k] + bit * (0.5 * c.N * c.bdx[(size_t)id]);
    }
    new_block(c, c.lvl[(size_t)id] + 1, co, o, 0.5 * c.bdx[(size_t)id], id);
    c.kids[(size_t)id][(size_t)ch] = c.nblocks() - 1;
  }
}

bool leaf(const Ctx& c, int id) { return c.kids[(size_t)id][0] < 0; }

void refine_balanced(Ctx& c, int id, int max_level) {  // mesh.hpp:252-278
  if (!leaf(c, id)) return;
  const int level = c.lvl[(size_t)id];
  if (level >= max_level)
    throw Err(PMG_ERR_INVALID_ARG, "2:1 balancing forced refinement beyond the maximum level");
  const int D = c.D;
  const int total = D == 3 ? 27 : 9;
  for (int q = 0; q < total; ++q) {  // offsets with axis 0 outermost
    int off[3] = {0, 0, 0};
    int r = q;
    for (int k = D - 1; k >= 0; --k) {
      off[k] = r % 3 - 1;
      r /= 3;
    }
    if (off[0] == 0 && off[1] == 0 && off[2] == 0) continue;
    auto nc = c.crd[(size_t)id];
    for (int k = 0; k < D; ++k) nc[(size_t)k] += off[k];
    if (!inb(c, level, nc) || find(c, level, nc) >= 0) continue;
    std::array<int, 3> pc = {nc[0] >> 1, nc[1] >> 1, nc[2] >> 1};
    const int p = find(c, level - 1, pc);
    if (p >= 0 && leaf(c, p)) refine_balanced(c, p, max_level);
  }
  refine_one(c, id);
}

void adapt_refine(Ctx& c, std::vector<int> ids, int max_level) {  // mesh.hpp:157-175,198
  std::vector<int> todo;
  for (int id : ids)
    if (leaf(c, id)) {
      if (c.lvl[(size_t)id] >= max_level)
        throw Err(PMG_ERR_INVALID_ARG, "refinement beyond the configured maximum level");
      todo.push_back(id);
    }
  std::sort(todo.begin(), todo.end(), [&](int a, int b) {
    if (c.lvl[(size_t)a] != c.lvl[(size_t)b]) return c.lvl[(size_t)a] < c.lvl[(size_t)b];
    return a < b;
  });
  for (int id : todo) refine_balanced(c, id, max_level);
  topology(c);
}

// ------------------------------------------------------------------ ghosts (mesh.hpp:471-554)
void fill_block(Ctx& c, int id, int var) {
  const int N = c.N, D = c.D;
  double* f = c.f(id, var);
  for (int dir = 0; dir < c.F; ++dir) {
    const int ax = dir / 2, side = dir & 1;
    const int gpos = side ? N : -1, ip1 = side ? N - 1 : 0, ip2 = side ? N - 2 : 1;
    const int n = c.nb[(size_t)id][(size_t)dir], cb = c.cnb[(size_t)id][(size_t)dir];
    const int T1 = N, T2 = D == 3 ? N : 1;
    for (int u = 0; u < T1 * T2; ++u) {
      int t[3] = {0, 0, 0};
      int free1 = ax == 0 ? 1 : 0, free2 = ax == 2 ? 1 : 2;
      t[free1] = u % N;
      if (D == 3) t[free2] = u / N;
      int g[3] = {t[0], t[1], t[2]}, a1[3] = {t[0], t[1], t[2]}, a2[3] = {t[0], t[1], t[2]};
      g[ax] = gpos;
      a1[ax] = ip1;
      a2[ax] = ip2;
      const int gl = c.lin(g[0], g[1], g[2]);
      if (n >= 0) {  // same-level copy
        int s[3] = {t[0], t[1], t[2]};
        s[ax] = side ? 0 : N - 1;
        f[gl] = c.f(n, var)[c.lin(s[0], s[1], s[2])];
      } else if (cb >= 0) {  // coarse-fine flux-matching interpolation
        const double* cf = c.f(cb, var);
        int lc[3] = {0, 0, 0}, sg[3] = {0, 0, 0};
        for (int k = 0; k < D; ++k) {
          if (k == ax) {
            lc[k] = side ? 0 : N - 1;
          } else {
            const int gk = c.crd[(size_t)id][(size_t)k] * N + t[k];
            lc[k] = (gk >> 1) - c.crd[(size_t)cb][(size_t)k] * N;
            sg[k] = (gk & 1) ? 1 : -1;
          }
        }
        double v = cf[c.lin(lc[0], lc[1], lc[2])];
        for (int k = 0; k < D; ++k) {
          if (k == ax) continue;
          int up[3] = {lc[0], lc[1], lc[2]}, dn[3] = {lc[0], lc[1], lc[2]};
          up[k] += 1;
          dn[k] -= 1;
          v += sg[k] * (cf[c.lin(up[0], up[1], up[2])] - cf[c.lin(dn[0], dn[1], dn[2])]) / 8.0;
        }
        f[gl] = 0.5 * v + 0.75 * f[c.lin(a1[0], a1[1], a1[2])] - 0.25 * f[c.lin(a2[0], a2[1], a2[2])];
      } else if (c.bct[dir] == PMG_BC_NEUMANN_ZERO) {
        f[gl] = f[c.lin(a1[0], a1[1], a1[2])];
      } else {
        double x[3];
        c.center(id, a1[0], a1[1], a1[2], x);
        x[ax] += 0.5 * c.bdx[(size_t)id] * (side ? 1 : -1);
        const double bv = c.bc_null(dir) ? 0.0 : c.bcval(dir, x);
        f[gl] = 2.0 * bv - f[c.lin(a1[0], a1[1], a1[2])];
      }
    }
  }
}

void fill(Ctx& c, int level, int var) {
  for (int id : c.levels[(size_t)level]) fill_block(c, id, var);
}

// ------------------------------------------------------------------ stencils (stencil.hpp)
void build_stencils(Ctx& c, const Lsf& L, const pmg_stencil_cfg_t& cfg) {  // :125-222
  const int D = c.D, N = c.N;
  c.st.assign((size_t)c.nblocks(), BlockSt{});
  c.phib.assign((size_t)L.n_obj(), 0.0);
  for (int o = 0; o < L.n_obj(); ++o)
    c.phib[(size_t)o] = L.composite() ? L.d[(size_t)o + 1].boundary_value : L.d[0].boundary_value;
  for (int id = 0; id < c.nblocks(); ++id) {
    BlockSt& b = c.st[(size_t)id];
    const double h = c.bdx[(size_t)id];
    std::vector<double> fc((size_t)c.NI);
    bool any = false;
    c.each([&](int i, int j, int k, int ii) {
      double x[3];
      c.center(id, i, j, k, x);
      fc[(size_t)ii] = lsf(L, x, D);
      if (fc[(size_t)ii] <= 0) any = true;
    });
    if (!any) {
      for (int k = -1; k <= (D == 3 ? N : -1) && !any; ++k)
        for (int j = -1; j <= N && !any; ++j)
          for (int i = -1; i <= N && !any; ++i) {
            double x[3];
            c.center(id, i, j, D == 3 ? k : 0, x);
            if (candidate(L, x, h, cfg.boundary_safety, D)) any = true;
          }
    }
    if (!any) continue;
    b.boundary = true;
    b.row_of.assign((size_t)c.NI, -1);
    c.each([&](int i, int j, int k, int ii) {
      double x[3];
      c.center(id, i, j, k, x);
      if (fc[(size_t)ii] <= 0) {
        Row r;
        r.mask = PMG_INSIDE;
        r.pin = (int8_t)attaining(L, x, D);
        r.center = 1.0;
        r.lin = c.lin(i, j, k);
        b.row_of[(size_t)ii] = (int)b.rows.size();
        b.rows.push_back(r);
        return;
      }
      if (!candidate(L, x, h, cfg.boundary_safety, D)) return;
      double dd[6] = {1, 1, 1, 1, 1, 1};
      int8_t ob[6] = {-1, -1, -1, -1, -1, -1};
      bool cut = false;
      for (int dir = 0; dir < 2 * D; ++dir) {  // cell_distances (levelset.hpp:313-327)
        double nb[3] = {x[0], x[1], x[2]};
        nb[dir / 2] += ((dir & 1) ? 1 : -1) * h;
        const double t = root_position(L, x, nb, cfg, D);
        if (t < 0) continue;
        const double dv = std::clamp(t, cfg.d_min, 1.0);
        if (dv < 1.0) {
          double p[3];
          lerp(x, nb, t, p, D);
          dd[dir] = dv;
          ob[dir] = (int8_t)attaining(L, p, D);
          cut = true;
        }
      }
      if (!cut && cfg.thin_rescue && h > cfg.w_min) {  // resolve_thin_boundary (:344-382)
        const double fa = fc[(size_t)ii];
        const int steps = (int)(h / cfg.w_min);
        double y[3] = {x[0], x[1], x[2]};
        for (int s = 0; s < steps; ++s) {
          double g[3];
          grad(L, y, h, D, g);
          const double gn = nrm(g, D);
          if (gn == 0) break;
          const double sc = cfg.w_min / gn;
          for (int k2 = 0; k2 < D; ++k2) y[k2] -= g[k2] * sc;
          if (fa * lsf(L, y, D) > 0) continue;
          const double t = bisect(L, x, y, 0.0, 1.0, cfg.eps_tol, D);
          double rt[3], rc[3];
          lerp(x, y, t, rt, D);
          for (int k2 = 0; k2 < D; ++k2) rc[k2] = rt[k2] - x[k2];
          const double hd = std::clamp(nrm(rc, D) / h, cfg.d_min, 1.0);
          int hdir = 0;
          double best = INF;
          for (int dir = 0; dir < 2 * D; ++dir) {
            double nb[3] = {x[0], x[1], x[2]};
            nb[dir / 2] += ((dir & 1) ? 1 : -1) * h;
            double rn[3];
            for (int k2 = 0; k2 < D; ++k2) rn[k2] = rt[k2] - nb[k2];
            const double dist = nrm(rn, D);
            if (dist < best) {
              best = dist;
              hdir = dir;
            }
          }
          dd[hdir] = hd;
          ob[hdir] = (int8_t)attaining(L, rt, D);
          cut = hd < 1.0;
          break;
        }
      }
      if (!cut) return;
      Row r;  // make_row (stencil.hpp:84-110)
      const double inv2 = 1.0 / (h * h);
      for (int a = 0; a < D; ++a) {
        const double dm = dd[2 * a], dp = dd[2 * a + 1];
        const double cm = 2.0 / ((dp + dm) * dm) * inv2;
        const double cp = 2.0 / ((dp + dm) * dp) * inv2;
        r.center -= 2.0 / (dm * dp) * inv2;
        if (dm < 1.0) {
          r.bc[2 * a] = cm;
          r.obj[2 * a] = ob[2 * a];
        } else {
          r.nb[2 * a] = cm;
        }
        if (dp < 1.0) {
          r.bc[2 * a + 1] = cp;
          r.obj[2 * a + 1] = ob[2 * a + 1];
        } else {
          r.nb[2 * a + 1] = cp;
        }
      }
      for (int dir = 0; dir < 2 * D; ++dir) r.d[dir] = dd[dir];
      r.lin = c.lin(i, j, k);
      b.row_of[(size_t)ii] = (int)b.rows.size();
      b.rows.push_back(r);
    });
  }
}

void pins(Ctx& c, int level) {  // apply_pins (stencil.hpp:225-237)
  for (int id : c.levels[(size_t)level]) {
    const BlockSt& b = c.st[(size_t)id];
    if (!b.boundary) continue;
    double* phi = c.f(id, PMG_VAR_PHI);
    for (const Row& r : b.rows)
      if (r.mask == PMG_INSIDE) phi[r.lin] = c.phib[(size_t)r.pin];
  }
}

// L(phi) of one cell: uniform (stencil.hpp:300-306) or row (:273-284)
double nbr_val(const Ctx& c, const double* phi, int l, int dir) {
  const int off = (dir / 2 == 0 ? 1 : dir / 2 == 1 ? c.s1 : c.s2) * ((dir & 1) ? 1 : -1);
  return phi[l + off];
}

double apply_cell(const Ctx& c, int id, const double* phi, int l, const Row* r, double w) {
  if (!r) {
    double s = -2.0 * c.D * phi[l];
    for (int dir = 0; dir < c.F; ++dir) s += nbr_val(c, phi, l, dir);
    return s * w;
  }
  (void)id;
  double s = r->center * phi[l];
  for (int dir = 0; dir < c.F; ++dir) {
    s += r->nb[dir] * nbr_val(c, phi, l, dir);
    if (r->bc[dir] != 0) s += r->bc[dir] * c.phib[(size_t)r->obj[dir]];
  }
  return s;
}

void residual_block(Ctx& c, int id) {  // stencil.hpp:325-359
  const double* phi = c.f(id, PMG_VAR_PHI);
  const double* g = c.f(id, PMG_VAR_RHS);
  double* out = c.f(id, PMG_VAR_RES);
  const double w = 1.0 / (c.bdx[(size_t)id] * c.bdx[(size_t)id]);
  c.each([&](int i, int j, int k, int ii) {
    const int l = c.lin(i, j, k);
    const Row* r = c.row(id, ii);
    if (r && r->mask == PMG_INSIDE) {
      out[l] = 0.0;
      return;
    }
    out[l] = g[l] - apply_cell(c, id, phi, l, r, w);
  });
}

void apply_block(Ctx& c, int id) {  // stencil.hpp:290-322, output into RHS
  const double* phi = c.f(id, PMG_VAR_PHI);
  double* out = c.f(id, PMG_VAR_RHS);
  const double w = 1.0 / (c.bdx[(size_t)id] * c.bdx[(size_t)id]);
  c.each([&](int i, int j, int k, int ii) {
    const int l = c.lin(i, j, k);
    const Row* r = c.row(id, ii);
    out[l] = (r && r->mask == PMG_INSIDE) ? 0.0 : apply_cell(c, id, phi, l, r, w);
  });
}

// ------------------------------------------------------------------ smoother (multigrid.hpp:621-695)
void gs_block(Ctx& c, int id, int parity) {
  double* phi = c.f(id, PMG_VAR_PHI);
  const double* g = c.f(id, PMG_VAR_RHS);
  const double h2 = c.bdx[(size_t)id] * c.bdx[(size_t)id];
  const BlockSt& b = c.st[(size_t)id];
  c.each([&](int i, int j, int k, int ii) {
    if (((i + j + k) & 1) != parity) return;
    const int l = c.lin(i, j, k);
    double p[6];
    for (int dir = 0; dir < c.F; ++dir) p[dir] = nbr_val(c, phi, l, dir);
    if (!b.boundary) {
      if (c.D == 3)
        phi[l] = (p[0] + p[1] + p[2] + p[3] + p[4] + p[5] - h2 * g[l]) / 6.0;
      else
        phi[l] = 0.25 * (p[0] + p[1] + p[2] + p[3] - h2 * g[l]);
      return;
    }
    const Row* r = c.row(id, ii);
    if (!r) {
      double s = -h2 * g[l];
      for (int dir = 0; dir < c.F; ++dir) s += p[dir];
      phi[l] = -s * (-1.0 / (2.0 * c.D));
      return;
    }
    if (r->mask == PMG_INSIDE) return;
    double num = g[l];
    for (int dir = 0; dir < c.F; ++dir) {
      num -= r->nb[dir] * p[dir];
      if (r->bc[dir] != 0) num -= r->bc[dir] * c.phib[(size_t)r->obj[dir]];
    }
    phi[l] = num / r->center;
  });
}

void gs_sweep(Ctx& c, int level, int parity) {
  for (int id : c.levels[(size_t)level]) gs_block(c, id, parity);
}

// ------------------------------------------------------------------ transfer operators
void restrict_to_parent(Ctx& c, int id, int var) {  // multigrid.hpp:697-722
  const int N = c.N, D = c.D, HN = N / 2;
  const double* src = c.f(id, var);
  double* dst = c.f(c.par[(size_t)id], var);
  int cp[3] = {0, 0, 0};
  for (int k = 0; k < D; ++k) cp[k] = (c.crd[(size_t)id][(size_t)k] & 1) * HN;
  for (int qz = 0; qz < (D == 3 ? HN : 1); ++qz)
    for (int qy = 0; qy < HN; ++qy)
      for (int qx = 0; qx < HN; ++qx) {
        double sum = 0;
        for (int dz = 0; dz < (D == 3 ? 2 : 1); ++dz)
          for (int dy = 0; dy < 2; ++dy)
            for (int dxx = 0; dxx < 2; ++dxx)
              sum += src[c.lin(2 * qx + dxx, 2 * qy + dy, D == 3 ? 2 * qz + dz : 0)];
        dst[c.lin(cp[0] + qx, cp[1] + qy, D == 3 ? cp[2] + qz : 0)] = sum / (1 << D);
      }
}

void restrict_level(Ctx& c, int l) {  // multigrid.hpp:374-398
  for (int id : c.levels[(size_t)l]) {
    restrict_to_parent(c, id, PMG_VAR_PHI);
    restrict_to_parent(c, id, PMG_VAR_RES);
  }
  pins(c, l - 1);
  fill(c, l - 1, PMG_VAR_PHI);
  for (int id : c.levels[(size_t)l - 1]) {
    if (!leaf(c, id)) {
      apply_block(c, id);
      double* g = c.f(id, PMG_VAR_RHS);
      const double* r = c.f(id, PMG_VAR_RES);
      for (int q = 0; q < c.S; ++q) g[q] += r[q];
    }
    std::memcpy(c.f(id, PMG_VAR_OLD), c.f(id, PMG_VAR_PHI), (size_t)c.S * sizeof(double));
  }
}

void restrict_level_no_guess(Ctx& c, int l) {  // multigrid.hpp:403-418
  for (int id : c.levels[(size_t)l]) {
    restrict_to_parent(c, id, PMG_VAR_PHI);
    restrict_to_parent(c, id, PMG_VAR_RHS);
  }
  pins(c, l - 1);
  fill(c, l - 1, PMG_VAR_PHI);
  for (int id : c.levels[(size_t)l - 1])
    std::memcpy(c.f(id, PMG_VAR_OLD), c.f(id, PMG_VAR_PHI), (size_t)c.S * sizeof(double));
}

void prolong(Ctx& c, int l, bool full) {  // multigrid.hpp:422-438,724-783
  const int N = c.N, D = c.D;
  for (int id : c.levels[(size_t)l]) {
    double* phi = c.f(id, PMG_VAR_PHI);
    const int p = c.par[(size_t)id];
    const double* pp = c.f(p, PMG_VAR_PHI);
    const double* po = c.f(p, PMG_VAR_OLD);
    c.each([&](int i, int j, int k, int ii) {
      if (c.inside(id, ii)) return;
      const int t[3] = {i, j, k};
      int pc[3] = {0, 0, 0}, sg[3] = {0, 0, 0};
      for (int a = 0; a < D; ++a) {
        const int gk = ((c.crd[(size_t)id][(size_t)a] & 1) ? N : 0) + t[a];
        pc[a] = gk >> 1;
        sg[a] = (gk & 1) ? 1 : -1;
      }
      const int pl = c.lin(pc[0], pc[1], pc[2]);
      if (full) {
        double v = (1.0 - 0.25 * D) * pp[pl];
        for (int a = 0; a < D; ++a) {
          int q[3] = {pc[0], pc[1], pc[2]};
          q[a] += sg[a];
          v += 0.25 * pp[c.lin(q[0], q[1], q[2])];
        }
        phi[c.lin(i, j, k)] = v;
      } else {
        double corr = (1.0 - 0.25 * D) * (pp[pl] - po[pl]);
        for (int a = 0; a < D; ++a) {
          int q[3] = {pc[0], pc[1], pc[2]};
          q[a] += sg[a];
          const int ql = c.lin(q[0], q[1], q[2]);
          corr += 0.25 * (pp[ql] - po[ql]);
        }
        phi[c.lin(i, j, k)] += corr;
      }
    });
  }
  fill(c, l, PMG_VAR_PHI);
}

// ------------------------------------------------------------------ coarse system (multigrid.hpp:62-280)
void assemble(Ctx& c) {  // assemble_level(mesh, set, 1)
  const int D = c.D, N = c.N;
  Coarse& cs = c.cs;
  cs = Coarse{};
  const auto& ids = c.levels[1];
  const int no = (int)c.phib.size();
  std::vector<std::vector<int>> unk(ids.size(), std::vector<int>((size_t)c.S, -1));
  std::map<int, size_t> order;
  for (size_t bi = 0; bi < ids.size(); ++bi) {
    order[ids[bi]] = bi;
    c.each([&](int i, int j, int k, int ii) {
      if (c.inside(ids[bi], ii)) return;
      unk[bi][(size_t)c.lin(i, j, k)] = cs.n++;
      cs.cell.emplace_back(ids[bi], c.lin(i, j, k));
    });
  }
  cs.c0.assign((size_t)cs.n, 0.0);
  cs.cobj.assign((size_t)no, std::vector<double>((size_t)cs.n, 0.0));
  std::vector<std::vector<std::pair<int, double>>> rows((size_t)cs.n);
  for (size_t bi = 0; bi < ids.size(); ++bi) {
    const int id = ids[bi];
    const double w = 1.0 / (c.bdx[(size_t)id] * c.bdx[(size_t)id]);
    c.each([&](int i, int j, int k, int ii) {
      const int row = unk[bi][(size_t)c.lin(i, j, k)];
      if (row < 0) return;
      const Row* r = c.row(id, ii);
      double diag, an[6];
      if (r) {
        diag = r->center;
        for (int dir = 0; dir < c.F; ++dir) {
          an[dir] = r->nb[dir];
          if (r->bc[dir] != 0) cs.cobj[(size_t)r->obj[dir]][(size_t)row] -= r->bc[dir];
        }
      } else {
        diag = -2.0 * D * w;
        for (int dir = 0; dir < c.F; ++dir) an[dir] = w;
      }
      for (int dir = 0; dir < c.F; ++dir) {
        const double a = an[dir];
        if (a == 0) continue;
        const int ax = dir / 2;
        int ni[3] = {i, j, k};
        ni[ax] += (dir & 1) ? 1 : -1;
        int nbk = id;
        size_t nord = bi;
        if (ni[ax] < 0 || ni[ax] >= N) {
          const int nid = c.nb[(size_t)id][(size_t)dir];
          if (nid < 0) {  // physical face folded through the ghost extrapolation
            if (c.bct[dir] == PMG_BC_NEUMANN_ZERO) {
              diag += a;
            } else {
              diag -= a;
              double x[3];
              c.center(id, i, j, k, x);
              x[ax] += 0.5 * c.bdx[(size_t)id] * ((dir & 1) ? 1 : -1);
              const double bv = c.bc_null(dir) ? 0.0 : c.bcval(dir, x);
              cs.c0[(size_t)row] -= 2.0 * a * bv;
            }
            continue;
          }
          nbk = nid;
          nord = order.at(nid);
          ni[ax] = ni[ax] < 0 ? N - 1 : 0;
        }
        const int col = unk[nord][(size_t)c.lin(ni[0], ni[1], ni[2])];
        if (col < 0) {
          const int nii = ni[0] + N * (ni[1] + N * ni[2]);
          cs.cobj[(size_t)c.row(nbk, nii)->pin][(size_t)row] -= a;
          continue;
        }
        rows[(size_t)row].emplace_back(col, a);
      }
      rows[(size_t)row].emplace_back(row, diag);
    });
  }
  cs.rp.assign((size_t)cs.n + 1, 0);
  for (int r = 0; r < cs.n; ++r) {
    auto& rw = rows[(size_t)r];
    std::sort(rw.begin(), rw.end());
    cs.rp[(size_t)r + 1] = cs.rp[(size_t)r] + (int)rw.size();
    for (auto& [col, v] : rw) {
      cs.ci.push_back(col);
      cs.val.push_back(v);
    }
  }
}

void spmv(const Coarse& A, const std::vector<double>& x, std::vector<double>& y) {
  for (int r = 0; r < A.n; ++r) {
    double s = 0;
    for (int q = A.rp[(size_t)r]; q < A.rp[(size_t)r + 1]; ++q) s += A.val[(size_t)q] * x[(size_t)A.ci[(size_t)q]];
    y[(size_t)r] = s;
  }
}

double norm2(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

struct Kry {
  bool conv = false;
  int iters = 0;
  double rel = 1.0;
};

Kry bicgstab(const Coarse& A, const std::vector<double>& b, std::vector<double>& x, double tol,
             int maxit) {  // multigrid.hpp:208-280
  const size_t n = (size_t)A.n;
  std::vector<double> dinv(n, 1.0);
  for (int r = 0; r < A.n; ++r)
    for (int q = A.rp[(size_t)r]; q < A.rp[(size_t)r + 1]; ++q)
      if (A.ci[(size_t)q] == r && A.val[(size_t)q] != 0) dinv[(size_t)r] = 1.0 / A.val[(size_t)q];
  std::vector<double> r(n), r0, p(n, 0.0), v(n, 0.0), s(n), t(n), ph(n), sh(n);
  spmv(A, x, r);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  r0 = r;
  const double n0 = norm2(r);
  Kry res;
  if (n0 == 0 || n0 < 1e-300) {
    res.conv = true;
    res.rel = 0;
    return res;
  }
  const double target = tol * n0;
  double rho = 1, alpha = 1, omega = 1;
  for (int it = 0; it < maxit; ++it) {
    double rho1 = 0;
    for (size_t i = 0; i < n; ++i) rho1 += r0[i] * r[i];
    if (rho1 == 0) break;
    if (it == 0) {
      p = r;
    } else {
      const double beta = (rho1 / rho) * (alpha / omega);
      for (size_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
    }
    for (size_t i = 0; i < n; ++i) ph[i] = dinv[i] * p[i];
    spmv(A, ph, v);
    double r0v = 0;
    for (size_t i = 0; i < n; ++i) r0v += r0[i] * v[i];
    if (r0v == 0) break;
    alpha = rho1 / r0v;
    for (size_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
    if (norm2(s) <= target) {
      for (size_t i = 0; i < n; ++i) x[i] += alpha * ph[i];
      res.conv = true;
      res.iters = it + 1;
      res.rel = norm2(s) / n0;
      return res;
    }
    for (size_t i = 0; i < n; ++i) sh[i] = dinv[i] * s[i];
    spmv(A, sh, t);
    double ts = 0, tt = 0;
    for (size_t i = 0; i < n; ++i) {
      ts += t[i] * s[i];
      tt += t[i] * t[i];
    }
    if (tt == 0) break;
    omega = ts / tt;
    for (size_t i = 0; i < n; ++i) {
      x[i] += alpha * ph[i] + omega * sh[i];
      r[i] = s[i] - omega * t[i];
    }
    rho = rho1;
    res.iters = it + 1;
    res.rel = norm2(r) / n0;
    if (res.rel <= tol) {
      res.conv = true;
      return res;
    }
    if (omega == 0) break;
  }
  return res;
}

// ------------------------------------------------------------------ records (multigrid.hpp:519-575)
void record(Ctx& c, int level) {
  Rec tot;
  for (int id : c.levels[(size_t)level]) {
    if (!leaf(c, id)) continue;
    residual_block(c, id);
    const double* r = c.f(id, PMG_VAR_RES);
    Rec b;
    c.each([&](int i, int j, int k, int ii) {
      if (c.inside(id, ii)) return;
      const double v = r[c.lin(i, j, k)];
      b.max = std::max(b.max, std::abs(v));
      b.sumsq += v * v;
      b.count += 1;
    });
    tot.max = std::max(tot.max, b.max);
    tot.sumsq += b.sumsq;
    tot.count += b.count;
  }
  c.recs[(size_t)level] = tot;
}

pmg_cycle_stats_t combine(const Ctx& c) {
  pmg_cycle_stats_t s{0, 0};
  double sq = 0;
  long n = 0;
  for (const Rec& r : c.recs) {
    s.max_resid = std::max(s.max_resid, r.max);
    sq += r.sumsq;
    n += r.count;
  }
  s.l2_resid = n > 0 ? std::sqrt(sq / (double)n) : 0;
  return s;
}

void reset_records(Ctx& c) { c.recs.assign((size_t)c.nlevels() + 1, Rec{}); }

double level_max_resid(Ctx& c, int level) {
  double m = 0;
  for (int id : c.levels[(size_t)level]) {
    const double* r = c.f(id, PMG_VAR_RES);
    c.each([&](int i, int j, int k, int ii) {
      if (!c.inside(id, ii)) m = std::max(m, std::abs(r[c.lin(i, j, k)]));
    });
  }
  return m;
}

void write_back(Ctx& c, const std::vector<double>& x) {
  for (size_t u = 0; u < x.size(); ++u) c.f(c.cs.cell[u].first, PMG_VAR_PHI)[c.cs.cell[u].second] = x[u];
}

void coarse_rhs(Ctx& c, std::vector<double>& b, std::vector<double>& x) {  // multigrid.hpp:443-453
  const size_t n = (size_t)c.cs.n;
  b.assign(n, 0.0);
  x.assign(n, 0.0);
  for (size_t u = 0; u < n; ++u) {
    b[u] = c.f(c.cs.cell[u].first, PMG_VAR_RHS)[c.cs.cell[u].second] + c.cs.c0[u];
    x[u] = c.f(c.cs.cell[u].first, PMG_VAR_PHI)[c.cs.cell[u].second];
  }
  for (size_t o = 0; o < c.phib.size(); ++o)
    for (size_t u = 0; u < n; ++u) b[u] += c.cs.cobj[o][u] * c.phib[o];
}

void coarse_solve(Ctx& c) {  // multigrid.hpp:442-472, 586-601
  std::vector<double> b, x;
  coarse_rhs(c, b, x);
  const Kry res = bicgstab(c.cs, b, x, c.cfg.coarse_rel_tol, c.cfg.coarse_max_iters);
  if (!res.conv) {
    if (c.cs.n <= (int)std::pow(8, c.D) + 1) {
      write_back(c, x);
      double r0 = -1;
      bool ok = false;
      for (int it = 0; it < 20000 && !ok; ++it) {
        gs_sweep(c, 1, 0);
        fill(c, 1, PMG_VAR_PHI);
        gs_sweep(c, 1, 1);
        fill(c, 1, PMG_VAR_PHI);
        if (it % 50 == 0) {
          for (int id : c.levels[1]) residual_block(c, id);
          const double m = level_max_resid(c, 1);
          if (r0 < 0) r0 = m;
          if (m <= c.cfg.coarse_rel_tol * r0 || m < 1e-300) ok = true;
        }
      }
      if (!ok) throw Err(PMG_ERR_COARSE_STALL, "coarse solve failed: smoothing fallback stalled");
    } else {
      throw Err(PMG_ERR_COARSE_STALL,
                "coarse solve failed: BiCGStab stalled at relative residual " +
                    std::to_string(res.rel) + " after " + std::to_string(res.iters) +
                    " iterations on " + std::to_string(c.cs.n) + " unknowns");
    }
  } else {
    write_back(c, x);
  }
  pins(c, 1);
  fill(c, 1, PMG_VAR_PHI);
  record(c, 1);
}

void smooth(Ctx& c, int l, int steps) {  // multigrid.hpp:501-508
  for (int s = 0; s < steps; ++s) {
    gs_sweep(c, l, 0);
    fill(c, l, PMG_VAR_PHI);
    gs_sweep(c, l, 1);
    fill(c, l, PMG_VAR_PHI);
  }
}

void residual_level(Ctx& c, int l) {
  for (int id : c.levels[(size_t)l]) residual_block(c, id);
}

void v_span(Ctx& c, int top) {  // multigrid.hpp:483-499
  if (top == 1) {
    coarse_solve(c);
    return;
  }
  for (int l = top; l >= 2; --l) {
    smooth(c, l, c.cfg.n_down);
    residual_level(c, l);
    restrict_level(c, l);
  }
  coarse_solve(c);
  for (int l = 2; l <= top; ++l) {
    prolong(c, l, false);
    smooth(c, l, c.cfg.n_up);
    record(c, l);
  }
}

void init(Ctx& c) {  // multigrid.hpp:304-311
  for (int l = 1; l <= c.nlevels(); ++l) pins(c, l);
  for (int l = 1; l <= c.nlevels(); ++l) fill(c, l, PMG_VAR_PHI);
  assemble(c);
  reset_records(c);
  c.have_guess = false;
}

pmg_cycle_stats_t v_cycle(Ctx& c) {  // :318-323
  reset_records(c);
  v_span(c, c.nlevels());
  c.have_guess = true;
  return combine(c);
}

pmg_cycle_stats_t fmg_cycle(Ctx& c) {  // :325-350
  reset_records(c);
  const int L = c.nlevels();
  for (int l = L; l >= 2; --l) {
    fill(c, l, PMG_VAR_PHI);
    if (c.have_guess) {
      residual_level(c, l);
      restrict_level(c, l);
    } else {
      restrict_level_no_guess(c, l);
    }
  }
  const bool guess = c.have_guess;
  coarse_solve(c);
  for (int l = 2; l <= L; ++l) {
    prolong(c, l, !guess);
    v_span(c, l);
  }
  c.have_guess = true;
  return combine(c);
}

pmg_cycle_stats_t measure(Ctx& c) {  // :353-360
  reset_records(c);
  for (int l = 1; l <= c.nlevels(); ++l) {
    fill(c, l, PMG_VAR_PHI);
    record(c, l);
  }
  return combine(c);
}

}  // namespace

// ================================================================== C interface
struct oc_ctx {
  Ctx c;
};

template <class Fn>
static int guard(oc_ctx* h, Fn&& fn) {
  if (!h) return PMG_ERR_STATE;
  try {
    h->c.err.clear();
    return fn(h->c);
  } catch (const Err& e) {
    h->c.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    h->c.err = e.what();
    return PMG_ERR_INVALID_ARG;
  }
}

static Lsf make_lsf(const pmg_lsf_t* l, int n) {
  Lsf L;
  L.d.assign(l, l + (l[0].shape == PMG_SHAPE_COMPOSITE_MIN ? n : 1));
  return L;
}

static void need_solver(Ctx& c) {
  if (!c.have_solver) throw Err(PMG_ERR_STATE, "solver not created");
}

extern "C" {

oc_ctx* oc_create(int dim, int N, const double* lo, const double* hi) {
  auto* h = new oc_ctx;
  Ctx& c = h->c;
  try {
    need(dim == 2 || dim == 3, "dim must be 2 or 3");
    need(N >= 4 && (N & (N - 1)) == 0, "block size N must be a power of two and at least 4");
    c.D = dim;
    c.N = N;
    c.F = 2 * dim;
    c.s1 = N + 2;
    c.s2 = (N + 2) * (N + 2);
    c.S = dim == 2 ? c.s2 : c.s2 * (N + 2);
    c.NI = dim == 2 ? N * N : N * N * N;
    const double ext = hi[0] - lo[0];
    for (int k = 0; k < dim; ++k) {
      c.lo[k] = lo[k];
      c.hi[k] = hi[k];
      need(std::abs((hi[k] - lo[k]) - ext) <= 1e-12 * std::abs(ext), "domain must be square/cubic");
    }
    need(ext > 0, "domain extent must be positive");
    new_block(c, 1, {0, 0, 0}, {lo[0], lo[1], dim == 3 ? lo[2] : 0.0}, ext / N, -1);
    topology(c);
    c.st.assign(1, BlockSt{});
  } catch (const std::exception& e) {
    c.err = e.what();
  }
  return h;
}
void oc_destroy(oc_ctx* h) { delete h; }
const char* oc_last_error(oc_ctx* h) { return h ? h->c.err.c_str() : "null handle"; }

int oc_build_uniform(oc_ctx* h, int levels) {  // mesh.hpp:565-572
  return guard(h, [&](Ctx& c) {
    need(levels >= 1, "levels must be at least 1");
    Ctx fresh;
    fresh.D = c.D, fresh.N = c.N, fresh.F = c.F, fresh.S = c.S, fresh.NI = c.NI;
    fresh.s1 = c.s1, fresh.s2 = c.s2;
    std::copy(c.lo, c.lo + 3, fresh.lo);
    std::copy(c.hi, c.hi + 3, fresh.hi);
    std::copy(c.bct, c.bct + 6, fresh.bct);
    std::copy(c.bcc, c.bcc + 6, fresh.bcc);
    std::memcpy(fresh.bcg, c.bcg, sizeof(c.bcg));
    new_block(fresh, 1, {0, 0, 0}, {c.lo[0], c.lo[1], c.lo[2]}, (c.hi[0] - c.lo[0]) / c.N, -1);
    topology(fresh);
    c = std::move(fresh);
    for (int t = 0; t < levels - 1; ++t) {
      std::vector<int> ids;
      for (int id = 0; id < c.nblocks(); ++id)
        if (leaf(c, id)) ids.push_back(id);
      adapt_refine(c, ids, levels);
    }
    c.st.assign((size_t)c.nblocks(), BlockSt{});
    return 0;
  });
}
int oc_refine_band(oc_ctx* h, const pmg_lsf_t* l, int n, double band, int max_level) {
  return guard(h, [&](Ctx& c) {  // harness.hpp:295-321 with want = |f(x)| < band * b.dx
    const Lsf L = make_lsf(l, n);
    for (;;) {
      std::vector<int> flags;
      for (int lv = 1; lv <= c.nlevels(); ++lv)
        for (int id : c.levels[(size_t)lv]) {
          if (!leaf(c, id) || c.lvl[(size_t)id] >= max_level) continue;
          bool f = false;
          c.each([&](int i, int j, int k, int) {
            if (f) return;
            double x[3];
            c.center(id, i, j, k, x);
            if (std::abs(lsf(L, x, c.D)) < band * c.bdx[(size_t)id]) f = true;
          });
          if (f) flags.push_back(id);
        }
      if (flags.empty()) break;
      adapt_refine(c, flags, max_level);
    }
    c.st.assign((size_t)c.nblocks(), BlockSt{});
    c.have_solver = false;
    return 0;
  });
}
int oc_adapt(oc_ctx* h, const uint8_t* flags, int n, int max_level) {
  return guard(h, [&](Ctx& c) {  // TreeMesh::adapt, refine flags (mesh.hpp:157-175,198)
    std::vector<int> ids;
    for (int id = 0; id < c.nblocks() && id < n; ++id)
      if (flags[id] == 1) ids.push_back(id);
    adapt_refine(c, ids, max_level);
    c.st.assign((size_t)c.nblocks(), BlockSt{});
    c.have_solver = false;
    return 0;
  });
}
int oc_refine_crit(oc_ctx* h, int kind, double p0, double p1, const double* centre, int max_level) {
  return guard(h, [&](Ctx& c) {  // harness.hpp:295-321 with the criteria of :351-355 (1) and :413-418 (2)
    for (;;) {
      std::vector<int> flags;
      for (int lv = 1; lv <= c.nlevels(); ++lv)
        for (int id : c.levels[(size_t)lv]) {
          if (!leaf(c, id) || c.lvl[(size_t)id] >= max_level) continue;
          bool f = false;
          const double bdx = c.bdx[(size_t)id];
          c.each([&](int i, int j, int k, int) {
            if (f) return;
            double x[3];
            c.center(id, i, j, k, x);
            double ss = 0;
            for (int a = 0; a < c.D; ++a) ss += (x[a] - centre[a]) * (x[a] - centre[a]);
            const double r = std::sqrt(ss);
            const bool w = kind == 1 ? bdx > p0 * std::max(1.0, r / p1) : (bdx > p0 && r < p1);
            if (w) f = true;
          });
          if (f) flags.push_back(id);
        }
      if (flags.empty()) break;
      adapt_refine(c, flags, max_level);
    }
    c.st.assign((size_t)c.nblocks(), BlockSt{});
    c.have_solver = false;
    return 0;
  });
}
int oc_n_blocks(oc_ctx* h) { return h ? h->c.nblocks() : -1; }
int oc_n_levels(oc_ctx* h) { return h ? h->c.nlevels() : -1; }
int oc_get_topology(oc_ctx* h, int32_t* level, int32_t* coords, double* origin, double* dx,
                    int32_t* parent, int32_t* children, int32_t* nbr, int32_t* cnbr) {
  return guard(h, [&](Ctx& c) {
    for (int id = 0; id < c.nblocks(); ++id) {
      level[id] = c.lvl[(size_t)id];
      dx[id] = c.bdx[(size_t)id];
      parent[id] = c.par[(size_t)id];
      for (int k = 0; k < 3; ++k) {
        coords[3 * id + k] = k < c.D ? c.crd[(size_t)id][(size_t)k] : 0;
        origin[3 * id + k] = k < c.D ? c.org[(size_t)id][(size_t)k] : 0.0;
      }
      for (int q = 0; q < 8; ++q) children[8 * id + q] = q < (1 << c.D) ? c.kids[(size_t)id][(size_t)q] : -1;
      for (int f = 0; f < 6; ++f) {
        nbr[6 * id + f] = f < c.F ? c.nb[(size_t)id][(size_t)f] : -1;
        cnbr[6 * id + f] = f < c.F ? c.cnb[(size_t)id][(size_t)f] : -1;
      }
    }
    return 0;
  });
}
int oc_level_blocks(oc_ctx* h, int level, int32_t* ids) {
  if (!h || level < 1 || level > h->c.nlevels()) return 0;
  const auto& v = h->c.levels[(size_t)level];
  std::copy(v.begin(), v.end(), ids);
  return (int)v.size();
}
int oc_set_face_bc(oc_ctx* h, int dir, int type, double cval, const double* g) {
  return guard(h, [&](Ctx& c) {
    c.bct[dir] = type;
    c.bcc[dir] = cval;
    for (int k = 0; k < 3; ++k) c.bcg[dir][k] = (g && k < c.D) ? g[k] : 0.0;
    return 0;
  });
}
int oc_set_field(oc_ctx* h, int var, const double* buf) {
  return guard(h, [&](Ctx& c) {
    for (int id = 0; id < c.nblocks(); ++id) std::copy(buf + (size_t)id * c.S, buf + (size_t)(id + 1) * c.S, c.f(id, var));
    return 0;
  });
}
int oc_get_field(oc_ctx* h, int var, double* buf) {
  return guard(h, [&](Ctx& c) {
    for (int id = 0; id < c.nblocks(); ++id) std::copy(c.f(id, var), c.f(id, var) + c.S, buf + (size_t)id * c.S);
    return 0;
  });
}
int oc_build_stencils(oc_ctx* h, const pmg_lsf_t* l, int n, const pmg_stencil_cfg_t* cfg) {
  return guard(h, [&](Ctx& c) {
    build_stencils(c, make_lsf(l, n), *cfg);
    c.have_solver = false;
    return 0;
  });
}
int oc_stencil_summary(oc_ctx* h, int32_t* boundary, int32_t* rc) {
  if (!h) return -PMG_ERR_STATE;
  int tot = 0;
  for (int id = 0; id < h->c.nblocks(); ++id) {
    const BlockSt& b = h->c.st[(size_t)id];
    if (boundary) boundary[id] = b.boundary;
    if (rc) rc[id] = (int)b.rows.size();
    tot += (int)b.rows.size();
  }
  return tot;
}
int oc_get_stencils(oc_ctx* h, int32_t* row_of, double* center, double* nb, double* bc, double* d,
                    int8_t* obj, uint8_t* mask, int8_t* pin, int32_t* lin) {
  return guard(h, [&](Ctx& c) {
    size_t r = 0;
    const int F = c.F;
    for (int id = 0; id < c.nblocks(); ++id) {
      const BlockSt& b = c.st[(size_t)id];
      for (int q = 0; q < c.NI; ++q) row_of[(size_t)id * c.NI + q] = b.boundary ? b.row_of[(size_t)q] : -1;
      for (const Row& w : b.rows) {
        center[r] = w.center;
        for (int f = 0; f < F; ++f) {
          nb[r * F + f] = w.nb[f];
          bc[r * F + f] = w.bc[f];
          d[r * F + f] = w.d[f];
          obj[r * F + f] = w.obj[f];
        }
        mask[r] = w.mask;
        pin[r] = w.pin;
        lin[r] = w.lin;
        ++r;
      }
    }
    return 0;
  });
}
int oc_set_stencils(oc_ctx* h, const int32_t* boundary, const int32_t* rc, const int32_t* row_of,
                    const double* center, const double* nb, const double* bc, const double* d,
                    const int8_t* obj, const uint8_t* mask, const int8_t* pin, const int32_t* lin,
                    int n_obj, const double* phi_b) {
  return guard(h, [&](Ctx& c) {
    c.st.assign((size_t)c.nblocks(), BlockSt{});
    c.phib.assign(phi_b, phi_b + n_obj);
    size_t r = 0;
    const int F = c.F;
    for (int id = 0; id < c.nblocks(); ++id) {
      BlockSt& b = c.st[(size_t)id];
      b.boundary = boundary[id] != 0;
      if (b.boundary) b.row_of.assign(row_of + (size_t)id * c.NI, row_of + (size_t)(id + 1) * c.NI);
      for (int q = 0; q < rc[id]; ++q, ++r) {
        Row w;
        w.center = center[r];
        for (int f = 0; f < F; ++f) {
          w.nb[f] = nb[r * F + f];
          w.bc[f] = bc[r * F + f];
          w.d[f] = d[r * F + f];
          w.obj[f] = obj[r * F + f];
        }
        w.mask = mask[r];
        w.pin = pin[r];
        w.lin = lin[r];
        b.rows.push_back(w);
      }
    }
    c.have_solver = false;
    return 0;
  });
}
int oc_set_boundary_value(oc_ctx* h, int obj, double v) {
  return guard(h, [&](Ctx& c) {
    c.phib.at((size_t)obj) = v;
    return 0;
  });
}
int oc_solver_create(oc_ctx* h, const pmg_mg_cfg_t* cfg) {
  return guard(h, [&](Ctx& c) {  // MgConfig::validate (multigrid.hpp:22-27) + init
    need(cfg->n_down >= 1 && cfg->n_up >= 1, "n_up and n_down must be at least 1");
    need(cfg->coarse_rel_tol > 0 && cfg->coarse_rel_tol < 1, "coarse_rel_tol must be in (0, 1)");
    need(cfg->threads >= 1, "thread count must be at least 1");
    if (c.st.size() != (size_t)c.nblocks()) c.st.assign((size_t)c.nblocks(), BlockSt{});
    c.cfg = *cfg;
    init(c);
    c.have_solver = true;
    return 0;
  });
}
#define OC_OP(sig, body) \
  int sig { return guard(h, [&](Ctx& c) { body; return 0; }); }
OC_OP(oc_init(oc_ctx* h), need_solver(c); init(c))
OC_OP(oc_v_cycle(oc_ctx* h, pmg_cycle_stats_t* out), need_solver(c); *out = v_cycle(c))
OC_OP(oc_fmg_cycle(oc_ctx* h, pmg_cycle_stats_t* out), need_solver(c); *out = fmg_cycle(c))
OC_OP(oc_measure_residual(oc_ctx* h, pmg_cycle_stats_t* out), need_solver(c); *out = measure(c))
OC_OP(oc_gsrb_sweep(oc_ctx* h, int level, int parity), gs_sweep(c, level, parity))
OC_OP(oc_fill_ghosts(oc_ctx* h, int level, int var), fill(c, level, var))
OC_OP(oc_apply_pins(oc_ctx* h, int level), pins(c, level))
OC_OP(oc_residual_level(oc_ctx* h, int level), residual_level(c, level))
OC_OP(oc_restrict_level(oc_ctx* h, int level), need_solver(c); restrict_level(c, level))
OC_OP(oc_restrict_level_no_guess(oc_ctx* h, int level), need_solver(c); restrict_level_no_guess(c, level))
OC_OP(oc_prolong_correction(oc_ctx* h, int level), need_solver(c); prolong(c, level, false))
OC_OP(oc_prolong_full(oc_ctx* h, int level), need_solver(c); prolong(c, level, true))
OC_OP(oc_coarse_solve(oc_ctx* h), need_solver(c); coarse_solve(c))
OC_OP(oc_set_have_guess(oc_ctx* h, int v), need_solver(c); c.have_guess = v != 0)
#undef OC_OP
int oc_coarse_sizes(oc_ctx* h, int32_t* n, int32_t* nnz, int32_t* nobj) {
  return guard(h, [&](Ctx& c) {
    need_solver(c);
    *n = c.cs.n;
    *nnz = (int32_t)c.cs.val.size();
    *nobj = (int32_t)c.cs.cobj.size();
    return 0;
  });
}
int oc_coarse_get(oc_ctx* h, int32_t* rp, int32_t* ci, double* val, double* c0, double* cobj,
                  int32_t* ub, int32_t* ul) {
  return guard(h, [&](Ctx& c) {
    need_solver(c);
    const Coarse& cs = c.cs;
    std::copy(cs.rp.begin(), cs.rp.end(), rp);
    std::copy(cs.ci.begin(), cs.ci.end(), ci);
    std::copy(cs.val.begin(), cs.val.end(), val);
    std::copy(cs.c0.begin(), cs.c0.end(), c0);
    for (size_t o = 0; o < cs.cobj.size(); ++o)
      std::copy(cs.cobj[o].begin(), cs.cobj[o].end(), cobj + o * (size_t)cs.n);
    for (int u = 0; u < cs.n; ++u) {
      ub[u] = cs.cell[(size_t)u].first;
      ul[u] = cs.cell[(size_t)u].second;
    }
    return 0;
  });
}
int oc_bicgstab_probe(oc_ctx* h, int32_t* conv, int32_t* iters, double* rel) {
  return guard(h, [&](Ctx& c) {
    need_solver(c);
    std::vector<double> b, x;
    coarse_rhs(c, b, x);
    const Kry r = bicgstab(c.cs, b, x, c.cfg.coarse_rel_tol, c.cfg.coarse_max_iters);
    *conv = r.conv;
    *iters = r.iters;
    *rel = r.rel;
    return 0;
  });
}

}  // extern "C"
