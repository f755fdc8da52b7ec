// capi.cu -- host orchestration of the B200 multigrid hot path and the C-ABI
// (include/pmg_b200.h).
//
// The cycle structure is MgSolver's (multigrid.hpp:318-350, 483-508); each
// reference phase maps to one or more kernels (see kernels.cuh) and every
// cycle type is captured once into a CUDA graph and replayed.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <tuple>

#include "ctx.h"
#include "dist.h"

using namespace pmghost;
using pmgdev::LevelView;

struct pmg_b200_ctx {
  Ctx c;
};

namespace pmghost {

Ctx::~Ctx() {
  dist.reset();
  g_v.reset();
  g_fmg[0].reset();
  g_fmg[1].reset();
  g_measure.reset();
  if (h_out) cudaFreeHost(h_out);
  if (h_buf) cudaFreeHost(h_buf);
  if (stream) cudaStreamDestroy(stream);
  if (side) cudaStreamDestroy(side);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (copy) cudaStreamDestroy(copy);
  if (ev_staged) cudaEventDestroy(ev_staged);
  if (ev_consumed) cudaEventDestroy(ev_consumed);
}

static void require(bool cond, const std::string& msg, int code = PMG_ERR_INVALID_ARG) {
  if (!cond) throw PmgError(code, msg);
}

static uint64_t morton(const int32_t* c, int dim) {
  uint64_t m = 0;
  for (int b = 0; b < 21; ++b)
    for (int k = 0; k < dim; ++k) m |= (uint64_t)((c[k] >> b) & 1) << (b * dim + k);
  return m;
}

static void set_views(Ctx& c) {
  for (int l = 1; l <= c.mesh.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    LevelView& v = d.view;
    v.nb = d.nb;
    v.level = l;
    const double dx = c.mesh.dx[(size_t)c.mesh.slots[(size_t)l][0]];
    v.dx = dx;
    v.h2 = dx * dx;
    v.w = 1.0 / (dx * dx);
    v.nbr = d.nbr.p;
    v.cnbr = d.cnbr.p;
    v.coords = d.coords.p;
    v.parent = d.parent.p;
    v.child = d.child.p;
    v.leaf = d.leaf.p;
    v.kind = d.kind.p;
    v.srow = d.srow.p;
    v.bcoff = d.bcoff.p;
    v.bcval = d.bcval.p;
    v.phi = d.phi.p;
    v.rhs = d.rhs.p;
    v.old = d.old.p;
    v.res = d.res.p;
    v.row_of = d.row_of.p;
    v.skind = d.skind.p;
    v.own = d.has_own ? d.own.p : nullptr;
    v.r_coef = d.r_coef.p;
    v.r_center = d.r_center.p;
    v.r_nb = d.r_nb.p;
    v.r_d = d.r_d.p;
    v.r_bc = d.r_bc.p;
    v.r_obj = d.r_obj.p;
    v.r_mask = d.r_mask.p;
    v.r_pin = d.r_pin.p;
    v.cfold = d.cfold.p;
    v.cfoff = d.has_cfold ? d.cfoff.p : nullptr;
    v.cfc = nullptr;  // the launchers that read the table set it (ops_impl.cuh Vt)
    for (int k = 0; k < 6; ++k) v.bctype[k] = c.bctype[k];
    v.dense = d.dense ? 1 : 0;
    v.nside = 1 << (l - 1);
    v.bczero = d.bczero ? 1 : 0;
  }
}

static void invalidate_graphs(Ctx& c) {
  if (c.dist) c.dist->g.reset(), c.dist->graph_failed = false;
  c.g_v.reset();
  c.g_fmg[0].reset();
  c.g_fmg[1].reset();
  c.g_measure.reset();
}

// colour-split entry address of interior cell ii (x-fastest) within a block
static inline int cs_addr(int ii, int N, int dim, int H) {
  const int i = ii % N, j = (ii / N) % N, k = dim == 3 ? ii / (N * N) : 0;
  return ((i + j + k) & 1) * H + (ii >> 1);
}

// multi-GPU ownership (pmg_b200_set_owned): blocks this rank computes
static bool own_slot(const Ctx& c, int l, int s) {
  const auto& o = c.owned;
  return (size_t)l >= o.size() || o[(size_t)l].empty() || o[(size_t)l][(size_t)s] != 0;
}

static void upload_bc(Ctx& c) {
  const HostMesh& m = c.mesh;
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    std::vector<int32_t> off((size_t)d.nb * c.F, -1);
    std::vector<double> vals;
    for (int s = 0; s < d.nb; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      for (int f = 0; f < c.F; ++f) {
        const int32_t o = c.face_off[f].empty() ? -1 : c.face_off[f][(size_t)id];
        if (o < 0) continue;
        off[(size_t)s * c.F + f] = (int32_t)vals.size();
        vals.insert(vals.end(), c.face_vals[f].begin() + o, c.face_vals[f].begin() + o + c.NT);
      }
    }
    d.bcoff.upload(off, c.stream);
    d.bcval.upload(vals, c.stream);
    d.bczero = vals.empty();
  }
}

// k_gs_cut tables: every cut (non-inside special) row of a lean interface
// block (no coarse-fine face), per level and colour, with its row index in
// the level's row arrays and the addresses of its 2D neighbour values
// (same block, same-level neighbour block, or a physical-face code).
// 3D N = 8 / 16: the streaming GS kernel also takes blocks with coarse-fine
// faces (their ghosts from the cfc table), unless a cut row sits near such a
// face (cf_streamable below)
static bool stream_dn(const Ctx& c) { return c.dim == 3 && (c.N == 8 || c.N == 16); }
static bool has_cf_face(const Ctx& c, int id) {
  for (int f = 0; f < c.F; ++f)
    if (c.mesh.nbr[(size_t)id * 6 + f] < 0 && c.mesh.cnbr[(size_t)id * 6 + f] >= 0) return true;
  return false;
}
// The criterion: no cut row within two cells of a coarse-fine face -- the
// 2x2x2 children of a parent with a cut child are gathered by k_restrict_fix,
// whose entries (like k_gs_cut's) cannot express such a ghost.  One criterion
// for the GS, record, restriction and FAS plans and the cut-row tables.
static bool cf_streamable(const Ctx& c, int id) {
  const HostStencils& st = c.st;
  if (!stream_dn(c) || !has_cf_face(c, id)) return false;
  if (!st.valid || !st.boundary[(size_t)id]) return true;
  const int N = c.N, r0 = st.row_start[(size_t)id];
  for (int f = 0; f < c.F; ++f) {
    if (!(c.mesh.nbr[(size_t)id * 6 + f] < 0 && c.mesh.cnbr[(size_t)id * 6 + f] >= 0)) continue;
    const int ax = f >> 1;
    for (int w = 0; w < 2; ++w)
      for (int v = 0; v < N; ++v)
        for (int u = 0; u < N; ++u) {
          int q[3];
          q[ax] = (f & 1) ? N - 1 - w : w;
          q[ax == 0 ? 1 : 0] = u;
          q[ax == 2 ? 1 : 2] = v;
          const int r = st.row_at((size_t)id, (size_t)(q[0] + N * (q[1] + N * q[2])));
          if (r >= 0 && st.mask[(size_t)(r0 + r)] != PMG_INSIDE) return false;
        }
  }
  return true;
}

static void build_cut_tables(Ctx& c) {
  const HostMesh& m = c.mesh;
  const HostStencils& st = c.st;
  const int N = c.N, D = c.dim, NI = c.NI, H = NI / 2, F = c.F;
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    std::vector<int32_t> ent[2], off[2], entc[2];
    std::vector<double> gbc[2], coef[2], gbcc[2], coefc[2];  // ..c: blocks with coarse-fine faces (gs_cf)
    int base = 0;  // row offset of the block within the level's row arrays (upload_stencils order)
    for (int s = 0; s < d.nb && st.valid; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      for (int cc = 0; cc < 2; ++cc) off[cc].push_back((int32_t)(ent[cc].size() / 8));  // k_gs_coop row ranges
      if (!st.boundary[(size_t)id]) continue;
      const int rc = st.row_count[(size_t)id];
      const int r0 = st.row_start[(size_t)id];
      bool no_cf = true, all_inside = true;
      for (int f = 0; f < F; ++f) no_cf = no_cf && !(m.nbr[(size_t)id * 6 + f] < 0 && m.cnbr[(size_t)id * 6 + f] >= 0);
      for (int ii = 0; ii < NI; ++ii) {
        const int r = st.row_at((size_t)id, (size_t)ii);
        if (r < 0 || st.mask[(size_t)(r0 + r)] != PMG_INSIDE) all_inside = false;
      }
      const bool cfs = !no_cf && cf_streamable(c, id);
      if ((no_cf || cfs) && !all_inside && own_slot(c, l, s))
        for (int ii = 0; ii < NI; ++ii) {
          const int r = st.row_at((size_t)id, (size_t)ii);
          if (r < 0 || st.mask[(size_t)(r0 + r)] == PMG_INSIDE) continue;
          const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
          const int cc = (i + j + k) & 1;
          int32_t e[8] = {(int32_t)((size_t)s * NI + cs_addr(ii, N, D, H)), base + r, 0, 0, 0, 0, 0, 0};
          double gb[6] = {0, 0, 0, 0, 0, 0};
          for (int f = 0; f < F; ++f) {
            const int ax = f / 2, sg = (f & 1) ? 1 : -1;
            int q[3] = {i, j, k};
            q[ax] += sg;
            if (q[ax] >= 0 && q[ax] < N) {
              e[2 + f] = (int32_t)((size_t)s * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
              continue;
            }
            const int nid = m.nbr[(size_t)id * 6 + f];
            if (nid >= 0) {
              q[ax] = sg > 0 ? 0 : N - 1;
              e[2 + f] = (int32_t)((size_t)m.slot_of[(size_t)nid] * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
              continue;
            }
            require(m.cnbr[(size_t)id * 6 + f] < 0, "cut row on a coarse-fine face in a streamed block", PMG_ERR_STATE);
            if (c.bctype[f] == PMG_BC_NEUMANN_ZERO) {
              e[2 + f] = -1;
              continue;
            }
            e[2 + f] = -2;
            if (!c.face_off[f].empty() && c.face_off[f][(size_t)id] >= 0) {
              const int t = D == 2 ? (ax == 0 ? j : i) : (ax == 0 ? j + N * k : ax == 1 ? i + N * k : i + N * j);
              gb[f] = c.face_vals[f][(size_t)c.face_off[f][(size_t)id] + t];
            }
          }
          (cfs ? entc : ent)[cc].insert((cfs ? entc : ent)[cc].end(), e, e + 8);
          (cfs ? gbcc : gbc)[cc].insert((cfs ? gbcc : gbc)[cc].end(), gb, gb + 6);
          // row coefficients, with each cut direction's bc * phi_b product formed
          // here exactly as the reference forms it (stencil.hpp:344-358)
          const size_t q = (size_t)(r0 + r);
          double cf[16] = {st.center[q]};
          int bm = 0;
          for (int f = 0; f < F; ++f) {
            cf[1 + f] = st.nb[q * F + f];
            const double b = st.bc[q * F + f];
            if (b != 0) {
              bm |= 1 << f;
              cf[7 + f] = b * st.phi_b[(size_t)st.obj[q * F + f]];
            }
          }
          cf[13] = (double)bm;
          (cfs ? coefc : coef)[cc].insert((cfs ? coefc : coef)[cc].end(), cf, cf + 16);
        }
      base += rc;
    }
    for (int cc = 0; cc < 2; ++cc) {
      off[cc].resize((size_t)d.nb, (int32_t)(ent[cc].size() / 8));
      off[cc].push_back((int32_t)(ent[cc].size() / 8));
      d.cut_off[cc].upload(off[cc], c.stream);
      d.n_cut[cc] = (int)ent[cc].size() / 8;
      d.cut_ent[cc].upload(ent[cc], c.stream);
      d.cut_gbc[cc].upload(gbc[cc], c.stream);
      d.cut_coef[cc].upload(coef[cc], c.stream);
      d.n_cutcf[cc] = (int)entc[cc].size() / 8;
      d.cutcf_ent[cc].upload(entc[cc], c.stream);
      d.cutcf_gbc[cc].upload(gbcc[cc], c.stream);
      d.cutcf_coef[cc].upload(coefc[cc], c.stream);
    }
  }
}

// small.cuh tables for levels of at most kSmallLevel blocks without
// coarse-fine faces: per cell (colour-split address) the row code, the 2D
// neighbour addresses / physical-ghost codes, the Dirichlet values, the leaf flag.
static void build_small_tables(Ctx& c) {
  const HostMesh& m = c.mesh;
  const HostStencils& st = c.st;
  const int N = c.N, D = c.dim, NI = c.NI, H = NI / 2, F = c.F;
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    d.has_tab = false;
    if (d.nb > kSmallLevel || d.has_cf || !st.valid) continue;
    std::vector<int32_t> tab((size_t)d.nb * NI * 8, 0);
    std::vector<double> gbc((size_t)d.nb * NI * 6, 0.0);
    int base = 0;
    for (int s = 0; s < d.nb; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      const bool bnd = st.boundary[(size_t)id] != 0;
      const int r0 = bnd ? st.row_start[(size_t)id] : 0;
      const int leaf = m.children[(size_t)id * 8] < 0 ? 1 : 0;
      for (int ii = 0; ii < NI; ++ii) {
        const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
        const size_t a = (size_t)s * NI + (size_t)cs_addr(ii, N, D, H);
        int32_t* e = tab.data() + a * 8;
        int code = -1;
        if (bnd) {
          const int r = st.row_at((size_t)id, (size_t)ii);
          if (r < 0) code = -2;
          else if (st.mask[(size_t)(r0 + r)] == PMG_INSIDE) code = -3 - (base + r);
          else code = base + r;
        }
        e[0] = code;
        e[7] = leaf;
        for (int f = 0; f < F; ++f) {
          const int ax = f / 2, sg = (f & 1) ? 1 : -1;
          int q[3] = {i, j, k};
          q[ax] += sg;
          if (q[ax] >= 0 && q[ax] < N) {
            e[1 + f] = (int32_t)((size_t)s * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
            continue;
          }
          const int nid = m.nbr[(size_t)id * 6 + f];
          if (nid >= 0) {
            q[ax] = sg > 0 ? 0 : N - 1;
            e[1 + f] = (int32_t)((size_t)m.slot_of[(size_t)nid] * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
            continue;
          }
          if (c.bctype[f] == PMG_BC_NEUMANN_ZERO) {
            e[1 + f] = -1;
            continue;
          }
          e[1 + f] = -2;
          if (!c.face_off[f].empty() && c.face_off[f][(size_t)id] >= 0) {
            const int t = D == 2 ? (ax == 0 ? j : i) : (ax == 0 ? j + N * k : ax == 1 ? i + N * k : i + N * j);
            gbc[a * 6 + f] = c.face_vals[f][(size_t)c.face_off[f][(size_t)id] + t];
          }
        }
      }
      if (bnd) base += st.row_count[(size_t)id];
    }
    d.tab.upload(tab, c.stream);
    d.tgbc.upload(gbc, c.stream);
    d.has_tab = true;
  }
}

// One cell's gather entry (small.cuh / stream.cuh fix kernels): e[0] row code
// (r >= 0 special row r in the level's row arrays, -1 uniform row of a
// uniform block, -2 uniform row of an interface block, -3 - r inside row r),
// e[1..2D] the neighbour value addresses (same block or same-level
// neighbour), -1 Neumann ghost f1, -2 Dirichlet ghost 2 bc - f1 with bc in gb.
// `base` is the block's first row in the level's row arrays.  Blocks with a
// coarse-fine face are not supported (callers exclude them).
static void cell_entry(const Ctx& c, int s, int id, int ii, int base, int32_t* e, double* gb) {
  const HostMesh& m = c.mesh;
  const HostStencils& st = c.st;
  const int N = c.N, D = c.dim, NI = c.NI, H = NI / 2, F = c.F;
  const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
  int code = -1;
  if (st.valid && st.boundary[(size_t)id]) {
    const int r = st.row_at((size_t)id, (size_t)ii);
    if (r < 0) code = -2;
    else if (st.mask[(size_t)(st.row_start[(size_t)id] + r)] == PMG_INSIDE) code = -3 - (base + r);
    else code = base + r;
  }
  e[0] = code;
  for (int f = 0; f < 6; ++f) gb[f] = 0.0;
  for (int f = 0; f < F; ++f) {
    const int ax = f / 2, sg = (f & 1) ? 1 : -1;
    int q[3] = {i, j, k};
    q[ax] += sg;
    if (q[ax] >= 0 && q[ax] < N) {
      e[1 + f] = (int32_t)((size_t)s * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
      continue;
    }
    const int nid = m.nbr[(size_t)id * 6 + f];
    if (nid >= 0) {
      q[ax] = sg > 0 ? 0 : N - 1;
      e[1 + f] = (int32_t)((size_t)m.slot_of[(size_t)nid] * NI + cs_addr(q[0] + N * (q[1] + N * q[2]), N, D, H));
      continue;
    }
    require(m.cnbr[(size_t)id * 6 + f] < 0, "gather entry next to a coarse-fine face", PMG_ERR_STATE);
    if (c.bctype[f] == PMG_BC_NEUMANN_ZERO) {
      e[1 + f] = -1;
      continue;
    }
    e[1 + f] = -2;
    if (!c.face_off[f].empty() && c.face_off[f][(size_t)id] >= 0) {
      const int t = D == 2 ? (ax == 0 ? j : i) : (ax == 0 ? j + N * k : ax == 1 ? i + N * k : i + N * j);
      gb[f] = c.face_vals[f][(size_t)c.face_off[f][(size_t)id] + t];
    }
  }
}

// Per level, per stencil row: center, nb[2D], each cut direction's bc * phi_b
// product (formed exactly as the reference forms it, stencil.hpp:344-358), the
// cut-direction mask, an inside flag -- 16 doubles, one 128-B line.
static void build_row_coef(Ctx& c) {
  for (int l = 1; l <= c.mesh.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    const int R = (int)d.n_rows;
    d.r_coef.alloc((size_t)std::max(R, 1) * 16);
    if (R > 0)
      pdl_launch(pmgdev::k_row_coef, (unsigned)((R + 255) / 256), 256, 0, c.stream, R, c.F,
                 (const double*)d.r_center.p, (const double*)d.r_nb.p, (const double*)d.r_bc.p,
                 (const int8_t*)d.r_obj.p, (const uint8_t*)d.r_mask.p, (const double*)c.phi_b.p, d.r_coef.p);
    PMG_CUDA(cudaGetLastError());
  }
}

// k_restrict_fix tables: per listed parent, the gather entries of its 2^D
// children (e[7] = the child's address), in child order.
static void build_rfix_tables(Ctx& c) {
  const HostMesh& m = c.mesh;
  const int N = c.N, NI = c.NI, H = NI / 2, HN = N / 2;
  if (c.dim != 3) return;
  for (int l = 2; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    const std::vector<int32_t>& host_list = d.rfix_host;
    std::vector<int32_t> tab((size_t)d.n_rfix * 8 * 8);
    std::vector<double> gbc((size_t)d.n_rfix * 8 * 6);
    std::vector<int> base((size_t)d.nb, 0);
    int acc = 0;
    for (int s = 0; s < d.nb; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      base[(size_t)s] = acc;
      if (c.st.valid && c.st.boundary[(size_t)id]) acc += c.st.row_count[(size_t)id];
    }
    for (int q = 0; q < d.n_rfix; ++q) {
      const int s = host_list[(size_t)2 * q], t = host_list[(size_t)2 * q + 1];
      const int id = m.slots[(size_t)l][(size_t)s];
      const int ii = t % HN, jj = (t / HN) % HN, kk = t / (HN * HN);
      for (int ch = 0; ch < 8; ++ch) {
        const int ci = (2 * ii + (ch & 1)) + N * ((2 * jj + ((ch >> 1) & 1)) + N * (2 * kk + (ch >> 2)));
        int32_t* e = tab.data() + ((size_t)q * 8 + ch) * 8;
        cell_entry(c, s, id, ci, base[(size_t)s], e, gbc.data() + ((size_t)q * 8 + ch) * 6);
        e[7] = (int32_t)((size_t)s * NI + cs_addr(ci, N, c.dim, H));
      }
    }
    d.rfix_tab.upload(tab, c.stream);
    d.rfix_gbc.upload(gbc, c.stream);
  }
}

// The StencilSet's rows on the device (block-id order, StencilSet row
// numbering; row_of pages in row_page order): kept from the device build, or
// uploaded once from a host StencilSet (set_stencils).
static void ensure_devrows(Ctx& c) {
  if (c.devrows) return;
  const HostStencils& st = c.st;
  auto R = std::make_unique<DevRows>();
  const size_t nr = st.center.size(), F = (size_t)c.F;
  R->center.upload(st.center, c.stream);
  R->nb.upload(st.nb, c.stream);
  R->bc.upload(st.bc, c.stream);
  if (st.d.size() == nr * F) R->d.upload(st.d, c.stream);
  else R->d.upload(std::vector<double>(nr * F, 1.0), c.stream);
  R->obj.upload(st.obj, c.stream);
  R->mask.upload(st.mask, c.stream);
  R->pin.upload(st.pin, c.stream);
  R->rowof.upload(st.row_pages, c.stream);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
  c.devrows = std::move(R);
}

static void upload_stencils(Ctx& c) {
  const HostMesh& m = c.mesh;
  const HostStencils& st = c.st;
  const int NI = c.NI, H = NI / 2, F = c.F;
  std::vector<std::vector<uint8_t>> kindv((size_t)m.L + 1);
  std::vector<int32_t> cs_perm((size_t)NI);  // interior index -> colour-split entry
  for (int ii = 0; ii < NI; ++ii) cs_perm[(size_t)ii] = cs_addr(ii, c.N, c.dim, H);
  ensure_devrows(c);
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    std::vector<int32_t> srow((size_t)d.nb, -1);
    std::vector<uint8_t> kind((size_t)d.nb, pmgdev::KIND_UNIFORM);
    std::vector<int4> rlist;  // per interface block in slot order: StencilSet page, first row, level row, count
    int n_if = 0, base = 0;
    for (int s = 0; s < d.nb; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      if (!st.valid || !st.boundary[(size_t)id]) continue;
      srow[(size_t)s] = n_if++;
      const int r0 = st.row_start[(size_t)id];
      const int rc = st.row_count[(size_t)id];
      bool all_inside = rc == NI;
      for (int r = 0; r < rc && all_inside; ++r) all_inside = st.mask[(size_t)(r0 + r)] == PMG_INSIDE;
      kind[(size_t)s] = all_inside ? pmgdev::KIND_ALL_INSIDE : pmgdev::KIND_IFACE;
      rlist.push_back(make_int4(st.row_page[(size_t)id], r0, base, rc));
      base += rc;
    }
    // the level's rows, row_of pages (colour-split, level row numbers) and
    // special-row kinds, gathered on the device from the StencilSet's rows
    d.n_rows = (size_t)base;
    const size_t R1 = (size_t)std::max(base, 1);
    d.r_center.alloc(R1);
    d.r_mask.alloc(R1);
    d.r_pin.alloc(R1);
    d.r_nb.alloc(R1 * F);
    d.r_bc.alloc(R1 * F);
    d.r_d.alloc(R1 * F);
    d.r_obj.alloc(R1 * F);
    d.row_of.alloc((size_t)std::max(n_if, 1) * NI);
    d.skind.alloc((size_t)std::max(n_if, 1) * NI);
    if (n_if > 0) {
      DevBuf<int4> dl;
      dl.upload(rlist, c.stream);
      const DevRows& R = *c.devrows;
      pdl_launch(pmgdev::k_level_rows, (unsigned)n_if, 256, 0, c.stream, (const int4*)dl.p, c.N, c.dim, F,
                 (const int32_t*)R.rowof.p, (const double*)R.center.p, (const double*)R.nb.p, (const double*)R.bc.p,
                 (const double*)R.d.p, (const int8_t*)R.obj.p, (const uint8_t*)R.mask.p, (const int8_t*)R.pin.p,
                 d.row_of.p, d.skind.p, d.r_center.p, d.r_nb.p, d.r_bc.p, d.r_d.p, d.r_obj.p, d.r_mask.p,
                 d.r_pin.p);
      PMG_CUDA(cudaStreamSynchronize(c.stream));  // dl
    }
    d.srow.upload(srow, c.stream);
    d.kind.upload(kind, c.stream);
    kindv[(size_t)l] = kind;
    // block classes for the specialised kernels
    {
      std::vector<int32_t> fast, slow, ufast, uslow, fix[2], gsl, rsl, url, gslow, rcl, rcslow, rrl, rrslow;
      d.gs_cf = false;
      for (int s = 0; s < d.nb; ++s) {
        if (!own_slot(c, l, s)) continue;
        const int id = m.slots[(size_t)l][(size_t)s];
        bool no_cf = true;  // lean kernels handle same-level and physical faces
        for (int f = 0; f < F; ++f)
          no_cf = no_cf && !(m.nbr[(size_t)id * 6 + f] < 0 && m.cnbr[(size_t)id * 6 + f] >= 0);
        (no_cf ? fast : slow).push_back(s);
        if (stream_dn(c)) {  // restriction plan: every block (all-inside ones restrict exactly in-stream)
          if (no_cf || cf_streamable(c, id)) {
            int pm = 0;
            int32_t ns[6] = {-1, -1, -1, -1, -1, -1};
            for (int f = 0; f < F; ++f) {
              const int nid = m.nbr[(size_t)id * 6 + f];
              if (nid >= 0) ns[f] = m.slot_of[(size_t)nid];
              else if (m.cnbr[(size_t)id * 6 + f] >= 0) ns[f] = -2 - d.cfoff_host[(size_t)s * F + f] / c.NT;
              else pm |= 1 << f;
            }
            const int sr = srow[(size_t)s] < 0 ? 0 : srow[(size_t)s];
            require(sr < (1 << 17), "too many interface blocks on one level for the streaming plan");
            const int32_t e[8] = {s, (int32_t)kind[(size_t)s] | (pm << 8) | (sr << 14), ns[0], ns[1], ns[2], ns[3], ns[4], ns[5]};
            rrl.insert(rrl.end(), e, e + 8);
          } else {
            rrslow.push_back(s);
          }
        }
        if (!no_cf && stream_dn(c)) {
          // coarse-fine faces: streamed with the faces' cfc pages as neighbour
          // codes -2 - page (stream.cuh BlockPlan), unless a cut row sits near one (cf_streamable)
          if (kind[(size_t)s] == pmgdev::KIND_ALL_INSIDE) {
            // nothing to sweep
          } else if (cf_streamable(c, id)) {
            int pm = 0;
            int32_t ns[6] = {-1, -1, -1, -1, -1, -1};
            for (int f = 0; f < F; ++f) {
              const int nid = m.nbr[(size_t)id * 6 + f];
              if (nid >= 0) ns[f] = m.slot_of[(size_t)nid];
              else if (m.cnbr[(size_t)id * 6 + f] >= 0) ns[f] = -2 - d.cfoff_host[(size_t)s * F + f] / c.NT;
              else pm |= 1 << f;
            }
            const int sr = srow[(size_t)s] < 0 ? 0 : srow[(size_t)s];
            require(sr < (1 << 17), "too many interface blocks on one level for the streaming plan");
            const int32_t e[8] = {s, (int32_t)kind[(size_t)s] | (pm << 8) | (sr << 14), ns[0], ns[1], ns[2], ns[3], ns[4], ns[5]};
            gsl.insert(gsl.end(), e, e + 8);
            d.gs_cf = true;
            if (m.children[(size_t)id * 8] < 0) rcl.insert(rcl.end(), e, e + 8);
          } else {
            gslow.push_back(s);
            if (m.children[(size_t)id * 8] < 0) rcslow.push_back(s);
          }
        }
        if (no_cf) {
          // stream.cuh BlockPlan: slot, kind | phys << 8 | srow << 14, 6 neighbour slots
          int pm = 0;
          int32_t ns[6] = {-1, -1, -1, -1, -1, -1};
          for (int f = 0; f < F; ++f) {
            const int nid = m.nbr[(size_t)id * 6 + f];
            if (nid < 0) pm |= 1 << f;
            else ns[f] = m.slot_of[(size_t)nid];
          }
          const int sr = srow[(size_t)s] < 0 ? 0 : srow[(size_t)s];
          require(sr < (1 << 17), "too many interface blocks on one level for the streaming plan");
          const int32_t e[8] = {s, (int32_t)kind[(size_t)s] | (pm << 8) | (sr << 14), ns[0], ns[1], ns[2], ns[3], ns[4], ns[5]};
          rsl.insert(rsl.end(), e, e + 8);
          if (kind[(size_t)s] == pmgdev::KIND_UNIFORM) url.insert(url.end(), e, e + 8);
          if (kind[(size_t)s] != pmgdev::KIND_ALL_INSIDE) gsl.insert(gsl.end(), e, e + 8);
          if (kind[(size_t)s] != pmgdev::KIND_ALL_INSIDE && m.children[(size_t)id * 8] < 0) rcl.insert(rcl.end(), e, e + 8);
        }
        (no_cf && kind[(size_t)s] == pmgdev::KIND_UNIFORM ? ufast : uslow).push_back(s);
        // cut (non-inside) rows of lean interface blocks, per colour, for k_gs_fix
        if (no_cf && kind[(size_t)s] == pmgdev::KIND_IFACE) {
          const int32_t* page = st.page((size_t)id);
          const int r0 = st.row_start[(size_t)id];
          for (int ii = 0; ii < NI; ++ii) {
            const int32_t r = page[ii];
            if (r >= 0 && st.mask[(size_t)(r0 + r)] != PMG_INSIDE) {
              const int a = cs_perm[(size_t)ii];
              fix[a / H].push_back(s), fix[a / H].push_back(a % H);
            }
          }
        }
      }
      d.n_gs = (int)gsl.size() / 8;
      d.coop = -1;
      d.gs_plan.upload(gsl, c.stream);
      d.n_rs = (int)rsl.size() / 8;
      d.rs_plan.upload(rsl, c.stream);
      d.n_ur = (int)url.size() / 8;
      d.ur_plan.upload(url, c.stream);
      d.n_fast = (int)fast.size();
      d.n_slow = (int)slow.size();
      d.fast_list.upload(fast, c.stream);
      d.slow_list.upload(slow, c.stream);
      d.n_gs_slow = (int)gslow.size();
      d.gs_slow.upload(gslow, c.stream);
      d.n_rc = (int)rcl.size() / 8;
      d.rc_plan.upload(rcl, c.stream);
      d.n_rc_slow = (int)rcslow.size();
      d.rc_slow.upload(rcslow, c.stream);
      d.n_rr = (int)rrl.size() / 8;
      d.rr_plan.upload(rrl, c.stream);
      d.n_rr_slow = (int)rrslow.size();
      d.rr_slow.upload(rrslow, c.stream);
      d.n_ufast = (int)ufast.size();
      d.n_uslow = (int)uslow.size();
      d.ufast_list.upload(ufast, c.stream);
      d.uslow_list.upload(uslow, c.stream);
      for (int cc = 0; cc < 2; ++cc) {
        d.n_fix[cc] = (int)fix[cc].size() / 2;
        d.fix_list[cc].upload(fix[cc], c.stream);
      }
    }
  }
  // k_restrict_fix lists (3D): parents of level l-1 whose fused restriction
  // needs the general path -- a child with a special row, or a pinned parent
  if (c.dim == 3) {
    const int N = c.N, HN = N / 2;
    auto row_at = [&](int id, int i, int j, int k) -> int {
      if (!st.valid || !st.boundary[(size_t)id]) return -1;
      const int r = st.row_at((size_t)id, (size_t)(i + N * (j + N * k)));
      return r < 0 ? -1 : st.row_start[(size_t)id] + r;
    };
    for (int l = 2; l <= m.L; ++l) {
      LevelDev& d = *c.lev[(size_t)l];
      std::vector<int32_t> fx;
      for (int s = 0; s < d.nb; ++s) {
        if (!own_slot(c, l, s)) continue;
        const int id = m.slots[(size_t)l][(size_t)s];
        const int p = m.parent[(size_t)id];
        const int cx = m.coords[(size_t)id * 3] & 1, cy = m.coords[(size_t)id * 3 + 1] & 1,
                  cz = m.coords[(size_t)id * 3 + 2] & 1;
        (void)p;
        (void)cx;
        (void)cy;
        (void)cz;
        // interface blocks only: all-inside blocks restrict exactly in the stream kernel
        if (!(st.valid && st.boundary[(size_t)id]) || kindv[(size_t)l][(size_t)s] != pmgdev::KIND_IFACE) continue;
        if (has_cf_face(c, id) && !cf_streamable(c, id)) continue;  // restricted by k_restrict_tile
        for (int t = 0; t < HN * HN * HN; ++t) {
          const int ii = t % HN, jj = (t / HN) % HN, kk = t / (HN * HN);
          bool need = false;
          for (int ch = 0; ch < 8 && !need; ++ch) {  // a cut child (inside children restrict exactly in-stream)
            const int r = row_at(id, 2 * ii + (ch & 1), 2 * jj + ((ch >> 1) & 1), 2 * kk + (ch >> 2));
            need = r >= 0 && st.mask[(size_t)r] != PMG_INSIDE;
          }
          if (need) fx.push_back(s), fx.push_back(t);
        }
      }
      d.n_rfix = (int)fx.size() / 2;
      d.rfix_list.upload(fx, c.stream);
      d.rfix_host = fx;
    }
  }
  // streaming prolongation plans (3D): fine blocks that are not entirely
  // inside; eligible when no parent octant face is a coarse-fine face
  if (c.dim == 3) {
    for (int l = 2; l <= m.L; ++l) {
      LevelDev& d = *c.lev[(size_t)l];
      std::vector<int32_t> pp;
      bool ok = true;
      d.pp_cf = false;
      const LevelDev& dpar = *c.lev[(size_t)(l - 1)];
      for (int s = 0; s < d.nb && ok; ++s) {
        if (kindv[(size_t)l][(size_t)s] == pmgdev::KIND_ALL_INSIDE || !own_slot(c, l, s)) continue;
        const int id = m.slots[(size_t)l][(size_t)s];
        const int pid = m.parent[(size_t)id];
        int oct = 0, pn[3];
        for (int ax = 0; ax < 3; ++ax) {
          const int cb = m.coords[(size_t)id * 3 + ax] & 1;
          oct |= cb << ax;
          const int dir = 2 * ax + cb;
          const int nid = m.nbr[(size_t)pid * 6 + dir];
          if (nid >= 0) pn[ax] = m.slot_of[(size_t)nid];
          else if (m.cnbr[(size_t)pid * 6 + dir] >= 0) {
            // the parent's face is coarse-fine: its cfc / cfold page (3D N = 8 / 16 kernels only)
            if (stream_dn(c)) {
              pn[ax] = -2 - dpar.cfoff_host[(size_t)m.slot_of[(size_t)pid] * F + dir] / c.NT;
              d.pp_cf = true;
            } else {
              ok = false;
            }
          }
          else pn[ax] = -1;
        }
        int edge = 0;  // a face of the fine block without a same-level neighbour
        for (int dir = 0; dir < 6; ++dir) edge |= m.nbr[(size_t)id * 6 + dir] < 0;
        const int32_t e[8] = {s, m.slot_of[(size_t)pid], oct, pn[0], pn[1], pn[2], kindv[(size_t)l][(size_t)s], edge};
        pp.insert(pp.end(), e, e + 8);
      }
      d.n_pp = ok ? (int)pp.size() / 8 : -1;
      if (!ok) pp.clear();
      d.pp_plan.upload(pp, c.stream);
    }
  }
  // pin lists (every level): colour-split address and object of each inside row
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    std::vector<int32_t> pl;
    if (st.valid)
      for (int s = 0; s < d.nb; ++s) {
        const int id = m.slots[(size_t)l][(size_t)s];
        if (!st.boundary[(size_t)id] || !own_slot(c, l, s)) continue;
        for (int ii = 0; ii < NI; ++ii) {
          const int r = st.row_at((size_t)id, (size_t)ii);
          if (r < 0) continue;
          const size_t q = (size_t)(st.row_start[(size_t)id] + r);
          if (st.mask[q] != PMG_INSIDE) continue;
          pl.push_back((int32_t)((size_t)s * NI + (size_t)cs_addr(ii, c.N, c.dim, H)));
          pl.push_back(st.pin[q]);
        }
      }
    d.n_pin = (int)pl.size() / 2;
    d.pin_list.upload(pl, c.stream);
  }
  std::vector<double> pb = st.phi_b;
  if (pb.empty()) pb.push_back(0.0);
  c.phi_b.upload(pb, c.stream);
  build_cut_tables(c);
  build_small_tables(c);
  build_row_coef(c);
  build_rfix_tables(c);
}

static void default_stencils(Ctx& c) {
  HostStencils& st = c.st;
  st = HostStencils{};
  st.valid = true;
  st.boundary.assign((size_t)c.mesh.nb, 0);
  st.row_count.assign((size_t)c.mesh.nb, 0);
  st.row_start.assign((size_t)c.mesh.nb + 1, 0);
  st.NI = c.NI;
  st.row_page.assign((size_t)c.mesh.nb, -1);
  st.row_pages.clear();
  c.devrows.reset();
}

// ---------------------------------------------------------------- coarse assembly
// Restates assemble_level(mesh, set, 1) (multigrid.hpp:62-190) for the single
// root block of level 1: unknowns = non-inside cells in x-fastest order,
// physical faces folded into diag / c0, pinned neighbours and cut directions
// into cobj, rows sorted by column.
static void assemble_coarse(Ctx& c) {
  const HostMesh& m = c.mesh;
  const HostStencils& st = c.st;
  const int N = c.N, D = c.dim, NI = c.NI, F = c.F, H = NI / 2;
  const int id = m.slots[1][0];
  const int n_obj = (int)st.phi_b.size();
  HostCoarse& cs = c.coarse;
  cs = HostCoarse{};
  std::vector<int> unk((size_t)NI, -1);
  const bool bnd = st.boundary[(size_t)id] != 0;
  const int r0 = st.row_start[(size_t)id];
  auto row_ptr = [&](int ii) -> int {
    if (!bnd) return -1;
    const int r = st.row_at((size_t)id, (size_t)ii);
    return r < 0 ? -1 : r0 + r;
  };
  auto inside = [&](int ii) {
    const int r = row_ptr(ii);
    return r >= 0 && st.mask[(size_t)r] == PMG_INSIDE;
  };
  const int s1 = N + 2;
  auto lin = [&](int i, int j, int k) { return (i + 1) + (j + 1) * s1 + (D == 3 ? (k + 1) * s1 * s1 : 0); };
  for (int ii = 0; ii < NI; ++ii) {
    if (inside(ii)) continue;
    unk[(size_t)ii] = cs.n++;
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    cs.unk_block.push_back(id);
    cs.unk_lin.push_back(lin(i, j, k));
    cs.uaddr.push_back(cs_addr(ii, N, D, H));  // slot 0
  }
  cs.c0.assign((size_t)cs.n, 0.0);
  cs.cobj.assign((size_t)n_obj * cs.n, 0.0);
  std::vector<std::vector<std::pair<int, double>>> rows((size_t)cs.n);
  const double bdx = m.dx[(size_t)id];
  const double w = 1.0 / (bdx * bdx);
  for (int ii = 0; ii < NI; ++ii) {
    const int row = unk[(size_t)ii];
    if (row < 0) continue;
    const int ic[3] = {ii % N, (ii / N) % N, D == 3 ? ii / (N * N) : 0};
    double diag;
    double an[6];
    const int rp = row_ptr(ii);
    if (rp >= 0) {
      diag = st.center[(size_t)rp];
      for (int f = 0; f < F; ++f) {
        an[f] = st.nb[(size_t)rp * F + f];
        const double b = st.bc[(size_t)rp * F + f];
        if (b != 0) cs.cobj[(size_t)st.obj[(size_t)rp * F + f] * cs.n + row] -= b;
      }
    } else {
      diag = -2.0 * D * w;
      for (int f = 0; f < F; ++f) an[f] = w;
    }
    auto& r = rows[(size_t)row];
    for (int f = 0; f < F; ++f) {
      const double a = an[f];
      if (a == 0) continue;
      const int axis = f >> 1, sgn = (f & 1) ? 1 : -1;
      int ni[3] = {ic[0], ic[1], ic[2]};
      ni[axis] += sgn;
      if (ni[axis] < 0 || ni[axis] >= N) {
        // level 1 is the root block: every face is physical (mesh.hpp:455)
        if (c.bctype[f] == PMG_BC_NEUMANN_ZERO) {
          diag += a;
        } else {
          diag -= a;
          double bcv = 0.0;
          if (!c.face_off[f].empty() && c.face_off[f][(size_t)id] >= 0) {
            int t;
            if (D == 2) t = axis == 0 ? ic[1] : ic[0];
            else t = axis == 0 ? ic[1] + N * ic[2] : (axis == 1 ? ic[0] + N * ic[2] : ic[0] + N * ic[1]);
            bcv = c.face_vals[f][(size_t)c.face_off[f][(size_t)id] + t];
          }
          cs.c0[(size_t)row] -= 2.0 * a * bcv;
        }
        continue;
      }
      const int nii = ni[0] + N * (ni[1] + N * ni[2]);
      const int col = unk[(size_t)nii];
      if (col < 0) {
        const int po = st.pin[(size_t)row_ptr(nii)];
        cs.cobj[(size_t)po * cs.n + row] -= a;
        continue;
      }
      r.emplace_back(col, a);
    }
    r.emplace_back(row, diag);
  }
  cs.rp.assign((size_t)cs.n + 1, 0);
  for (int r = 0; r < cs.n; ++r) {
    auto& row = rows[(size_t)r];
    std::sort(row.begin(), row.end());
    cs.rp[(size_t)r + 1] = cs.rp[(size_t)r] + (int)row.size();
    for (auto& [col, v] : row) {
      cs.ci.push_back(col);
      cs.val.push_back(v);
    }
  }
  // Jacobi preconditioner (multigrid.hpp:213-217)
  cs.dinv.assign((size_t)cs.n, 1.0);
  for (int r = 0; r < cs.n; ++r)
    for (int q = cs.rp[(size_t)r]; q < cs.rp[(size_t)r + 1]; ++q)
      if (cs.ci[(size_t)q] == r && cs.val[(size_t)q] != 0) cs.dinv[(size_t)r] = 1.0 / cs.val[(size_t)q];
  c.c_rp.upload(cs.rp, c.stream);
  c.c_ci.upload(cs.ci, c.stream);
  c.c_val.upload(cs.val, c.stream);
  c.c_dinv.upload(cs.dinv, c.stream);
  c.c_c0.upload(cs.c0, c.stream);
  c.c_cobj.upload(cs.cobj, c.stream);
  c.c_uaddr.upload(cs.uaddr, c.stream);
  c.c_scratch.alloc((size_t)10 * std::max(cs.n, 1));

  // cell-indexed form for the on-chip solver (coarse.cuh): per cell the diagonal,
  // a mask of neighbours whose coefficient is w, or an explicit special row
  std::vector<uint8_t> fl((size_t)NI, 0);
  std::vector<double> dg((size_t)NI, 0.0), c0c((size_t)NI, 0.0), spc, obv;
  std::vector<int16_t> sp((size_t)NI, -1);
  std::vector<int32_t> obs((size_t)NI + 1, 0);
  std::vector<int8_t> obo;
  const int offs[6] = {-1, 1, -N, N, -N * N, N * N};
  std::vector<int> cell_of_unk((size_t)cs.n);
  for (int ii = 0; ii < NI; ++ii)
    if (unk[(size_t)ii] >= 0) cell_of_unk[(size_t)unk[(size_t)ii]] = ii;
  for (int u = 0; u < cs.n; ++u) {
    const int ii = cell_of_unk[(size_t)u];
    double coef[6] = {0, 0, 0, 0, 0, 0};
    bool special = false;
    for (int q = cs.rp[(size_t)u]; q < cs.rp[(size_t)u + 1]; ++q) {
      const int col = cs.ci[(size_t)q];
      if (col == u) {
        dg[(size_t)ii] = cs.val[(size_t)q];
        continue;
      }
      const int dj = cell_of_unk[(size_t)col] - ii;
      int dir = -1;
      for (int f = 0; f < F; ++f)
        if (offs[f] == dj) dir = f;
      require(dir >= 0, "coarse operator is not a face stencil");
      coef[dir] = cs.val[(size_t)q];
      if (coef[dir] != w) special = true;
    }
    uint8_t f8 = 0x40;
    if (special) {
      f8 |= 0x80;
      sp[(size_t)ii] = (int16_t)(spc.size() / F);
      for (int f = 0; f < F; ++f) spc.push_back(coef[f]);
    } else {
      for (int f = 0; f < F; ++f)
        if (coef[f] != 0) f8 |= (uint8_t)(1u << f);
    }
    fl[(size_t)ii] = f8;
    c0c[(size_t)ii] = cs.c0[(size_t)u];
  }
  for (int ii = 0; ii < NI; ++ii) {
    obs[(size_t)ii + 1] = obs[(size_t)ii];
    const int u = unk[(size_t)ii];
    if (u < 0) continue;
    for (int o = 0; o < n_obj; ++o) {
      const double v = cs.cobj[(size_t)o * cs.n + u];
      if (v == 0) continue;
      obo.push_back((int8_t)o);
      obv.push_back(v);
      obs[(size_t)ii + 1]++;
    }
  }
  require(spc.size() / std::max(F, 1) < 32767, "too many special coarse rows");
  c.cf_flags.upload(fl, c.stream);
  c.cf_diag.upload(dg, c.stream);
  c.cf_spec.upload(sp, c.stream);
  c.cf_spec_c.upload(spc, c.stream);
  c.cf_c0.upload(c0c, c.stream);
  c.cf_ob_start.upload(obs, c.stream);
  c.cf_ob_obj.upload(obo, c.stream);
  c.cf_ob_val.upload(obv, c.stream);
  c.cf_w = w;
}

// ---------------------------------------------------------------- cycle sequences
// residual_level(l) + restrict_level(l) up to apply_pins(l-1): one pass unless
// level l has coarse-fine faces (their ghosts read level l-1 cells being restricted)
static void enq_restrict_only(Ctx& c, int l) {
  if (c.lev[(size_t)l]->has_cf && !c.ops->cf_table()) {
    c.ops->residual(c, l);
    c.ops->restrict_(c, l, pmgdev::RM_RES);
  } else {
    c.ops->restrict_(c, l, pmgdev::RM_FUSED);
  }
}
// the rest of restrict_level(l): the FAS right-hand side and OLD of level l-1
static void enq_fas_level(Ctx& c, int l) { c.ops->fas_cfold(c, l - 1, true); }
static void enq_restrict_level(Ctx& c, int l) {
  enq_restrict_only(c, l);
  enq_fas_level(c, l);
}
static void enq_restrict_level_no_guess(Ctx& c, int l) {
  c.ops->restrict_(c, l, pmgdev::RM_RHS);
  c.ops->fas_cfold(c, l - 1, false);
}
static void enq_smooth(Ctx& c, int l, int steps) {
  if (c.ops->smooth(c, l, steps)) return;  // one cooperative launch (coop.cuh)
  for (int s = 0; s < steps; ++s) {
    c.ops->gs(c, l, 0);
    c.ops->gs(c, l, 1);
  }
}
static void enq_coarse(Ctx& c) { c.ops->coarse(c); }
static void enq_v_span(Ctx& c, int top) {
  if (top == 1) {
    enq_coarse(c);
    return;
  }
  for (int l = top; l >= 2; --l) {
    enq_smooth(c, l, c.cfg.n_down);
    enq_restrict_level(c, l);
  }
  enq_coarse(c);
  for (int l = 2; l <= top; ++l) {
    // the red half-sweep that follows overwrites every red cell the
    // prolongation would write, except where a physical-face ghost reads it
    c.prolong_dead = c.cfg.n_up > 0 ? 0 : -1;
    c.ops->prolong(c, l, false);
    c.prolong_dead = -1;
    enq_smooth(c, l, c.cfg.n_up);
    c.ops->record(c, l);
  }
}
static void enq_reset_records(Ctx& c) {
  PMG_CUDA(cudaMemsetAsync(c.rec.p, 0, c.rec.n * sizeof(pmgdev::Rec), c.stream));
}
// stats, diag and status to the host in one copy (Ctx::outbuf)
static void enq_copy_out(Ctx& c) {
  PMG_CUDA(cudaMemcpyAsync(c.h_out, c.outbuf.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
}
static void enq_finish(Ctx& c) {
  if (c.finished) {  // the last record wrote the stats and the host copy (ops record)
    c.finished = false;
    return;
  }
  pdl_launch(pmgdev::k_combine, 1, 32, 0, c.stream, c.rec.p, c.mesh.L, c.stats.p);
  PMG_CUDA(cudaGetLastError());
  enq_copy_out(c);
}
static void enq_clear_status(Ctx& c) {
  PMG_CUDA(cudaMemsetAsync(c.status.p, 0, sizeof(int), c.stream));
}
// status and the level records, adjacent in Ctx::outbuf: one memset
static void enq_clear_cycle(Ctx& c) {
  PMG_CUDA(cudaMemsetAsync(c.status.p, 0, sizeof(double) + c.rec.n * sizeof(pmgdev::Rec), c.stream));
}

enum CycleKind { CK_V = 0, CK_FMG_NOGUESS = 1, CK_FMG_GUESS = 2, CK_MEASURE = 3 };

static void enq_cycle(Ctx& c, int kind) {
  const int L = c.mesh.L;
  enq_clear_cycle(c);
  c.finished = false;
  if (kind == CK_V) {
    c.finish_level = L;
    enq_v_span(c, L);
    c.finish_level = 0;
  } else if (kind == CK_MEASURE) {
    for (int l = 1; l <= L; ++l) c.ops->record(c, l);
  } else {
    const bool guess = kind == CK_FMG_GUESS;
    for (int l = L; l >= 2; --l) {
      if (guess) enq_restrict_level(c, l);
      else enq_restrict_level_no_guess(c, l);
    }
    enq_coarse(c);
    for (int l = 2; l <= L; ++l) {
      c.ops->prolong(c, l, !guess);
      c.finish_level = l == L ? L : 0;
      enq_v_span(c, l);
      c.finish_level = 0;
    }
  }
  enq_finish(c);
}

static Graph& graph_for(Ctx& c, int kind) {
  Graph& g = kind == CK_V ? c.g_v : kind == CK_MEASURE ? c.g_measure : c.g_fmg[kind == CK_FMG_GUESS];
  if (g.exec) return g;
  cudaGraph_t graph;
  cfc_all_dirty(c);  // a replay may start from any state: the graph rebuilds the cfc tables it reads
  PMG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    enq_cycle(c, kind);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  PMG_CUDA(cudaStreamEndCapture(c.stream, &graph));
  cfc_all_dirty(c);  // nothing was executed
  size_t nn = 0;
  PMG_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  PMG_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
  int kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    PMG_CUDA(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel) ++kernels;
  }
  PMG_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
  cudaGraphDestroy(graph);
  g.kernels = kernels;
  return g;
}

static void launch_cycle(Ctx& c, int kind) {
  require(c.solver, "solver not created (call pmg_b200_solver_create)", PMG_ERR_STATE);
  Graph& g = graph_for(c, kind);
  PMG_CUDA(cudaGraphLaunch(g.exec, c.stream));
  if (kind != CK_MEASURE) c.have_guess = true;
}

static void cycle_result(Ctx& c, pmg_cycle_stats_t* out) {
  PMG_CUDA(cudaStreamSynchronize(c.stream));
  const int st = *c.h_status;
  if (st == 3) {
    char buf[64];
    const std::string rel = std::to_string(c.h_out[2]);
    (void)buf;
    throw PmgError(PMG_ERR_COARSE_STALL,
                   "coarse solve failed: BiCGStab stalled at relative residual " + rel +
                       " after " + std::to_string((int)c.h_out[3]) + " iterations on " +
                       std::to_string(c.coarse.n) + " unknowns");
  }
  if (st == 4) throw PmgError(PMG_ERR_COARSE_STALL, "coarse solve failed: smoothing fallback stalled");
  if (out) {
    out->max_resid = c.h_out[0];
    out->l2_resid = c.h_out[1];
  }
}

static void do_init(Ctx& c) {
  for (int l = 1; l <= c.mesh.L; ++l) c.ops->pins(c, l);
  assemble_coarse(c);
  enq_reset_records(c);
  c.have_guess = false;
  invalidate_graphs(c);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

static void need_mesh(Ctx& c) { require(c.have_mesh, "mesh not set (call pmg_b200_set_mesh)", PMG_ERR_STATE); }
static void need_level(Ctx& c, int l, int lo = 1) {
  need_mesh(c);
  require(l >= lo && l <= c.mesh.L, "level out of range");
}

// ---------------------------------------------------------------- partitioned cycle (dist.h)
static void enq_smooth_dist(Ctx& c, int l, int steps) {
  if (c.dist->world == 1 && c.ops->smooth(c, l, steps)) return;  // no exchange between half-sweeps
  for (int s = 0; s < steps; ++s)
    for (int par = 0; par < 2; ++par) {
      c.ops->gs(c, l, par);
      dist_xchg(c, PMG_VAR_PHI, l, par);  // the colour just updated
    }
}
// v_cycle (multigrid.hpp:483-499) over this rank's blocks, exchanging halo
// layers after every phase that changes them; the coarse tail on rank 0
static void enq_dist_cycle(Ctx& c) {
  DistState& ds = *c.dist;
  const int L = c.mesh.L, g = ds.split;
  enq_clear_cycle(c);
  // halo phi as the owners hold it now (after init, an upload or the last cycle)
  for (int l = g; l <= L; ++l) dist_xchg(c, PMG_VAR_PHI, l, 2);
  for (int l = L; l >= std::max(g, 2); --l) {
    enq_smooth_dist(c, l, c.cfg.n_down);
    enq_restrict_only(c, l);  // restriction into l-1 and its pins, owned parents
    if (l - 1 >= g) {
      dist_xchg(c, PMG_VAR_PHI, l - 1, 2);
      enq_fas_level(c, l);
      dist_xchg(c, PMG_VAR_OLD, l - 1, 2);
    } else {  // the split level's parents: octants gathered to rank 0, pinned there
      dist_move(c, -1, 0, level_var(c, PMG_VAR_PHI, l - 1));
      dist_move(c, -1, 0, level_var(c, PMG_VAR_RHS, l - 1));
      phi_written(c, l - 1);
      if (ds.rank == 0) {
        c.ops->pins(c, l - 1);
        enq_fas_level(c, l);
      }
    }
  }
  if (g >= 2) {
    if (ds.rank == 0) enq_v_span(c, g - 1);  // the coarse tail alone
    dist_bcast_level(c, PMG_VAR_PHI, g - 1);
    dist_bcast_level(c, PMG_VAR_OLD, g - 1);
  } else {
    enq_coarse(c);
  }
  for (int l = std::max(g, 2); l <= L; ++l) {
    c.prolong_dead = c.cfg.n_up > 0 ? 0 : -1;
    c.ops->prolong(c, l, false);
    c.prolong_dead = -1;
    dist_xchg(c, PMG_VAR_PHI, l, 2);
    enq_smooth_dist(c, l, c.cfg.n_up);
    c.ops->record(c, l);
  }
  dist_records(c);
  enq_copy_out(c);
}
// one partitioned V-cycle: a CUDA graph (no transport, or NCCL -- pack kernels
// and NCCL calls captured together), eager with the in-process transport
static void launch_dist_cycle(Ctx& c) {
  require(c.solver, "solver not created (call pmg_b200_solver_create)", PMG_ERR_STATE);
  require(c.dist != nullptr, "no partition (call pmg_b200_set_partition)", PMG_ERR_STATE);
  DistState& ds = *c.dist;
  require(ds.world == 1 || ds.transport != TR_NONE, "partition over several ranks without a transport "
          "(pmg_b200_dist_init_nccl / pmg_b200_dist_local_group)", PMG_ERR_STATE);
  if (ds.transport == TR_LOCAL || ds.graph_failed) {
    enq_dist_cycle(c);
  } else {
    if (!ds.g.exec) {
      cudaGraph_t graph = nullptr;
      cfc_all_dirty(c);
      PMG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      bool ok = true;
      try {
        enq_dist_cycle(c);
      } catch (...) {
        ok = false;
      }
      const cudaError_t e = cudaStreamEndCapture(c.stream, &graph);
      cfc_all_dirty(c);
      if (ok && e == cudaSuccess && graph && cudaGraphInstantiate(&ds.g.exec, graph, 0) == cudaSuccess) {
        size_t nn = 0;
        PMG_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        PMG_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
        ds.g.kernels = 0;
        for (auto nd : nodes) {
          cudaGraphNodeType t;
          PMG_CUDA(cudaGraphNodeGetType(nd, &t));
          if (t == cudaGraphNodeTypeKernel) ++ds.g.kernels;
        }
        cudaGraphDestroy(graph);
      } else {  // a transport that cannot be captured: replay the enqueue every cycle
        if (graph) cudaGraphDestroy(graph);
        (void)cudaGetLastError();
        ds.g.exec = nullptr;
        ds.graph_failed = true;
        enq_dist_cycle(c);
        c.have_guess = true;
        return;
      }
    }
    PMG_CUDA(cudaGraphLaunch(ds.g.exec, c.stream));
  }
  c.have_guess = true;
}

// ownership from the caller's partition (owner rank per block id on the
// levels >= split; the levels below belong to rank 0), then the halo plans
static void set_partition(Ctx& c, int world, int rank, int split, const int32_t* owner) {
  need_mesh(c);
  const HostMesh& m = c.mesh;
  require(world >= 1 && rank >= 0 && rank < world, "bad world / rank");
  require(split >= 1 && split <= m.L, "split level out of range");
  require(world == 1 || split >= 2, "a partition over several ranks needs a split level >= 2 "
          "(the coarse solve of level 1 runs on rank 0)");
  auto ds = std::make_unique<DistState>();
  ds->world = world;
  ds->rank = rank;
  ds->split = world == 1 ? 1 : split;
  ds->owner.assign((size_t)m.nb, 0);
  if (owner) ds->owner.assign(owner, owner + m.nb);
  for (int id = 0; id < m.nb; ++id)
    require(ds->owner[(size_t)id] >= 0 && ds->owner[(size_t)id] < world, "owner rank out of range");
  for (int id = 0; id < m.nb; ++id) {  // a subtree stays on its split-level ancestor's rank
    const int p = m.parent[(size_t)id];
    if (m.level[(size_t)id] > ds->split && p >= 0)
      require(ds->owner[(size_t)id] == ds->owner[(size_t)p], "a block and its parent on different ranks");
  }
  PMG_CUDA(cudaEventCreateWithFlags(&ds->ev_packed, cudaEventDisableTiming));
  PMG_CUDA(cudaEventCreateWithFlags(&ds->ev_copied, cudaEventDisableTiming));
  c.dist = std::move(ds);
  c.owned.assign((size_t)m.L + 1, {});
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    auto& o = c.owned[(size_t)l];
    o.assign((size_t)d.nb, 0);
    d.n_own = 0;
    for (int s = 0; s < d.nb; ++s) {
      o[(size_t)s] = dist_owner_slot(c, l, s) == rank ? 1 : 0;
      d.n_own += o[(size_t)s];
    }
    d.own.upload(o, c.stream);
    d.has_own = world > 1;
    if (!d.has_own) o.clear();
  }
  if (c.st.valid) upload_stencils(c);
  build_dist_plans(c);
  if (world > 1) shrink_fields(c);
  set_views(c);
  invalidate_graphs(c);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

static void set_mesh(Ctx& c, int nb, const int32_t* level, const int32_t* coords,
                     const double* origin, const double* dx, const int32_t* parent,
                     const int32_t* children, const int32_t* nbr, const int32_t* cnbr) {
  require(nb >= 1, "mesh needs at least one block");
  HostMesh& m = c.mesh;
  m = HostMesh{};
  m.nb = nb;
  m.level.assign(level, level + nb);
  m.coords.assign(coords, coords + (size_t)nb * 3);
  m.origin.assign(origin, origin + (size_t)nb * 3);
  m.dx.assign(dx, dx + nb);
  m.parent.assign(parent, parent + nb);
  m.children.assign(children, children + (size_t)nb * 8);
  m.nbr.assign(nbr, nbr + (size_t)nb * 6);
  m.cnbr.assign(cnbr, cnbr + (size_t)nb * 6);
  m.L = *std::max_element(m.level.begin(), m.level.end());
  require(m.L < pmgdev::kMaxLevels, "too many levels");
  m.slots.assign((size_t)m.L + 1, {});
  m.ref_order.assign((size_t)m.L + 1, {});
  m.slot_of.assign((size_t)nb, -1);
  for (int id = 0; id < nb; ++id) {
    require(m.level[(size_t)id] >= 1, "block level must be >= 1");
    m.slots[(size_t)m.level[(size_t)id]].push_back(id);
  }
  require(m.slots[1].size() == 1, "level 1 must hold exactly the root block");
  const int D = c.dim;
  for (int l = 1; l <= m.L; ++l) {
    auto& v = m.slots[(size_t)l];
    require(!v.empty(), "every level 1..L must hold blocks");
    m.ref_order[(size_t)l] = v;
    std::sort(m.ref_order[(size_t)l].begin(), m.ref_order[(size_t)l].end(), [&](int a, int b) {
      for (int k = 0; k < D; ++k)
        if (m.coords[(size_t)a * 3 + k] != m.coords[(size_t)b * 3 + k])
          return m.coords[(size_t)a * 3 + k] < m.coords[(size_t)b * 3 + k];
      return false;
    });
    std::stable_sort(v.begin(), v.end(), [&](int a, int b) {
      return morton(&m.coords[(size_t)a * 3], D) < morton(&m.coords[(size_t)b * 3], D);
    });
    for (size_t s = 0; s < v.size(); ++s) m.slot_of[(size_t)v[s]] = (int)s;
    for (int id : v)
      require(m.dx[(size_t)id] == m.dx[(size_t)v[0]], "blocks of one level must share dx");
  }
  // topology per level, in slot order
  c.lev.clear();
  c.lev.resize((size_t)m.L + 1);
  const int F = c.F, NC = 1 << D;
  for (int l = 1; l <= m.L; ++l) {
    c.lev[(size_t)l] = std::make_unique<LevelDev>();
    LevelDev& d = *c.lev[(size_t)l];
    const auto& v = m.slots[(size_t)l];
    d.nb = (int)v.size();
    std::vector<int32_t> nbrs((size_t)d.nb * F), cnbrs((size_t)d.nb * F), crd((size_t)d.nb * D),
        par((size_t)d.nb), chl((size_t)d.nb * NC), sid((size_t)d.nb), rpos((size_t)d.nb),
        cfoff((size_t)d.nb * F, -1);
    std::vector<uint8_t> leaf((size_t)d.nb);
    for (size_t s = 0; s < v.size(); ++s) {
      const int id = v[s];
      sid[s] = id;
      for (int k = 0; k < D; ++k) crd[s * D + k] = m.coords[(size_t)id * 3 + k];
      const int p = m.parent[(size_t)id];
      require(l == 1 ? p < 0 : (p >= 0 && m.level[(size_t)p] == l - 1), "bad parent link");
      par[s] = p < 0 ? -1 : m.slot_of[(size_t)p];
      bool lf = true;
      for (int ch = 0; ch < NC; ++ch) {
        const int cid = m.children[(size_t)id * 8 + ch];
        chl[s * NC + ch] = cid < 0 ? -1 : m.slot_of[(size_t)cid];
        if (ch == 0) lf = cid < 0;
      }
      leaf[s] = lf ? 1 : 0;
      for (int f = 0; f < F; ++f) {
        const int nid = m.nbr[(size_t)id * 6 + f];
        const int cid = m.cnbr[(size_t)id * 6 + f];
        nbrs[s * F + f] = nid < 0 ? -1 : m.slot_of[(size_t)nid];
        cnbrs[s * F + f] = -1;
        if (nid >= 0) require(m.level[(size_t)nid] == l, "nbr must be on the same level", PMG_ERR_TOPOLOGY);
        if (nid < 0 && cid >= 0) {
          require(m.level[(size_t)cid] == l - 1, "coarse nbr must be one level up", PMG_ERR_TOPOLOGY);
          cnbrs[s * F + f] = m.slot_of[(size_t)cid];
          d.has_cf = true;
          // transverse faces of the coarse neighbour must not be coarse-fine
          // (2:1 corner balance, mesh.hpp:252-290)
          for (int g = 0; g < F; ++g) {
            if ((g >> 1) == (f >> 1)) continue;
            require(!(m.nbr[(size_t)cid * 6 + g] < 0 && m.cnbr[(size_t)cid * 6 + g] >= 0),
                    "mesh is not 2:1 corner balanced at a coarse-fine face", PMG_ERR_TOPOLOGY);
          }
        }
      }
    }
    {  // dense level: every block present and its slot equals its Morton code
      const long nside = 1L << (l - 1);
      long full = 1;
      for (int k = 0; k < D; ++k) full *= nside;
      bool dense = d.nb == full && nside <= 1024;
      for (size_t s = 0; dense && s < v.size(); ++s)
        dense = morton(&m.coords[(size_t)v[s] * 3], D) == (uint64_t)s;
      d.dense = dense;
    }
    const auto& ro = m.ref_order[(size_t)l];
    for (size_t q = 0; q < ro.size(); ++q) rpos[(size_t)m.slot_of[(size_t)ro[q]]] = (int32_t)q;
    d.nbr.upload(nbrs, c.stream);
    d.cnbr.upload(cnbrs, c.stream);
    d.coords.upload(crd, c.stream);
    d.parent.upload(par, c.stream);
    d.child.upload(chl, c.stream);
    d.n_own = d.nb;
    d.leaf.upload(leaf, c.stream);
    d.n_leaf = 0;
    for (uint8_t f : leaf) d.n_leaf += f ? 1 : 0;
    d.slot_id.upload(sid, c.stream);
    d.ref_slot.upload(rpos, c.stream);
    const size_t cells = (size_t)d.nb * c.NI;
    d.phi.alloc(cells);
    d.rhs.alloc(cells);
    d.old.alloc(cells);
    d.res.alloc(cells);
    PMG_CUDA(cudaMemsetAsync(d.phi.p, 0, cells * 8, c.stream));
    PMG_CUDA(cudaMemsetAsync(d.rhs.p, 0, cells * 8, c.stream));
    PMG_CUDA(cudaMemsetAsync(d.old.p, 0, cells * 8, c.stream));
    PMG_CUDA(cudaMemsetAsync(d.res.p, 0, cells * 8, c.stream));
  }
  // VAR_OLD coarse-fine ghost tables: needed on level l-1 blocks that are
  // parents of level-l blocks and have a coarse-fine face
  for (int l = 1; l <= m.L; ++l) {
    LevelDev& d = *c.lev[(size_t)l];
    std::vector<int32_t> cfo((size_t)d.nb * F, -1);
    int n = 0;
    for (int s = 0; s < d.nb; ++s) {
      const int id = m.slots[(size_t)l][(size_t)s];
      for (int f = 0; f < F; ++f)
        if (m.nbr[(size_t)id * 6 + f] < 0 && m.cnbr[(size_t)id * 6 + f] >= 0) {
          cfo[(size_t)s * F + f] = n;
          n += c.NT;
        }
    }
    d.has_cfold = n > 0;
    d.cfoff_host = cfo;
    d.cfoff.upload(cfo, c.stream);
    d.cfold.alloc((size_t)std::max(n, 1));
    // the same faces, listed, and their cfc pages (LevelView::cfc)
    std::vector<int32_t> cff;
    for (int s = 0; s < d.nb; ++s)
      for (int f = 0; f < F; ++f)
        if (cfo[(size_t)s * F + f] >= 0) {
          cff.push_back(s);
          cff.push_back(f);
        }
    d.n_cf = (int)(cff.size() / 2);
    if (d.n_cf > 0) d.cf_faces.upload(cff, c.stream);
    // k_cfc_build descriptors, 8 int32 per face: {slot, dir | h0 << 3 | h1 << 4,
    // cfc offset, coarse slot, the coarse block's same-level neighbours across
    // the two transverse axes (-/+ of the lower, -/+ of the higher; -1 none)}.
    // h_a: the fine block lies in the upper half of the coarse block along
    // transverse axis a, i.e. coarse cell = (h_a N + t_a) >> 1.
    std::vector<int32_t> cfd;
    for (int q = 0; q < d.n_cf; ++q) {
      const int s = cff[(size_t)2 * q], f = cff[(size_t)2 * q + 1];
      const int id = m.slots[(size_t)l][(size_t)s];
      const int cid = m.cnbr[(size_t)id * 6 + f];
      const int ax = f >> 1;
      int h[2], nn[4], u = 0;
      for (int a = 0; a < D; ++a) {
        if (a == ax) continue;
        const int b = m.coords[(size_t)id * 3 + a] - 2 * m.coords[(size_t)cid * 3 + a];
        require(b == 0 || b == 1, "coarse neighbour does not cover the fine face", PMG_ERR_TOPOLOGY);
        h[u] = b;
        for (int sd = 0; sd < 2; ++sd) {
          const int nid = m.nbr[(size_t)cid * 6 + 2 * a + sd];
          nn[2 * u + sd] = nid < 0 ? -1 : m.slot_of[(size_t)nid];
        }
        ++u;
      }
      for (; u < 2; ++u) h[u] = 0, nn[2 * u] = nn[2 * u + 1] = -1;  // 2D: one transverse axis
      const int32_t e[8] = {s, f | (h[0] << 3) | (h[1] << 4), cfo[(size_t)s * F + f], m.slot_of[(size_t)cid],
                            nn[0], nn[1], nn[2], nn[3]};
      cfd.insert(cfd.end(), e, e + 8);
    }
    if (d.n_cf > 0) d.cf_desc.upload(cfd, c.stream);
    d.cfc.alloc((size_t)std::max(n, 1));
    d.cfc_dirty = true;
  }
  for (int f = 0; f < 6; ++f) {
    c.face_vals[f].clear();
    c.face_off[f].clear();
  }
  int maxnb = 0;
  for (int l = 1; l <= m.L; ++l) maxnb = std::max(maxnb, c.lev[(size_t)l]->nb);
  c.partial.alloc((size_t)maxnb + 8192);  // + per-CTA partials of k_record_cut
  {
    static_assert(sizeof(pmgdev::Rec) == 3 * sizeof(double), "records follow the five output doubles");
    const size_t nrec = pmgdev::kMaxLevels + 1;
    c.outbuf.alloc(5 + 3 * nrec);
    PMG_CUDA(cudaMemsetAsync(c.outbuf.p, 0, c.outbuf.n * sizeof(double), c.stream));
    c.stats.p = c.outbuf.p, c.stats.n = 2;
    c.diag.p = c.outbuf.p + 2, c.diag.n = 2;
    c.status.p = reinterpret_cast<int*>(c.outbuf.p + 4), c.status.n = 1;
    c.rec.p = reinterpret_cast<pmgdev::Rec*>(c.outbuf.p + 5), c.rec.n = nrec;
  }
  c.counter.alloc(1);
  PMG_CUDA(cudaMemsetAsync(c.counter.p, 0, sizeof(unsigned), c.stream));
  c.have_mesh = true;
  c.solver = false;
  default_stencils(c);
  upload_bc(c);
  upload_stencils(c);
  set_views(c);
  invalidate_graphs(c);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

static void set_face_bc(Ctx& c, int dir, int type, const double* values) {
  need_mesh(c);
  require(dir >= 0 && dir < c.F, "face direction out of range");
  require(type == PMG_BC_DIRICHLET || type == PMG_BC_NEUMANN_ZERO, "bad face bc type");
  c.bctype[dir] = type;
  c.face_vals[dir].clear();
  c.face_off[dir].assign((size_t)c.mesh.nb, -1);
  if (values) {
    size_t q = 0;
    for (int id = 0; id < c.mesh.nb; ++id) {
      if (c.mesh.nbr[(size_t)id * 6 + dir] >= 0 || c.mesh.cnbr[(size_t)id * 6 + dir] >= 0) continue;
      c.face_off[dir][(size_t)id] = (int32_t)c.face_vals[dir].size();
      c.face_vals[dir].insert(c.face_vals[dir].end(), values + q, values + q + c.NT);
      q += (size_t)c.NT;
    }
  }
  upload_bc(c);
  if (c.st.valid) {
    build_cut_tables(c);
    build_small_tables(c);
    build_rfix_tables(c);
  }
  set_views(c);
  invalidate_graphs(c);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

static double* staging(Ctx& c, size_t n) {
  if (c.staging.n < n) c.staging.alloc(n);
  return c.staging.p;
}

static double* var_ptr(LevelDev& d, int var) {
  switch (var) {
    case PMG_VAR_PHI: return d.phi.p;
    case PMG_VAR_RHS: return d.rhs.p;
    case PMG_VAR_RES: return d.res.p;
    case PMG_VAR_OLD: return d.old.p;
    default: throw PmgError(PMG_ERR_INVALID_ARG, "unsupported field variable");
  }
}

static void upload_field(Ctx& c, int var, int level, const double* host, int layout) {
  need_mesh(c);
  require(layout == PMG_LAYOUT_PADDED || layout == PMG_LAYOUT_INTERIOR, "bad layout");
  const size_t per = layout == PMG_LAYOUT_PADDED ? (size_t)c.S : (size_t)c.NI;
  const size_t nblk = level > 0 ? (size_t)c.lev[(size_t)level]->nb : (size_t)c.mesh.nb;
  double* stg = staging(c, nblk * per);
  PMG_CUDA(cudaMemcpyAsync(stg, host, nblk * per * 8, cudaMemcpyHostToDevice, c.stream));
  for (int l = 1; l <= c.mesh.L; ++l) {
    if (level > 0 && l != level) continue;
    LevelDev& d = *c.lev[(size_t)l];
    c.ops->scatter(c, l, var_ptr(d, var), stg, level > 0 ? d.ref_slot.p : d.slot_id.p, layout);
  }
}

// Double-buffered upload: the H2D copy runs on its own stream into a second
// staging buffer (overlapping whatever the solver stream is doing, e.g. the
// previous V-cycle); commit scatters it into the field on the solver stream.
static void stage_field_async(Ctx& c, int var, int level, const double* host, int layout) {
  need_mesh(c);
  require(layout == PMG_LAYOUT_PADDED || layout == PMG_LAYOUT_INTERIOR, "bad layout");
  require(var >= 0 && var <= 3, "unsupported field variable");
  require(level >= 0 && level <= c.mesh.L, "level out of range");
  if (!c.copy) {
    PMG_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    PMG_CUDA(cudaEventCreateWithFlags(&c.ev_staged, cudaEventDisableTiming));
    PMG_CUDA(cudaEventCreateWithFlags(&c.ev_consumed, cudaEventDisableTiming));
    PMG_CUDA(cudaEventRecord(c.ev_consumed, c.stream));
  }
  const size_t per = layout == PMG_LAYOUT_PADDED ? (size_t)c.S : (size_t)c.NI;
  const size_t nblk = level > 0 ? (size_t)c.lev[(size_t)level]->nb : (size_t)c.mesh.nb;
  if (c.stage2.n < nblk * per) {
    PMG_CUDA(cudaStreamSynchronize(c.copy));
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    c.stage2.alloc(nblk * per);
  }
  PMG_CUDA(cudaStreamWaitEvent(c.copy, c.ev_consumed, 0));  // the previous commit has read the buffer
  PMG_CUDA(cudaMemcpyAsync(c.stage2.p, host, nblk * per * 8, cudaMemcpyHostToDevice, c.copy));
  PMG_CUDA(cudaEventRecord(c.ev_staged, c.copy));
  c.staged_var = var;
  c.staged_level = level;
  c.staged_layout = layout;
}
static void commit_staged_field(Ctx& c) {
  require(c.staged_var >= 0, "no staged field (call pmg_b200_stage_field_async)", PMG_ERR_STATE);
  PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_staged, 0));
  for (int l = 1; l <= c.mesh.L; ++l) {
    if (c.staged_level > 0 && l != c.staged_level) continue;
    LevelDev& d = *c.lev[(size_t)l];
    c.ops->scatter(c, l, var_ptr(d, c.staged_var), c.stage2.p, c.staged_level > 0 ? d.ref_slot.p : d.slot_id.p,
                   c.staged_layout);
  }
  PMG_CUDA(cudaEventRecord(c.ev_consumed, c.stream));
  c.staged_var = -1;
}
static void download_field(Ctx& c, int var, int level, double* host, int layout) {
  need_mesh(c);
  require(layout == PMG_LAYOUT_PADDED || layout == PMG_LAYOUT_INTERIOR, "bad layout");
  require(var >= 0 && var <= 3, "unsupported field variable");
  const size_t per = layout == PMG_LAYOUT_PADDED ? (size_t)c.S : (size_t)c.NI;
  const size_t nblk = level > 0 ? (size_t)c.lev[(size_t)level]->nb : (size_t)c.mesh.nb;
  double* stg = staging(c, nblk * per);
  for (int l = 1; l <= c.mesh.L; ++l) {
    if (level > 0 && l != level) continue;
    LevelDev& d = *c.lev[(size_t)l];
    c.ops->gather(c, l, var, stg, level > 0 ? d.ref_slot.p : d.slot_id.p, layout);
  }
  PMG_CUDA(cudaMemcpyAsync(host, stg, nblk * per * 8, cudaMemcpyDeviceToHost, c.stream));
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

static void set_stencils(Ctx& c, const int32_t* boundary, const int32_t* row_count,
                         const int32_t* row_of, const double* center, const double* nb,
                         const double* bc, const double* d, const int8_t* obj,
                         const uint8_t* mask, const int8_t* pin, const int32_t* lin, int n_obj,
                         const double* phi_b) {
  need_mesh(c);
  require(n_obj >= 0 && n_obj <= 127, "at most 127 boundary objects (int8 ids)");
  HostStencils& st = c.st;
  st = HostStencils{};
  const int nbk = c.mesh.nb, F = c.F;
  st.boundary.assign(boundary, boundary + nbk);
  st.row_count.assign(row_count, row_count + nbk);
  st.row_start.assign((size_t)nbk + 1, 0);
  for (int i = 0; i < nbk; ++i) st.row_start[(size_t)i + 1] = st.row_start[(size_t)i] + st.row_count[(size_t)i];
  const size_t R = (size_t)st.row_start[(size_t)nbk];
  st.NI = c.NI;
  st.row_page.assign((size_t)nbk, -1);
  st.row_pages.clear();
  for (int i = 0; i < nbk; ++i)
    if (st.boundary[(size_t)i]) {
      st.row_page[(size_t)i] = (int32_t)(st.row_pages.size() / (size_t)c.NI);
      st.row_pages.insert(st.row_pages.end(), row_of + (size_t)i * c.NI, row_of + (size_t)(i + 1) * c.NI);
    }
  st.center.assign(center, center + R);
  st.nb.assign(nb, nb + R * F);
  st.bc.assign(bc, bc + R * F);
  st.d.assign(d, d + R * F);
  st.obj.assign(obj, obj + R * F);
  st.mask.assign(mask, mask + R);
  st.pin.assign(pin, pin + R);
  st.lin.assign(lin, lin + R);
  st.phi_b.assign(phi_b, phi_b + n_obj);
  for (size_t r = 0; r < R; ++r) {
    if (st.mask[r] == PMG_INSIDE) require(st.pin[r] >= 0 && st.pin[r] < n_obj, "pin_obj out of range");
    for (int f = 0; f < F; ++f)
      if (st.bc[r * F + f] != 0)
        require(st.obj[r * F + f] >= 0 && st.obj[r * F + f] < n_obj, "stencil object id out of range");
  }
  st.valid = true;
  c.devrows.reset();
  upload_stencils(c);
  set_views(c);
  c.solver = false;
  invalidate_graphs(c);
  PMG_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace pmghost

// ============================================================================ C ABI
template <typename Fn>
static int guard(pmg_b200_ctx* h, Fn&& fn) {
  if (!h) return PMG_ERR_STATE;
  try {
    h->c.err.clear();
    PMG_CUDA(cudaSetDevice(h->c.device));
    // the caller may have written PHI through pmg_b200_level_field_ptr
    pmghost::cfc_all_dirty(h->c);
    fn(h->c);
    return PMG_OK;
  } catch (const PmgError& e) {
    h->c.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    h->c.err = e.what();
    return PMG_ERR_INVALID_ARG;
  }
}

extern "C" {

pmg_b200_ctx* pmg_b200_create(int dim, int N, const double* lo, const double* hi, int device) {
  auto* h = new (std::nothrow) pmg_b200_ctx;
  if (!h) return nullptr;
  Ctx& c = h->c;
  try {
    require(dim == 2 || dim == 3, "dim must be 2 or 3");
    require(N >= 4 && (N & (N - 1)) == 0, "block size N must be a power of two and at least 4");
    c.dim = dim;
    c.N = N;
    c.F = 2 * dim;
    c.NI = dim == 2 ? N * N : N * N * N;
    c.S = dim == 2 ? (N + 2) * (N + 2) : (N + 2) * (N + 2) * (N + 2);
    c.NT = dim == 2 ? N : N * N;
    const double ext = hi[0] - lo[0];
    for (int k = 0; k < dim; ++k) {
      c.lo[k] = lo[k];
      c.hi[k] = hi[k];
      require(std::abs((hi[k] - lo[k]) - ext) <= 1e-12 * std::abs(ext), "domain must be square/cubic");
    }
    require(ext > 0, "domain extent must be positive");
    c.device = device;
    PMG_CUDA(cudaSetDevice(device));
    PMG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    PMG_CUDA(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, device));
    PMG_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    PMG_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    PMG_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    PMG_CUDA(cudaHostAlloc(&c.h_out, 5 * sizeof(double), cudaHostAllocMapped));
    std::memset(c.h_out, 0, 5 * sizeof(double));
    if (cudaHostGetDevicePointer(&c.h_out_dev, c.h_out, 0) != cudaSuccess) {
      c.h_out_dev = nullptr;  // no mapped access: the cycles end with a copy node
      cudaGetLastError();
    }
    c.h_status = reinterpret_cast<int*>(c.h_out + 4);
    c.gbar.alloc(2);
    PMG_CUDA(cudaMemset(c.gbar.p, 0, 2 * sizeof(unsigned)));
    c.ops = make_ops(dim, N);
  } catch (const std::exception& e) {
    c.err = e.what();
  }
  return h;
}

void pmg_b200_destroy(pmg_b200_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->c.device);
  if (h->c.stream) cudaStreamSynchronize(h->c.stream);
  delete h;
}

const char* pmg_b200_last_error(pmg_b200_ctx* h) { return h ? h->c.err.c_str() : "null context"; }
void* pmg_b200_stream(pmg_b200_ctx* h) { return h ? (void*)h->c.stream : nullptr; }

int pmg_b200_set_mesh(pmg_b200_ctx* h, int n_blocks, const int32_t* level, const int32_t* coords,
                      const double* origin, const double* dx, const int32_t* parent,
                      const int32_t* children, const int32_t* nbr, const int32_t* cnbr) {
  return guard(h, [&](Ctx& c) {
    require(c.ops != nullptr, c.err.empty() ? "context not initialised" : c.err);
    set_mesh(c, n_blocks, level, coords, origin, dx, parent, children, nbr, cnbr);
  });
}
int pmg_b200_set_face_bc(pmg_b200_ctx* h, int dir, int type, const double* values) {
  return guard(h, [&](Ctx& c) { set_face_bc(c, dir, type, values); });
}
int pmg_b200_set_stencils(pmg_b200_ctx* h, const int32_t* boundary, const int32_t* row_count,
                          const int32_t* row_of, const double* center, const double* nb,
                          const double* bc, const double* d, const int8_t* obj,
                          const uint8_t* mask, const int8_t* pin_obj, const int32_t* lin,
                          int n_obj, const double* phi_b) {
  return guard(h, [&](Ctx& c) {
    set_stencils(c, boundary, row_count, row_of, center, nb, bc, d, obj, mask, pin_obj, lin, n_obj,
                 phi_b);
  });
}
int pmg_b200_build_stencils(pmg_b200_ctx* h, const pmg_lsf_t* lsf, int n_lsf,
                            const pmg_stencil_cfg_t* cfg) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(lsf && n_lsf >= 1 && cfg, "bad level-set description");
    c.ops->build_stencils(c, lsf, n_lsf, cfg);
    upload_stencils(c);
    set_views(c);
    c.solver = false;
    invalidate_graphs(c);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_stencil_summary(pmg_b200_ctx* h, int32_t* boundary, int32_t* row_count) {
  int total = 0;
  int rc = guard(h, [&](Ctx& c) {
    need_mesh(c);
    for (int i = 0; i < c.mesh.nb; ++i) {
      if (boundary) boundary[i] = c.st.boundary[(size_t)i];
      if (row_count) row_count[i] = c.st.row_count[(size_t)i];
    }
    total = c.st.row_start.empty() ? 0 : c.st.row_start.back();
  });
  return rc == 0 ? total : -rc;
}
int pmg_b200_get_stencils(pmg_b200_ctx* h, int32_t* row_of, double* center, double* nb,
                          double* bc, double* d, int8_t* obj, uint8_t* mask, int8_t* pin_obj,
                          int32_t* lin) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    const HostStencils& st = c.st;
    for (int i = 0; i < c.mesh.nb; ++i)
      for (int q = 0; q < c.NI; ++q)
        row_of[(size_t)i * c.NI + q] = st.boundary[(size_t)i] ? st.row_at((size_t)i, (size_t)q) : -1;
    std::copy(st.center.begin(), st.center.end(), center);
    std::copy(st.nb.begin(), st.nb.end(), nb);
    std::copy(st.bc.begin(), st.bc.end(), bc);
    std::copy(st.d.begin(), st.d.end(), d);
    std::copy(st.obj.begin(), st.obj.end(), obj);
    std::copy(st.mask.begin(), st.mask.end(), mask);
    std::copy(st.pin.begin(), st.pin.end(), pin_obj);
    std::copy(st.lin.begin(), st.lin.end(), lin);
  });
}
int pmg_b200_set_boundary_value(pmg_b200_ctx* h, int obj, double value) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(obj >= 0 && obj < (int)c.st.phi_b.size(), "boundary object out of range");
    c.st.phi_b[(size_t)obj] = value;
    PMG_CUDA(cudaMemcpyAsync(c.phi_b.p + obj, &c.st.phi_b[(size_t)obj], sizeof(double),
                             cudaMemcpyHostToDevice, c.stream));
    if (c.st.valid) {  // their bc * phi_b products
      build_cut_tables(c);
      build_row_coef(c);
      set_views(c);          // the tables were reallocated: views and graphs
      invalidate_graphs(c);  // hold their device pointers
    }
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_upload_field(pmg_b200_ctx* h, int var, const double* host, int layout) {
  return guard(h, [&](Ctx& c) { upload_field(c, var, 0, host, layout); });
}
int pmg_b200_download_field(pmg_b200_ctx* h, int var, double* host, int layout) {
  return guard(h, [&](Ctx& c) { download_field(c, var, 0, host, layout); });
}
int pmg_b200_upload_level_field(pmg_b200_ctx* h, int var, int level, const double* host, int layout) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    upload_field(c, var, level, host, layout);
  });
}
int pmg_b200_stage_field_async(pmg_b200_ctx* h, int var, int level, const double* host, int layout) {
  return guard(h, [&](Ctx& c) { stage_field_async(c, var, level, host, layout); });
}
int pmg_b200_commit_staged_field(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) { commit_staged_field(c); });
}
int pmg_b200_download_level_field(pmg_b200_ctx* h, int var, int level, double* host, int layout) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    download_field(c, var, level, host, layout);
  });
}
int pmg_b200_solver_create(pmg_b200_ctx* h, const pmg_mg_cfg_t* cfg) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(cfg != nullptr, "null MgConfig");
    // MgConfig::validate (multigrid.hpp:22-27)
    require(cfg->n_down >= 1 && cfg->n_up >= 1, "n_up and n_down must be at least 1");
    require(cfg->coarse_rel_tol > 0 && cfg->coarse_rel_tol < 1, "coarse_rel_tol must be in (0, 1)");
    require(cfg->threads >= 1, "thread count must be at least 1");
    c.cfg = *cfg;
    c.solver = true;
    do_init(c);
  });
}
int pmg_b200_init(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    do_init(c);
  });
}
int pmg_b200_v_cycle_async(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) { launch_cycle(c, CK_V); });
}
int pmg_b200_fmg_cycle_async(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) { launch_cycle(c, c.have_guess ? CK_FMG_GUESS : CK_FMG_NOGUESS); });
}
int pmg_b200_cycle_result(pmg_b200_ctx* h, pmg_cycle_stats_t* out) {
  return guard(h, [&](Ctx& c) { cycle_result(c, out); });
}
int pmg_b200_v_cycle(pmg_b200_ctx* h, pmg_cycle_stats_t* out) {
  return guard(h, [&](Ctx& c) {
    launch_cycle(c, CK_V);
    cycle_result(c, out);
  });
}
int pmg_b200_fmg_cycle(pmg_b200_ctx* h, pmg_cycle_stats_t* out) {
  return guard(h, [&](Ctx& c) {
    launch_cycle(c, c.have_guess ? CK_FMG_GUESS : CK_FMG_NOGUESS);
    cycle_result(c, out);
  });
}
int pmg_b200_measure_residual(pmg_b200_ctx* h, pmg_cycle_stats_t* out) {
  return guard(h, [&](Ctx& c) {
    launch_cycle(c, CK_MEASURE);
    cycle_result(c, out);
  });
}
int pmg_b200_gsrb_sweep(pmg_b200_ctx* h, int level, int parity) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    require(parity == 0 || parity == 1, "parity must be 0 or 1");
    c.ops->gs(c, level, parity);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_fill_ghosts(pmg_b200_ctx* h, int level, int var) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    (void)var;  // ghost layers are evaluated on read: always current
  });
}
int pmg_b200_apply_pins(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    c.ops->pins(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_residual_level(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level);
    c.ops->residual(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_restrict_level(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 2);
    enq_restrict_level(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_restrict_level_no_guess(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 2);
    enq_restrict_level_no_guess(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_prolong_correction(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 2);
    c.ops->prolong(c, level, false);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_prolong_full(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 2);
    c.ops->prolong(c, level, true);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_coarse_solve(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    enq_clear_status(c);
    enq_coarse(c);
    enq_copy_out(c);
    cycle_result(c, nullptr);
  });
}
int pmg_b200_set_have_guess(pmg_b200_ctx* h, int v) {
  return guard(h, [&](Ctx& c) { c.have_guess = v != 0; });
}
int pmg_b200_coarse_sizes(pmg_b200_ctx* h, int32_t* n, int32_t* nnz, int32_t* n_obj) {
  return guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    *n = c.coarse.n;
    *nnz = (int32_t)c.coarse.val.size();
    *n_obj = (int32_t)c.st.phi_b.size();
  });
}
int pmg_b200_coarse_get(pmg_b200_ctx* h, int32_t* rp, int32_t* ci, double* val, double* c0,
                        double* cobj, int32_t* ub, int32_t* ul) {
  return guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    const HostCoarse& cs = c.coarse;
    std::copy(cs.rp.begin(), cs.rp.end(), rp);
    std::copy(cs.ci.begin(), cs.ci.end(), ci);
    std::copy(cs.val.begin(), cs.val.end(), val);
    std::copy(cs.c0.begin(), cs.c0.end(), c0);
    std::copy(cs.cobj.begin(), cs.cobj.end(), cobj);
    std::copy(cs.unk_block.begin(), cs.unk_block.end(), ub);
    std::copy(cs.unk_lin.begin(), cs.unk_lin.end(), ul);
  });
}
int pmg_b200_cycle_kernel_count(pmg_b200_ctx* h, int kind) {
  int k = -1;
  int rc = guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    const int ck = kind == 0 ? CK_V : kind == 2 ? CK_MEASURE : (c.have_guess ? CK_FMG_GUESS : CK_FMG_NOGUESS);
    k = graph_for(c, ck).kernels;
  });
  return rc == 0 ? k : -rc;
}
int pmg_b200_n_levels(pmg_b200_ctx* h) { return h && h->c.have_mesh ? h->c.mesh.L : 0; }
int pmg_b200_n_leaves(pmg_b200_ctx* h) {
  if (!h || !h->c.have_mesh) return 0;
  int n = 0;
  for (int id = 0; id < h->c.mesh.nb; ++id) n += h->c.mesh.children[(size_t)id * 8] < 0 ? 1 : 0;
  return n;
}
// leaves in dump order: level-major, x-major within a level (mesh.hpp:229-235,
// io.hpp:17-21); uploads (level, slot) per leaf, returns the block ids
static std::vector<int32_t> upload_leaf_tab(Ctx& c) {
  const HostMesh& m = c.mesh;
  std::vector<int2> tab;
  std::vector<int32_t> ids;
  for (int l = 1; l <= m.L; ++l)
    for (int id : m.ref_order[(size_t)l])
      if (m.children[(size_t)id * 8] < 0) {
        tab.push_back(make_int2(l, m.slot_of[(size_t)id]));
        ids.push_back(id);
      }
  c.leaf_tab.upload(tab, c.stream);
  return ids;
}
// pmg::write_dump (io.hpp:23-71): "pmg dump 1" text header of the leaf blocks
// (level-major, x-major inside a level), then every leaf interior as raw
// little-endian float64, x fastest.  The field streams from the device one
// level at a time (host memory bounded by the largest level).
int pmg_b200_write_dump(pmg_b200_ctx* h, int var, const char* path, const char* field_name) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(var >= 0 && var <= 3, "unsupported field variable");
    require(path && field_name, "write_dump: path and field name required");
    const HostMesh& m = c.mesh;
    FILE* out = std::fopen(path, "wb");
    require(out != nullptr, std::string("cannot open dump file: ") + path);
    struct Closer {
      FILE* f;
      ~Closer() {
        if (f) std::fclose(f);
      }
    } closer{out};
    const int N = c.N, D = c.dim;
    size_t nleaf = 0;
    for (int id = 0; id < m.nb; ++id) nleaf += m.children[(size_t)id * 8] < 0 ? 1 : 0;
    std::fprintf(out, "pmg dump 1\nfield %s\ndim %d\n", field_name, D);
    for (int v = 0; v < 2; ++v) {
      std::fprintf(out, v ? "domain_hi" : "domain_lo");
      for (int k = 0; k < D; ++k) std::fprintf(out, " %.17g", v ? c.hi[k] : c.lo[k]);
      std::fprintf(out, "\n");
    }
    std::fprintf(out, "block_size %d\nblocks %zu\n", N, nleaf);
    size_t offset = 0;
    for (int l = 1; l <= m.L; ++l)
      for (int id : m.ref_order[(size_t)l]) {
        if (m.children[(size_t)id * 8] >= 0) continue;
        std::fprintf(out, "block %d", l);
        for (int k = 0; k < D; ++k) std::fprintf(out, " %d", m.coords[(size_t)id * 3 + k] * N);
        std::fprintf(out, " %zu\n", offset);
        offset += (size_t)c.NI;
      }
    std::fprintf(out, "data_doubles %zu\nDATA\n", offset);
    std::vector<double> lvl;
    for (int l = 1; l <= m.L; ++l) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (d.n_leaf == 0) continue;
      lvl.resize((size_t)d.nb * c.NI);
      download_field(c, var, l, lvl.data(), PMG_LAYOUT_INTERIOR);  // reference (x-major) order
      const auto& ro = m.ref_order[(size_t)l];
      for (size_t q = 0; q < ro.size(); ++q)
        if (m.children[(size_t)ro[q] * 8] < 0)
          require(std::fwrite(lvl.data() + q * c.NI, sizeof(double), (size_t)c.NI, out) == (size_t)c.NI,
                  std::string("failed writing dump file: ") + path);
    }
    require(std::fflush(out) == 0, std::string("failed writing dump file: ") + path);
  });
}
int pmg_b200_error_norms(pmg_b200_ctx* h, int var, int tag, double phi_b, double a, double R,
                         int volume_weighted, double* linf, double* l2) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(var == 0, "error_norms: only VAR_PHI lives on the device");
    require(tag == 0 || tag == 1, "error_norms: tag 0 (sphere2d) or 1 (sphere3d)");
    require(linf && l2, "error_norms: output pointers required");
    const std::vector<int32_t> ids = upload_leaf_tab(c);
    const int nl = (int)ids.size();
    std::vector<double> org((size_t)nl * 3);
    for (int q = 0; q < nl; ++q)
      for (int k = 0; k < 3; ++k) org[(size_t)q * 3 + k] = c.mesh.origin[(size_t)ids[(size_t)q] * 3 + k];
    DevBuf<double> dorg, part;
    DevBuf<int> err;
    dorg.upload(org, c.stream);
    part.alloc((size_t)nl * c.NI / 256 * 3 + 3 * (c.mesh.L + 2) + 3);
    err.alloc(1);
    PMG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
    const int nb = c.ops->error_norms(c, nl, dorg.p, tag, phi_b, a, R, volume_weighted, part.p, err.p);
    std::vector<double> hp((size_t)nb * 3);
    int herr = 0;
    if (nb > 0) PMG_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    PMG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    if (herr) throw std::domain_error("analytic solution undefined inside");
    double mx = 0, ss = 0, ws = 0;  // fixed order: the CTAs of each level in dump order
    for (int b = 0; b < nb; ++b) {
      mx = std::max(mx, hp[(size_t)b * 3]);
      ss += hp[(size_t)b * 3 + 1];
      ws += hp[(size_t)b * 3 + 2];
    }
    *linf = mx;
    *l2 = ws > 0 ? std::sqrt(ss / ws) : 0;
  });
}
int pmg_b200_face_gradient(pmg_b200_ctx* h, int var, double* faces, double* magnitude, int32_t* leaf_ids) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    require(var == 0, "face_gradient: only VAR_PHI lives on the device");
    require(faces != nullptr, "face_gradient: faces buffer required");
    const std::vector<int32_t> ids = upload_leaf_tab(c);
    const int nl = (int)ids.size();
    int pa = c.N + 1;
    for (int k = 1; k < c.dim; ++k) pa *= c.N;
    const size_t nf = (size_t)nl * c.dim * pa, nm = (size_t)nl * c.NI;
    if (c.ff_faces.n < nf) c.ff_faces.alloc(nf);
    if (magnitude && c.ff_mag.n < nm) c.ff_mag.alloc(nm);
    c.ops->face_gradient(c, nl, c.ff_faces.p, magnitude ? c.ff_mag.p : nullptr);
    PMG_CUDA(cudaMemcpyAsync(faces, c.ff_faces.p, nf * 8, cudaMemcpyDeviceToHost, c.stream));
    if (magnitude) PMG_CUDA(cudaMemcpyAsync(magnitude, c.ff_mag.p, nm * 8, cudaMemcpyDeviceToHost, c.stream));
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    if (leaf_ids) std::copy(ids.begin(), ids.end(), leaf_ids);
  });
}
int pmg_b200_level_size(pmg_b200_ctx* h, int level) {
  if (!h || !h->c.have_mesh || level < 1 || level > h->c.mesh.L) return 0;
  return h->c.lev[(size_t)level]->nb;
}
int pmg_b200_level_classes(pmg_b200_ctx* h, int level, int32_t* out8) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 1);
    require(out8 != nullptr, "out8 is null");
    const LevelDev& d = *c.lev[(size_t)level];
    const int32_t v[8] = {d.nb, d.n_cf, d.n_gs, d.n_gs_slow, d.n_rc, d.n_rc_slow, d.n_rr, d.n_rr_slow};
    for (int k = 0; k < 8; ++k) out8[k] = v[k];
  });
}
int pmg_b200_time_op(pmg_b200_ctx* h, int op, int level, int reps, double* ms_avg) {
  return guard(h, [&](Ctx& c) {
    require(c.solver, "solver not created", PMG_ERR_STATE);
    // op + 100: the reps are captured into one CUDA graph and replayed (the
    // in-cycle cost of a small op, launch gaps as inside the cycle graphs)
    const bool in_graph = op >= 100;
    if (in_graph) op -= 100;
    require(reps >= 1 && op >= 0 && op <= 10 && !(in_graph && op == 6), "bad op/reps");
    if (op <= 3 || op >= 7) need_level(c, level, op == 0 || op == 3 || op == 9 ? 1 : 2);
    auto one = [&](int k) {
      switch (op) {
        case 0: c.ops->gs(c, level, k & 1); break;
        case 1: enq_restrict_level(c, level); break;
        case 2: c.ops->prolong(c, level, false); break;
        case 3: c.ops->record(c, level); break;
        case 4: enq_coarse(c); break;
        case 5:  // in a graph: the V-cycle's nodes themselves, `reps` cycles in ONE graph
          if (in_graph) enq_cycle(c, CK_V);
          else PMG_CUDA(cudaGraphLaunch(graph_for(c, CK_V).exec, c.stream));
          break;
        case 7:
          c.ops->restrict_(c, level, c.lev[(size_t)level]->has_cf && !c.ops->cf_table() ? pmgdev::RM_RES : pmgdev::RM_FUSED);
          break;
        case 8: c.ops->fas(c, level - 1, true); break;
        case 9: enq_smooth(c, level, 1); break;  // one smoothing step (both colours)
        case 10:  // the V-cycle's prolongation (red cells left to the next half-sweep)
          c.prolong_dead = 0;
                c.ops->prolong(c, level, false);
                c.prolong_dead = -1;
          break;
        default: PMG_CUDA(cudaGraphLaunch(graph_for(c, CK_FMG_GUESS).exec, c.stream)); break;
      }
    };
    one(0);
    cudaGraphExec_t gx = nullptr;
    if (in_graph) {
      cudaGraph_t gr;
      PMG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < reps; ++k) one(k + 1);
      PMG_CUDA(cudaStreamEndCapture(c.stream, &gr));
      PMG_CUDA(cudaGraphInstantiate(&gx, gr, 0));
      cudaGraphDestroy(gr);
      PMG_CUDA(cudaGraphLaunch(gx, c.stream));  // warm
    }
    cudaEvent_t e0, e1;
    PMG_CUDA(cudaEventCreate(&e0));
    PMG_CUDA(cudaEventCreate(&e1));
    PMG_CUDA(cudaEventRecord(e0, c.stream));
    if (in_graph) PMG_CUDA(cudaGraphLaunch(gx, c.stream));
    else
      for (int k = 0; k < reps; ++k) one(k + 1);
    PMG_CUDA(cudaEventRecord(e1, c.stream));
    PMG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    PMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (gx) cudaGraphExecDestroy(gx);
    if (op >= 5) c.have_guess = true;
    *ms_avg = (double)ms / reps;
  });
}
// ---- multi-GPU hooks (paper_2205_09411_b200/distributed.py) ---------------
int pmg_b200_set_owned(pmg_b200_ctx* h, int level, const uint8_t* owned_by_slot) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 1);
    LevelDev& d = *c.lev[(size_t)level];
    if (c.owned.size() < (size_t)c.mesh.L + 1) c.owned.resize((size_t)c.mesh.L + 1);
    auto& o = c.owned[(size_t)level];
    if (owned_by_slot) {
      o.assign(owned_by_slot, owned_by_slot + d.nb);
      d.own.upload(o, c.stream);
      d.has_own = true;
    } else {
      o.clear();
      d.has_own = false;
    }
    d.n_own = 0;
    for (int s = 0; s < d.nb; ++s) d.n_own += own_slot(c, level, s) ? 1 : 0;
    if (c.st.valid) upload_stencils(c);
    set_views(c);
    invalidate_graphs(c);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
void* pmg_b200_level_field_ptr(pmg_b200_ctx* h, int var, int level) {
  void* out = nullptr;
  guard(h, [&](Ctx& c) {
    need_level(c, level, 1);
    LevelDev& d = *c.lev[(size_t)level];
    require(var >= 0 && var <= 3, "var must be PHI, RHS, RES or OLD");
    out = var == 0 ? (void*)d.phi.p : var == 1 ? (void*)d.rhs.p : var == 2 ? (void*)d.res.p : (void*)d.old.p;
  });
  return out;
}
int pmg_b200_restrict_only(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 2);
    enq_restrict_only(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_fas_level(pmg_b200_ctx* h, int level) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 1);
    c.ops->fas(c, level, true);
    if (c.lev[(size_t)level]->has_cfold) c.ops->cfold(c, level);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int pmg_b200_level_record(pmg_b200_ctx* h, int level, double* out3) {
  return guard(h, [&](Ctx& c) {
    need_level(c, level, 1);
    PMG_CUDA(cudaMemsetAsync(c.rec.p + level, 0, sizeof(pmgdev::Rec), c.stream));
    c.ops->record(c, level);
    pmgdev::Rec r;
    PMG_CUDA(cudaMemcpyAsync(&r, c.rec.p + level, sizeof(r), cudaMemcpyDeviceToHost, c.stream));
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    out3[0] = r.max;
    out3[1] = r.sumsq;
    out3[2] = (double)r.count;
  });
}

int pmg_b200_coarse_info(pmg_b200_ctx* h, int32_t* iters, double* rel) {
  return guard(h, [&](Ctx& c) {
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    *iters = (int32_t)c.h_out[3];
    *rel = c.h_out[2];
  });
}
int pmg_b200_set_partition(pmg_b200_ctx* h, int world, int rank, int split_level, const int32_t* owner_of_block) {
  return guard(h, [&](Ctx& c) { set_partition(c, world, rank, split_level, owner_of_block); });
}
int pmg_b200_nccl_unique_id(unsigned char* out) {
  if (!out) return PMG_ERR_INVALID_ARG;
  NcclApi& n = nccl_api();
  if (!n.ok) return PMG_ERR_CUDA;
  ncclUniqueId id;
  if (n.GetUniqueId(&id) != ncclSuccess) return PMG_ERR_CUDA;
  std::memcpy(out, id.internal, sizeof(id.internal));
  return PMG_OK;
}
int pmg_b200_dist_init_nccl(pmg_b200_ctx* h, const unsigned char* id) {
  return guard(h, [&](Ctx& c) {
    require(c.dist != nullptr, "no partition (call pmg_b200_set_partition)", PMG_ERR_STATE);
    NcclApi& n = nccl_api();
    require(n.ok, "NCCL unavailable: " + n.why, PMG_ERR_CUDA);
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    DistState& ds = *c.dist;
    if (ds.comm) {
      PMG_NCCL(n.CommDestroy(ds.comm));
      ds.comm = nullptr;
    }
    PMG_NCCL(n.CommInitRank(&ds.comm, ds.world, uid, ds.rank));
    ds.transport = TR_NCCL;
    invalidate_graphs(c);
  });
}
int pmg_b200_dist_local_group(int n, pmg_b200_ctx* const* ctxs) {
  if (n < 1 || !ctxs) return PMG_ERR_INVALID_ARG;
  auto grp = std::make_shared<LocalGroup>();
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r] || !ctxs[r]->c.dist) return PMG_ERR_STATE;
    grp->ctx.push_back(&ctxs[r]->c);
  }
  for (int r = 0; r < n; ++r) {
    DistState& ds = *ctxs[r]->c.dist;
    if (ds.world != n || ds.rank != r) {
      ctxs[r]->c.err = "local group: context " + std::to_string(r) + " is not rank " + std::to_string(r) +
                       " of a " + std::to_string(n) + "-rank partition";
      return PMG_ERR_STATE;
    }
  }
  for (int r = 0; r < n; ++r) {
    DistState& ds = *ctxs[r]->c.dist;
    ds.group = grp;
    ds.transport = TR_LOCAL;
    invalidate_graphs(ctxs[r]->c);
  }
  return PMG_OK;
}
int pmg_b200_dist_v_cycle_async(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) { launch_dist_cycle(c); });
}
int pmg_b200_dist_v_cycle(pmg_b200_ctx* h, pmg_cycle_stats_t* out) {
  return guard(h, [&](Ctx& c) {
    launch_dist_cycle(c);
    cycle_result(c, out);
  });
}
int pmg_b200_dist_info(pmg_b200_ctx* h, int32_t* out6) {
  return guard(h, [&](Ctx& c) {
    require(c.dist != nullptr, "no partition", PMG_ERR_STATE);
    const DistState& ds = *c.dist;
    long long halo = 0;
    for (const auto& lv : ds.halo) halo += lv[2].nr;
    out6[0] = ds.world;
    out6[1] = ds.split;
    out6[2] = ds.transport;
    out6[3] = (int32_t)std::min<long long>(halo, INT32_MAX);
    out6[4] = ds.g.exec ? ds.g.kernels : 0;
    out6[5] = ds.g.exec ? 1 : 0;
  });
}

int pmg_b200_field_bytes(pmg_b200_ctx* h, double* out) {
  return guard(h, [&](Ctx& c) {
    need_mesh(c);
    double b = 0;
    for (int l = 1; l <= c.mesh.L; ++l) {
      const LevelDev& d = *c.lev[(size_t)l];
      b += (double)(d.phi.bytes() + d.rhs.bytes() + d.old.bytes() + d.res.bytes());
    }
    *out = b;
  });
}
void* pmg_b200_host_buffer(pmg_b200_ctx* h, size_t bytes) {
  void* out = nullptr;
  guard(h, [&](Ctx& c) {
    if (c.h_buf_bytes < bytes) {
      if (c.h_buf) PMG_CUDA(cudaFreeHost(c.h_buf));
      c.h_buf = nullptr;
      c.h_buf_bytes = 0;
      PMG_CUDA(cudaMallocHost(&c.h_buf, bytes));
      c.h_buf_bytes = bytes;
    }
    out = c.h_buf;
  });
  return out;
}
int pmg_b200_synchronize(pmg_b200_ctx* h) {
  return guard(h, [&](Ctx& c) { PMG_CUDA(cudaStreamSynchronize(c.stream)); });
}

}  // extern "C"
