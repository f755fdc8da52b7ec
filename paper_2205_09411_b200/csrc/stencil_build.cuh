// stencil_build.cuh -- K5: level-set stencil construction on the GPU.
//
// Replaces build_stencils / build_block_stencil (stencil.hpp:125-222) and the
// level-set machinery it runs (levelset.hpp:80-382).  Three passes:
//   1. k_block_flag   one CTA per block: any interior f <= 0, else the boundary
//                     mask |f| < L ||grad f|| over the (N+2)^D cells incl. corners
//                     (stencil.hpp:143-161)
//   2. k_cell_rows    one thread per interior cell of a flagged block: inside
//                     row with pin_obj, or 2D line searches (golden bracketing +
//                     bisection), thin-object rescue, make_row (stencil.hpp:166-191);
//      k_cell_search  for composites of many objects, one WARP per boundary
//                     candidate: the lanes evaluate the children (WarpEval)
//   3. k_compact      one CTA per flagged block: rows compacted in interior-index
//                     order (BlockStencil::set_row order, stencil.hpp:75-79)
// Every decision is an fp64 threshold test; with --fmad=false and the
// reference's operation order the flags, patterns and coefficients are
// bit-identical to the CPU build.  The heart/astroid shapes call std::cbrt,
// which is not correctly rounded in glibc; libm_cbrt restates glibc's
// algorithm so those shapes stay bit-exact too.
#pragma once
#include <cfloat>
#include <cmath>

#include "ctx.h"

namespace pmgdev {

struct LsfDev {
  int n;  // descriptors: [0] = root, [1..n-1] = composite children
  const pmg_lsf_t* d;
};

template <int D>
struct V {
  double v[3];
};

template <int D>
__device__ __forceinline__ double vnorm(const double* a) {
  double s = 0;
  for (int k = 0; k < D; ++k) s += a[k] * a[k];
  return sqrt(s);
}

// std::cbrt as the reference's host libm computes it: glibc 2.39 (the image's
// libc) sysdeps/ieee754/dbl-64/s_cbrt.c -- a degree-6 polynomial seed for
// cbrt(m), m in [0.5,1), one Halley step u (u^3 + 2m) / (2u^3 + m), scaled by
// 2^(e mod 3 / 3) and 2^(e/3) (C truncating division).  Pinned against the
// host libm on 2e7 random inputs (0 mismatches, tests/test_host.py).
__device__ __forceinline__ double libm_cbrt(double x) {
  if (x == 0.0 || isnan(x) || isinf(x)) return x + x;
  int xe;
  const double xm = frexp(fabs(x), &xe);
  const double u =
      (0.354895765043919860 +
       ((1.50819193781584896 +
         ((-2.11499494167371287 +
           ((2.44693122563534430 +
             ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) * xm)) *
            xm)) *
          xm)) *
        xm));
  const double t2 = u * u * u;
  const double c2 = 1.2599210498948731648, s2 = 1.5874010519681994748;
  double f;
  switch (2 + xe % 3) {
    case 0: f = 1.0 / s2; break;
    case 1: f = 1.0 / c2; break;
    case 3: f = c2; break;
    case 4: f = s2; break;
    default: f = 1.0; break;
  }
  const double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * f;
  return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

template <int D>
__device__ double eval_simple(const pmg_lsf_t& s, const double* x) {
  switch (s.shape) {
    case PMG_SHAPE_NONE:
      return 1.0;
    case PMG_SHAPE_SPHERE: {
      double a[3];
      for (int k = 0; k < D; ++k) a[k] = x[k] - s.center[k];
      return vnorm<D>(a) - s.radius;
    }
    case PMG_SHAPE_ROD: {  // dist_point_segment2 (levelset.hpp:56-70)
      double ab2 = 0, t = 0;
      for (int k = 0; k < D; ++k) {
        ab2 += (s.seg_b[k] - s.seg_a[k]) * (s.seg_b[k] - s.seg_a[k]);
        t += (x[k] - s.seg_a[k]) * (s.seg_b[k] - s.seg_a[k]);
      }
      if (ab2 > 0) {
        t = t / ab2;
        t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
      } else {
        t = 0.0;
      }
      double d2 = 0;
      for (int k = 0; k < D; ++k) {
        const double p = s.seg_a[k] + t * (s.seg_b[k] - s.seg_a[k]);
        d2 += (x[k] - p) * (x[k] - p);
      }
      return sqrt(d2) - s.radius;
    }
    default:
      break;
  }
  double p, q;
  if (D == 2) {
    p = s.scale * (x[0] - s.shift_p);
    q = s.scale * (x[1] - s.shift_q);
  } else if (s.cylindrical) {
    p = s.scale * (sqrt(x[0] * x[0] + x[1] * x[1]) - s.shift_p);
    q = s.scale * (x[2] - s.shift_q);
  } else {
    p = s.scale * (x[0] - s.shift_p);
    q = s.scale * (x[1] - s.shift_q);
  }
  switch (s.shape) {
    case PMG_SHAPE_SPHEROID:
      return sqrt(8 * p * p + q * q) - 1.0;
    case PMG_SHAPE_RHOMBUS:
      return 8 * fabs(p) + fabs(q) - 1.5;
    case PMG_SHAPE_HEART: {
      const double u = q - libm_cbrt(p * p);
      return p * p + u * u - 1.0;
    }
    case PMG_SHAPE_ASTROID:
      return libm_cbrt(p * p) / 0.8 + libm_cbrt(q * q) / 1.5 - 0.8;
    default:
      return 0.0;
  }
}

template <int D>
__device__ __forceinline__ double lsf_eval(const LsfDev& L, const double* x) {
  if (L.d[0].shape != PMG_SHAPE_COMPOSITE_MIN) return eval_simple<D>(L.d[0], x);
  double f = DBL_MAX * 2.0;  // +inf
  for (int i = 1; i < L.n; ++i) {
    const double e = eval_simple<D>(L.d[i], x);
    f = e < f ? e : f;  // std::min(f, e)
  }
  return f;
}

template <int D>
__device__ __forceinline__ int lsf_attaining(const LsfDev& L, const double* x) {
  if (L.d[0].shape != PMG_SHAPE_COMPOSITE_MIN) return 0;
  int best = 0;
  double fb = DBL_MAX * 2.0;
  for (int i = 1; i < L.n; ++i) {
    const double f = eval_simple<D>(L.d[i], x);
    if (f < fb) {
      fb = f;
      best = i - 1;
    }
  }
  return best;
}

// Level-set evaluators for the line searches.  SeqEval: one thread evaluates
// the composite min child by child (lsf_eval / lsf_attaining).  WarpEval: the
// 32 lanes of a warp evaluate the children of a composite in parallel (lane k
// takes children k, k+32, ...) and reduce (value, index) lexicographically --
// the minimum value and the first child attaining it, exactly what the
// sequential strict-< scan yields (levelset.hpp:127-148), so decisions stay
// bit-identical.  Every lane returns the same result; the callers' control
// flow is then uniform across the warp.
template <int D>
struct SeqEval {
  LsfDev L;
  __device__ __forceinline__ double f(const double* x) const { return lsf_eval<D>(L, x); }
  __device__ __forceinline__ int obj(const double* x) const { return lsf_attaining<D>(L, x); }
};
template <int D>
struct WarpEval {
  LsfDev L;
  __device__ __forceinline__ void reduce(const double* x, double& v, int& idx) const {
    v = DBL_MAX * 2.0;
    idx = 0x7fffffff;
    for (int i = 1 + (int)(threadIdx.x & 31); i < L.n; i += 32) {
      const double e = eval_simple<D>(L.d[i], x);
      if (e < v) v = e, idx = i;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov < v || (!(v < ov) && oi < idx)) v = ov, idx = oi;
    }
  }
  __device__ __forceinline__ double f(const double* x) const {
    double v;
    int i;
    reduce(x, v, i);
    return v;
  }
  __device__ __forceinline__ int obj(const double* x) const {
    double v;
    int i;
    reduce(x, v, i);
    return i - 1;
  }
};

template <int D, class E>
__device__ __forceinline__ void lsf_gradient(const E& ev, const double* x, double dx, double* g) {
  for (int k = 0; k < D; ++k) {
    double xp[3], xm[3];
    for (int a = 0; a < D; ++a) xp[a] = xm[a] = x[a];
    xp[k] += dx;
    xm[k] -= dx;
    g[k] = (ev.f(xp) - ev.f(xm)) / (2 * dx);
  }
}

// boundary_candidate (levelset.hpp:277-289)
template <int D, class E>
__device__ __forceinline__ bool boundary_candidate(const E& ev, const double* x, double dx, double safety) {
  const double Ls = safety * sqrt((double)D) * dx;
  double g[3];
  lsf_gradient<D>(ev, x, dx, g);
  return fabs(ev.f(x)) < Ls * vnorm<D>(g);
}

// p = a + t (b - a)   (Vec operator*, operator+, core.hpp:27-55)
template <int D>
__device__ __forceinline__ void along(const double* a, const double* b, double t, double* p) {
  for (int k = 0; k < D; ++k) p[k] = a[k] + (b[k] - a[k]) * t;
}

template <int D, class E>
__device__ double bisect_t(const E& ev, const double* a, const double* b, double lo, double hi, double eps) {
  while (hi - lo > eps) {
    const double mid = 0.5 * (lo + hi);
    double p[3];
    along<D>(a, b, mid, p);
    if (ev.f(p) > 0)
      lo = mid;
    else
      hi = mid;
  }
  return 0.5 * (lo + hi);
}

// find_root_position (levelset.hpp:223-257)
template <int D, class E>
__device__ double find_root_position(const E& ev, const double* a, const double* b, const pmg_stencil_cfg_t& cfg) {
  const double fa = ev.f(a);
  if (fa * ev.f(b) <= 0) return bisect_t<D>(ev, a, b, 0.0, 1.0, cfg.eps_tol);
  const double invphi = 0.6180339887498949;
  double lo = 0.0, hi = 1.0;
  double t1 = hi - invphi * (hi - lo);
  double t2 = lo + invphi * (hi - lo);
  double p[3];
  along<D>(a, b, t1, p);
  double g1 = fa * ev.f(p);
  along<D>(a, b, t2, p);
  double g2 = fa * ev.f(p);
  if (g1 <= 0) return bisect_t<D>(ev, a, b, 0.0, t1, cfg.eps_tol);
  if (g2 <= 0) return bisect_t<D>(ev, a, b, 0.0, t2, cfg.eps_tol);
  for (int it = 0; it < cfg.max_bracket_iters && hi - lo > cfg.eps_tol; ++it) {
    if (g1 <= g2) {
      hi = t2;
      t2 = t1;
      g2 = g1;
      t1 = hi - invphi * (hi - lo);
      along<D>(a, b, t1, p);
      g1 = fa * ev.f(p);
      if (g1 <= 0) return bisect_t<D>(ev, a, b, 0.0, t1, cfg.eps_tol);
    } else {
      lo = t1;
      t1 = t2;
      g1 = g2;
      t2 = lo + invphi * (hi - lo);
      along<D>(a, b, t2, p);
      g2 = fa * ev.f(p);
      if (g2 <= 0) return bisect_t<D>(ev, a, b, 0.0, t2, cfg.eps_tol);
    }
  }
  return -1.0;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// Dense per-cell row written by pass 2 (one per interior cell of a flagged block).
struct RowScratch {
  double center;
  double nb[6], bc[6], d[6];
  int8_t obj[6];
  uint8_t mask;
  int8_t pin;
  uint8_t has;  // 1 = special row (inside or cut)
};

struct BuildArgs {
  int nflag;
  const int32_t* flagged;   // block ids
  const double* origin;     // [nb*3] by block id
  const double* dx;         // [nb]
  RowScratch* rows;         // [nflag * NI]
  int32_t* counts;          // [nflag]
  uint8_t* flag;            // [nb]
};

// lip1: every piece of the level set is a Euclidean distance (spheres, rods),
// so f is 1-Lipschitz and each central-difference gradient component is at
// most 1: a block whose padded cells all lie farther than the mask band from
// the boundary is decided from its centre alone (no cell can be inside or
// pass |f| < L ||grad f|| <= L sqrt(D)); the same flag, without the per-cell work.
template <int D, int N>
__global__ void __launch_bounds__(256) k_block_flag(LsfDev L, const double* __restrict__ origin,
                                                    const double* __restrict__ dx, int nb,
                                                    double safety, uint8_t* flag, int lip1) {
  pdl_begin();
  __shared__ int any;
  const int b = blockIdx.x;
  if (b >= nb) return;
  const double h = dx[b];
  if (lip1) {
    double xc[3];
    for (int k = 0; k < D; ++k) xc[k] = origin[b * 3 + k] + 0.5 * N * h;
    const double fc = lsf_eval<D>(L, xc);
    const double reach = sqrt((double)D) * 0.5 * (N + 1) * h;  // centre to the farthest padded cell centre
    const double band = safety * sqrt((double)D) * h * sqrt((double)D);
    const double slack = 1e-9 * (1.0 + fabs(fc) + h);
    if (fc - reach > band + slack) {  // every padded cell outside and beyond the band
      if (threadIdx.x == 0) flag[b] = 0;
      return;
    }
    if (fc + 0.5 * N * h * sqrt((double)D) < -slack) {  // every interior cell inside
      if (threadIdx.x == 0) flag[b] = 1;
      return;
    }
  }
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  constexpr int NI = D == 2 ? N * N : N * N * N;
  for (int ii = threadIdx.x; ii < NI; ii += blockDim.x) {
    const int i[3] = {ii % N, (ii / N) % N, D == 3 ? ii / (N * N) : 0};
    double x[3];
    for (int k = 0; k < D; ++k) x[k] = origin[b * 3 + k] + (i[k] + 0.5) * h;
    if (lsf_eval<D>(L, x) <= 0) any = 1;
  }
  __syncthreads();
  if (!any) {
    constexpr int S1 = N + 2;
    constexpr int S = D == 2 ? S1 * S1 : S1 * S1 * S1;
    for (int q = threadIdx.x; q < S; q += blockDim.x) {
      if (any) break;  // early exit (the result is an OR)
      const int i[3] = {q % S1 - 1, (q / S1) % S1 - 1, D == 3 ? q / (S1 * S1) - 1 : 0};
      double x[3];
      for (int k = 0; k < D; ++k) x[k] = origin[b * 3 + k] + (i[k] + 0.5) * h;
      if (boundary_candidate<D>(SeqEval<D>{L}, x, h, 0.0 + safety)) any = 1;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) flag[b] = any ? 1 : 0;
}

__device__ __forceinline__ void row_init(RowScratch& r) {
  r.center = 0;
  for (int f = 0; f < 6; ++f) {
    r.nb[f] = 0;
    r.bc[f] = 0;
    r.d[f] = 1.0;
    r.obj[f] = -1;
  }
  r.mask = PMG_SOLVED;
  r.pin = -1;
  r.has = 0;
}

// cell centre of interior cell t of the flagged-block list
template <int D, int N>
__device__ __forceinline__ void cell_at(const BuildArgs& A, long long t, double* x, double& h) {
  constexpr int NI = D == 2 ? N * N : N * N * N;
  const int b = A.flagged[(int)(t / NI)];
  const int ii = (int)(t % NI);
  h = A.dx[b];
  const int i[3] = {ii % N, (ii / N) % N, D == 3 ? ii / (N * N) : 0};
  for (int k = 0; k < D; ++k) x[k] = A.origin[b * 3 + k] + (i[k] + 0.5) * h;
}

// A boundary-candidate cell (not inside): cell_distances, the thin-object
// rescue and make_row (stencil.hpp:166-191, levelset.hpp:293-382).
template <int D, class E>
__device__ void cell_search(const E& ev, const double* x, double h, double fc, const pmg_stencil_cfg_t& cfg,
                            RowScratch& r) {
  double dd[6];
  int8_t ob[6];
  for (int f = 0; f < 2 * D; ++f) {
    dd[f] = 1.0;
    ob[f] = -1;
  }
  bool cut = false;
  for (int f = 0; f < 2 * D; ++f) {  // cell_distances (levelset.hpp:313-327)
    double nbp[3];
    for (int k = 0; k < D; ++k) nbp[k] = x[k];
    nbp[f >> 1] += ((f & 1) ? 1 : -1) * h;
    const double tr = find_root_position<D>(ev, x, nbp, cfg);
    if (tr < 0) continue;
    const double d = clampd(tr, cfg.d_min, 1.0);
    if (d < 1.0) {
      double p[3];
      along<D>(x, nbp, tr, p);
      dd[f] = d;
      ob[f] = (int8_t)ev.obj(p);
      cut = true;
    }
  }
  if (!cut && cfg.thin_rescue && h > cfg.w_min) {
    // resolve_thin_boundary (levelset.hpp:344-382)
    const double fa = fc;
    const int max_steps = (int)(h / cfg.w_min);
    double y[3];
    for (int k = 0; k < D; ++k) y[k] = x[k];
    for (int step = 0; step < max_steps; ++step) {
      double g[3];
      lsf_gradient<D>(ev, y, h, g);
      const double gn = vnorm<D>(g);
      if (gn == 0) break;
      const double sc = cfg.w_min / gn;
      for (int k = 0; k < D; ++k) y[k] -= g[k] * sc;
      if (fa * ev.f(y) > 0) continue;
      const double tt = bisect_t<D>(ev, x, y, 0.0, 1.0, cfg.eps_tol);
      double root[3], rc[3];
      along<D>(x, y, tt, root);
      for (int k = 0; k < D; ++k) rc[k] = root[k] - x[k];
      const double hd = clampd(vnorm<D>(rc) / h, cfg.d_min, 1.0);
      const int hobj = ev.obj(root);
      int hdir = 0;
      double best = DBL_MAX * 2.0;
      for (int f = 0; f < 2 * D; ++f) {
        double nbp[3];
        for (int k = 0; k < D; ++k) nbp[k] = x[k];
        nbp[f >> 1] += ((f & 1) ? 1 : -1) * h;
        double rn[3];
        for (int k = 0; k < D; ++k) rn[k] = root[k] - nbp[k];
        const double dist = vnorm<D>(rn);
        if (dist < best) {
          best = dist;
          hdir = f;
        }
      }
      dd[hdir] = hd;
      ob[hdir] = (int8_t)hobj;
      cut = hd < 1.0;
      for (int f = 0; f < 2 * D && !cut; ++f) cut = dd[f] < 1.0;
      break;
    }
  }
  if (cut) {  // make_row (stencil.hpp:84-110)
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
    for (int f = 0; f < 2 * D; ++f) r.d[f] = dd[f];
    r.has = 1;
  }
}

// One thread per interior cell of a flagged block.  cand == nullptr: the
// whole row here (a plain or few-child level set).  Otherwise the boundary
// candidates are only listed in cand[] for k_cell_search.
template <int D, int N>
__global__ void __launch_bounds__(128) k_cell_rows(LsfDev L, BuildArgs A, pmg_stencil_cfg_t cfg,
                                                   long long* cand, int* n_cand) {
  pdl_begin();
  constexpr int NI = D == 2 ? N * N : N * N * N;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)A.nflag * NI) return;
  const int fb = (int)(t / NI);
  double x[3], h;
  cell_at<D, N>(A, t, x, h);
  RowScratch r;
  row_init(r);
  const SeqEval<D> ev{L};
  const double fc = ev.f(x);
  if (fc <= 0) {  // inside: identity row pinned to the attaining object
    r.mask = PMG_INSIDE;
    r.pin = (int8_t)ev.obj(x);
    r.center = 1.0;
    r.has = 1;
  } else if (boundary_candidate<D>(ev, x, h, cfg.boundary_safety)) {
    if (cand) {
      cand[atomicAdd(n_cand, 1)] = t;
      return;  // the row is written by k_cell_search
    }
    cell_search<D>(ev, x, h, fc, cfg, r);
  }
  A.rows[t] = r;
  if (r.has) atomicAdd(&A.counts[fb], 1);
}

// One warp per boundary-candidate cell of a composite level set with many
// children: the lanes evaluate the children (WarpEval), so the line searches
// run without divergence.
template <int D, int N>
__global__ void __launch_bounds__(128) k_cell_search(LsfDev L, BuildArgs A, pmg_stencil_cfg_t cfg,
                                                     const long long* __restrict__ cand, const int* n_cand) {
  pdl_begin();
  constexpr int NI = D == 2 ? N * N : N * N * N;
  const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (w >= *n_cand) return;
  const long long t = cand[w];
  double x[3], h;
  cell_at<D, N>(A, t, x, h);
  RowScratch r;
  row_init(r);
  const WarpEval<D> ev{L};
  cell_search<D>(ev, x, h, ev.f(x), cfg, r);
  if ((threadIdx.x & 31) == 0) {
    A.rows[t] = r;
    if (r.has) atomicAdd(&A.counts[(int)(t / NI)], 1);
  }
}

// One CTA per flagged block: exclusive scan of `has` in interior order.
template <int D, int N>
__global__ void __launch_bounds__(1024) k_compact(BuildArgs A, const int32_t* __restrict__ offs,
                                                  int32_t* row_of, double* center, double* nbv,
                                                  double* bcv, double* dv, int8_t* objv,
                                                  uint8_t* maskv, int8_t* pinv, int32_t* linv) {
  pdl_begin();
  constexpr int NI = D == 2 ? N * N : N * N * N;
  constexpr int F = 2 * D;
  constexpr int PER = (NI + 1023) / 1024;
  __shared__ int wsum[32];
  const int fb = blockIdx.x;
  const RowScratch* rs = A.rows + (size_t)fb * NI;
  const int base = threadIdx.x * PER;
  int cnt = 0;
  for (int q = 0; q < PER; ++q)
    if (base + q < NI && rs[base + q].has) ++cnt;
  // block exclusive scan
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  int r = incl - cnt + (wid > 0 ? wsum[wid - 1] : 0);
  const int s1 = N + 2;
  for (int q = 0; q < PER; ++q) {
    const int ii = base + q;
    if (ii >= NI) break;
    const RowScratch& c = rs[ii];
    if (!c.has) {
      row_of[(size_t)fb * NI + ii] = -1;
      continue;
    }
    row_of[(size_t)fb * NI + ii] = r;
    const size_t g = (size_t)offs[fb] + r;
    center[g] = c.center;
    for (int f = 0; f < F; ++f) {
      nbv[g * F + f] = c.nb[f];
      bcv[g * F + f] = c.bc[f];
      dv[g * F + f] = c.d[f];
      objv[g * F + f] = c.obj[f];
    }
    maskv[g] = c.mask;
    pinv[g] = c.pin;
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    linv[g] = (i + 1) + (j + 1) * s1 + (D == 3 ? (k + 1) * s1 * s1 : 0);
    ++r;
  }
}

}  // namespace pmgdev

namespace pmghost {

// composite level sets with at least this many children search their
// boundary cells one warp per cell (the lanes evaluate the children)
constexpr int kWarpSearchChildren = 8;

template <int D, int N>
void run_stencil_build(Ctx& c, const pmg_lsf_t* lsf, int n_lsf, const pmg_stencil_cfg_t* cfg) {
  using namespace pmgdev;
  constexpr int NI = D == 2 ? N * N : N * N * N;
  constexpr int F = 2 * D;
  // RootSearchConfig::validate (levelset.hpp:175-182)
  if (!(cfg->eps_tol > 0 && cfg->eps_tol < 1)) throw PmgError(PMG_ERR_INVALID_ARG, "eps_tol must be in (0, 1)");
  const int needed = (int)std::ceil(std::log(cfg->eps_tol) / std::log(0.6180339887498949));
  if (cfg->max_bracket_iters < needed)
    throw PmgError(PMG_ERR_INVALID_ARG, "max_bracket_iters too small to reach eps_tol resolution");
  if (!(cfg->d_min > 0 && cfg->d_min < 1)) throw PmgError(PMG_ERR_INVALID_ARG, "d_min must be in (0, 1)");
  const bool composite = lsf[0].shape == PMG_SHAPE_COMPOSITE_MIN;
  const int n_obj = composite ? n_lsf - 1 : 1;
  if (n_obj > 127) throw PmgError(PMG_ERR_INVALID_ARG, "at most 127 boundary objects (int8 ids)");
  if (composite && n_obj < 1) throw PmgError(PMG_ERR_INVALID_ARG, "composite level set without children");
  const HostMesh& m = c.mesh;
  const int nb = m.nb;
  std::vector<pmg_lsf_t> descs(lsf, lsf + (composite ? n_lsf : 1));
  DevBuf<pmg_lsf_t> d_lsf;
  d_lsf.upload(descs, c.stream);
  LsfDev L{(int)descs.size(), d_lsf.p};
  DevBuf<double> d_origin, d_dx;
  d_origin.upload(m.origin, c.stream);
  d_dx.upload(m.dx, c.stream);
  DevBuf<uint8_t> d_flag;
  d_flag.alloc((size_t)nb);
  int lip1 = 1;  // only Euclidean-distance pieces (k_block_flag's far-block test)
  for (const auto& dsc : descs)
    if (dsc.shape != PMG_SHAPE_SPHERE && dsc.shape != PMG_SHAPE_ROD && dsc.shape != PMG_SHAPE_COMPOSITE_MIN) lip1 = 0;
  k_block_flag<D, N><<<nb, 256, 0, c.stream>>>(L, d_origin.p, d_dx.p, nb, cfg->boundary_safety,
                                               d_flag.p, lip1);
  PMG_CUDA(cudaGetLastError());
  std::vector<uint8_t> flag((size_t)nb);
  PMG_CUDA(cudaMemcpyAsync(flag.data(), d_flag.p, (size_t)nb, cudaMemcpyDeviceToHost, c.stream));
  PMG_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<int32_t> flagged;
  for (int b = 0; b < nb; ++b)
    if (flag[(size_t)b]) flagged.push_back(b);
  HostStencils& st = c.st;
  st = HostStencils{};
  c.devrows.reset();
  st.valid = true;
  st.boundary.assign((size_t)nb, 0);
  st.row_count.assign((size_t)nb, 0);
  st.row_start.assign((size_t)nb + 1, 0);
  st.NI = NI;
  st.row_page.assign((size_t)nb, -1);
  st.row_pages.clear();
  st.phi_b.resize((size_t)n_obj);
  for (int o = 0; o < n_obj; ++o) st.phi_b[(size_t)o] = composite ? lsf[o + 1].boundary_value : lsf[0].boundary_value;
  const int nf = (int)flagged.size();
  if (nf > 0) {
    DevBuf<int32_t> d_flagged, d_counts, d_offs, d_rowof;
    DevBuf<RowScratch> d_rows;
    d_flagged.upload(flagged, c.stream);
    d_counts.alloc((size_t)nf);
    PMG_CUDA(cudaMemsetAsync(d_counts.p, 0, (size_t)nf * sizeof(int32_t), c.stream));
    d_rows.alloc((size_t)nf * NI);
    BuildArgs A{nf, d_flagged.p, d_origin.p, d_dx.p, d_rows.p, d_counts.p, d_flag.p};
    const long long tot = (long long)nf * NI;
    if (composite && n_obj >= kWarpSearchChildren) {
      // candidates listed by k_cell_rows, searched one warp per cell
      DevBuf<long long> d_cand;
      DevBuf<int> d_ncand;
      d_cand.alloc((size_t)tot);
      d_ncand.alloc(1);
      PMG_CUDA(cudaMemsetAsync(d_ncand.p, 0, sizeof(int), c.stream));
      k_cell_rows<D, N><<<(unsigned)((tot + 127) / 128), 128, 0, c.stream>>>(L, A, *cfg, d_cand.p, d_ncand.p);
      PMG_CUDA(cudaGetLastError());
      int ncand = 0;
      PMG_CUDA(cudaMemcpyAsync(&ncand, d_ncand.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      PMG_CUDA(cudaStreamSynchronize(c.stream));
      if (ncand > 0)
        k_cell_search<D, N><<<(unsigned)(((long long)ncand * 32 + 127) / 128), 128, 0, c.stream>>>(
            L, A, *cfg, d_cand.p, d_ncand.p);
      PMG_CUDA(cudaGetLastError());
    } else {
      k_cell_rows<D, N><<<(unsigned)((tot + 127) / 128), 128, 0, c.stream>>>(L, A, *cfg, (long long*)nullptr,
                                                                              (int*)nullptr);
      PMG_CUDA(cudaGetLastError());
    }
    std::vector<int32_t> counts((size_t)nf), offs((size_t)nf + 1, 0);
    PMG_CUDA(cudaMemcpyAsync(counts.data(), d_counts.p, (size_t)nf * 4, cudaMemcpyDeviceToHost, c.stream));
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    for (int i = 0; i < nf; ++i) offs[(size_t)i + 1] = offs[(size_t)i] + counts[(size_t)i];
    const size_t R = (size_t)offs[(size_t)nf];
    d_offs.upload(offs, c.stream);
    d_rowof.alloc((size_t)nf * NI);
    DevBuf<double> d_center, d_nb, d_bc, d_d;
    DevBuf<int8_t> d_obj, d_pin;
    DevBuf<uint8_t> d_mask;
    DevBuf<int32_t> d_lin;
    d_center.alloc(R);
    d_nb.alloc(R * F);
    d_bc.alloc(R * F);
    d_d.alloc(R * F);
    d_obj.alloc(R * F);
    d_pin.alloc(R);
    d_mask.alloc(R);
    d_lin.alloc(R);
    k_compact<D, N><<<nf, 1024, 0, c.stream>>>(A, d_offs.p, d_rowof.p, d_center.p, d_nb.p, d_bc.p,
                                               d_d.p, d_obj.p, d_mask.p, d_pin.p, d_lin.p);
    PMG_CUDA(cudaGetLastError());
    std::vector<int32_t>& rowof = st.row_pages;  // the flagged blocks' pages, in block-id order
    rowof.resize((size_t)nf * NI);
    st.center.resize(R);
    st.nb.resize(R * F);
    st.bc.resize(R * F);
    st.d.resize(R * F);
    st.obj.resize(R * F);
    st.pin.resize(R);
    st.mask.resize(R);
    st.lin.resize(R);
    auto dl = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) PMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    };
    dl(rowof.data(), d_rowof.p, rowof.size() * 4);
    dl(st.center.data(), d_center.p, R * 8);
    dl(st.nb.data(), d_nb.p, R * F * 8);
    dl(st.bc.data(), d_bc.p, R * F * 8);
    dl(st.d.data(), d_d.p, R * F * 8);
    dl(st.obj.data(), d_obj.p, R * F);
    dl(st.pin.data(), d_pin.p, R);
    dl(st.mask.data(), d_mask.p, R);
    dl(st.lin.data(), d_lin.p, R * 4);
    PMG_CUDA(cudaStreamSynchronize(c.stream));
    // the device copy the per-level row arrays are gathered from (upload_stencils)
    auto DR = std::make_unique<DevRows>();
    DR->center = std::move(d_center);
    DR->nb = std::move(d_nb);
    DR->bc = std::move(d_bc);
    DR->d = std::move(d_d);
    DR->obj = std::move(d_obj);
    DR->pin = std::move(d_pin);
    DR->mask = std::move(d_mask);
    DR->rowof = std::move(d_rowof);
    c.devrows = std::move(DR);
    // rows are concatenated in block-id order; flagged[] is increasing
    for (int i = 0; i < nf; ++i) {
      const int b = flagged[(size_t)i];
      st.boundary[(size_t)b] = 1;
      st.row_count[(size_t)b] = counts[(size_t)i];
      st.row_page[(size_t)b] = i;
    }
  }
  for (int b = 0; b < nb; ++b) st.row_start[(size_t)b + 1] = st.row_start[(size_t)b] + st.row_count[(size_t)b];
}

}  // namespace pmghost
