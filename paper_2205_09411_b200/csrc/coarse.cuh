// coarse.cuh -- K6: on-chip Jacobi-BiCGStab for the level-1 system.
//
// Replaces coarse_solve + detail::bicgstab (multigrid.hpp:194-280, 442-472).
// The assembled CoarseSystem (assemble_level, multigrid.hpp:62-190) is, for the
// single root block, a 7-point (5-point in 2D) operator on the block's cells.
// We store it CELL-indexed: per cell a diagonal, a bitmask of neighbours whose
// coefficient is the uniform w = 1/dx^2, and for the few boundary-modified rows
// an explicit 2D-vector of off-diagonals.  Row sums are evaluated in the CSR's
// sorted-column order (z-, y-, x-, diag, x+, y+, z+).  Absent entries are added
// as exact zeros (0*x, x finite) instead of being skipped: the running sum
// starts at +0 and can never become -0, so s + (+-0) == s and every row is
// bit-identical to CoarseSystem::spmv.  The vectors the SpMV gathers live in a
// zero-padded (N+2)^D shared-memory image, so a row reads fixed offsets with no
// bounds tests.  Inside (pinned) cells carry zeros and are excluded from every
// dot product.
//
// One CTA of 1024 threads, CPT cells per thread; every dot product is one
// deterministic CTA reduction with a single barrier.  The iteration replays
// the reference's recurrences, stopping rules and breakdown checks exactly.
#pragma once
#include "kernels.cuh"

namespace pmgdev {

struct CoarseFast {
  const uint8_t* flags;     // [NI]: bits 0..2D-1 neighbour coef == w; bit 6 unknown; bit 7 special
  const double* diag;       // [NI]
  const int16_t* spec;      // [NI] special row ordinal or -1
  const double* spec_c;     // [n_spec * 2D] off-diagonals (0 where absent)
  const double* c0;         // [NI]
  const int32_t* ob_start;  // [NI+1] sparse cobj per cell (objects ascending)
  const int8_t* ob_obj;
  const double* ob_val;
  double w;
  double rel_tol;
  int max_iters;
  int fallback_ok;
  int n_unknowns;
  const int2* pins;  // level-1 pin list (cell address, object)
  int n_pins;
};

constexpr int kCoarseThreads = 512;  // 16 warps, CPT = 8 cells per thread in 3D N=16
constexpr int kCoarseWarps = kCoarseThreads / 32;

// deterministic CTA reduction of one / two values; `buf` must not be in use
// by another reduction that some thread may still be reading.
__device__ __forceinline__ double cta_sum1(double v, double* buf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) buf[wid] = v;
  __syncthreads();
  return warp_sum(lane < kCoarseWarps ? buf[lane] : 0.0);
}
__device__ __forceinline__ void cta_sum2(double& a, double& b, double* buf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    buf[wid] = a;
    buf[32 + wid] = b;
  }
  __syncthreads();
  a = warp_sum(lane < kCoarseWarps ? buf[lane] : 0.0);
  b = warp_sum(lane < kCoarseWarps ? buf[32 + lane] : 0.0);
}

template <int D, int N>
struct CoarseGeo {
  static constexpr int P = N + 2;
  static constexpr int PS = D == 2 ? P * P : P * P * P;
  static constexpr int NI = Geo<D, N>::NI;
  static constexpr int CPT = (NI + kCoarseThreads - 1) / kCoarseThreads;
  __device__ __forceinline__ static int pad(int ii) {
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    return (i + 1) + (j + 1) * P + (D == 3 ? (k + 1) * P * P : 0);
  }
};

// One row of A x, x a padded shared image, in CSR sorted-column order.
template <int D, int N>
__device__ __forceinline__ double coarse_row(const CoarseFast& C, const double* __restrict__ X,
                                             uint8_t f, double dg, int pi, int ii) {
  constexpr int P = N + 2;
  const double* x = X + pi;
  double s = 0;
  if (f & 0x80) {  // boundary-modified row: explicit coefficients
    const double* sc = C.spec_c + (size_t)C.spec[ii] * 2 * D;
    if (D == 3) s += sc[4] * x[-P * P];
    s += sc[2] * x[-P];
    s += sc[0] * x[-1];
    s += dg * x[0];
    s += sc[1] * x[1];
    s += sc[3] * x[P];
    if (D == 3) s += sc[5] * x[P * P];
    return s;
  }
  const double w = C.w;
  if (D == 3) s += ((f & 16) ? w : 0.0) * x[-P * P];
  s += ((f & 4) ? w : 0.0) * x[-P];
  s += ((f & 1) ? w : 0.0) * x[-1];
  s += dg * x[0];
  s += ((f & 2) ? w : 0.0) * x[1];
  s += ((f & 8) ? w : 0.0) * x[P];
  if (D == 3) s += ((f & 32) ? w : 0.0) * x[P * P];
  return s;
}

template <int D, int N>
__global__ void __launch_bounds__(kCoarseThreads, 1) k_coarse_fast(LevelView L, CoarseFast C,
                                                                   const double* __restrict__ phi_b,
                                                                   Rec* rec, int* status,
                                                                   double* diag_out) {
  pdl_begin();
  using G = Geo<D, N>;
  using CG = CoarseGeo<D, N>;
  constexpr int NI = G::NI;
  constexpr int CPT = CG::CPT;
  extern __shared__ double smem[];
  double* Gx = smem;              // padded gather image: x, then p^, then s^
  double* R0 = Gx + CG::PS;       // r0
  double* XX = R0 + NI;           // x
  double* PP = XX + NI;           // p
  double* DG = PP + NI;           // diagonal
  double* DI = DG + NI;           // dinv
  double* RB = DI + NI;           // reduction buffers: 4 x 64
  uint8_t* FL = reinterpret_cast<uint8_t*>(RB + 4 * 64);
  int rb = 0;
  auto buf = [&]() {
    double* b = RB + 64 * rb;
    rb = (rb + 1) & 3;
    return b;
  };
  const int tid = threadIdx.x;
  double r[CPT], v[CPT], s[CPT], t[CPT];
  int pi[CPT];
  bool unk[CPT];
  for (int q = tid; q < CG::PS; q += kCoarseThreads) Gx[q] = 0.0;
  __syncthreads();
  // ---- setup: b, x, dinv (multigrid.hpp:213-217, 445-453)
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int ii = tid + q * kCoarseThreads;
    unk[q] = false;
    r[q] = 0;
    v[q] = 0;
    pi[q] = 0;
    if (ii >= NI) continue;
    const uint8_t f = C.flags[ii];
    FL[ii] = f;
    const double dg = C.diag[ii];
    DG[ii] = dg;
    DI[ii] = (dg != 0) ? 1.0 / dg : 1.0;
    PP[ii] = 0;
    pi[q] = CG::pad(ii);
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    const size_t a = G::addr(0, i, j, k);
    unk[q] = (f & 0x40) != 0;
    const double x0 = unk[q] ? L.phi[a] : 0.0;
    XX[ii] = x0;
    Gx[pi[q]] = x0;
    if (unk[q]) {
      double bu = L.rhs[a] + C.c0[ii];
      for (int z = C.ob_start[ii]; z < C.ob_start[ii + 1]; ++z) bu += C.ob_val[z] * phi_b[C.ob_obj[z]];
      r[q] = bu;  // holds b for now
    }
  }
  __syncthreads();
  double acc = 0;
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int ii = tid + q * kCoarseThreads;
    if (ii >= NI) continue;
    if (unk[q]) {
      r[q] = r[q] - coarse_row<D, N>(C, Gx, FL[ii], DG[ii], pi[q], ii);
      acc += r[q] * r[q];
    }
    R0[ii] = r[q];
  }
  const double norm0 = sqrt(cta_sum1(acc, buf()));
  bool converged = false;
  double rel = 1.0;
  int iters = 0;
  if (norm0 == 0 || norm0 < 1e-300) {
    converged = true;
    rel = 0;
  } else {
    const double target = C.rel_tol * norm0;
    double rho = 1, alpha = 1, omega = 1;
    // rho1 of the first iteration: (r0, r) = (r, r) summed as dot(r0, r)
    acc = 0;
#pragma unroll
    for (int q = 0; q < CPT; ++q)
      if (unk[q]) acc += R0[tid + q * kCoarseThreads] * r[q];
    double rho1 = cta_sum1(acc, buf());
    for (int it = 0; it < C.max_iters; ++it) {
      if (rho1 == 0) break;
      const double beta = it == 0 ? 0.0 : (rho1 / rho) * (alpha / omega);
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int ii = tid + q * kCoarseThreads;
        if (!unk[q]) continue;
        const double pq = it == 0 ? r[q] : r[q] + beta * (PP[ii] - omega * v[q]);
        PP[ii] = pq;
        Gx[pi[q]] = DI[ii] * pq;  // p^ = D^-1 p
      }
      __syncthreads();
      acc = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int ii = tid + q * kCoarseThreads;
        if (!unk[q]) continue;
        v[q] = coarse_row<D, N>(C, Gx, FL[ii], DG[ii], pi[q], ii);
        acc += R0[ii] * v[q];
      }
      const double r0v = cta_sum1(acc, buf());
      if (r0v == 0) break;
      alpha = rho1 / r0v;
      acc = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        if (!unk[q]) continue;
        s[q] = r[q] - alpha * v[q];
        acc += s[q] * s[q];
      }
      const double ns = sqrt(cta_sum1(acc, buf()));
      double ph[CPT];
#pragma unroll
      for (int q = 0; q < CPT; ++q) ph[q] = unk[q] ? Gx[pi[q]] : 0.0;
      if (ns <= target) {
#pragma unroll
        for (int q = 0; q < CPT; ++q)
          if (unk[q]) XX[tid + q * kCoarseThreads] += alpha * ph[q];
        converged = true;
        iters = it + 1;
        rel = ns / norm0;
        break;
      }
      __syncthreads();  // every thread has finished reading p^ from Gx
#pragma unroll
      for (int q = 0; q < CPT; ++q)
        if (unk[q]) Gx[pi[q]] = DI[tid + q * kCoarseThreads] * s[q];  // s^
      __syncthreads();
      double ts = 0, tt = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int ii = tid + q * kCoarseThreads;
        if (!unk[q]) continue;
        t[q] = coarse_row<D, N>(C, Gx, FL[ii], DG[ii], pi[q], ii);
        ts += t[q] * s[q];
        tt += t[q] * t[q];
      }
      cta_sum2(ts, tt, buf());
      if (tt == 0) break;
      omega = ts / tt;
      double rr = 0, r0r = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int ii = tid + q * kCoarseThreads;
        if (!unk[q]) continue;
        XX[ii] += alpha * ph[q] + omega * Gx[pi[q]];
        r[q] = s[q] - omega * t[q];
        rr += r[q] * r[q];
        r0r += R0[ii] * r[q];
      }
      cta_sum2(rr, r0r, buf());
      rho = rho1;
      iters = it + 1;
      rel = sqrt(rr) / norm0;
      if (rel <= C.rel_tol) {
        converged = true;
        break;
      }
      if (omega == 0) break;
      rho1 = r0r;
      __syncthreads();  // Gx is overwritten at the top of the next iteration
    }
  }
  __syncthreads();
  const bool wb = converged || C.fallback_ok;
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int ii = tid + q * kCoarseThreads;
    if (!unk[q] || !wb) continue;
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    L.phi[G::addr(0, i, j, k)] = XX[ii];
  }
  __syncthreads();
  if (tid == 0) {
    status[0] = wb ? 0 : 3;
    diag_out[0] = rel;
    diag_out[1] = (double)iters;
  }
  double* sm = RB;
  if (!converged && C.fallback_ok) {
    double r0m = -1;
    bool ok = false;
    for (int it = 0; it < 20000 && !ok; ++it) {
      for (int par = 0; par < 2; ++par) {
        for (int e = tid; e < G::H; e += blockDim.x) gs_cell<D, N>(L, L, phi_b, 0, par, e);
        __syncthreads();
      }
      if (it % 50 == 0) {
        double m = 0;
        for (int ce = tid; ce < NI; ce += blockDim.x) {
          bool ins;
          const double rr = resid_cell<D, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
          if (!ins) m = fmax(m, fabs(rr));
        }
        m = block_max(m, sm);
        if (r0m < 0) r0m = m;
        if (m <= C.rel_tol * r0m || m < 1e-300) ok = true;
      }
    }
    if (!ok && tid == 0) status[0] = 4;
    __syncthreads();
  }
  // pins (multigrid.hpp:469)
  if (L.srow[0] >= 0)
    for (int ce = tid; ce < NI; ce += blockDim.x) {
      const int rr = L.row_of[(size_t)L.srow[0] * NI + ce];
      if (rr >= 0 && L.r_mask[rr] == 1) L.phi[ce] = phi_b[L.r_pin[rr]];
    }
  __syncthreads();
  // record_leaf_residual(1) (multigrid.hpp:471)
  double mx = 0, ss = 0, cnt = 0;
  if (L.leaf[0]) {
    for (int ce = tid; ce < NI; ce += blockDim.x) {
      bool ins;
      const double rr = resid_cell<D, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
      if (ins) continue;
      mx = fmax(mx, fabs(rr));
      ss += rr * rr;
      cnt += 1;
    }
  }
  mx = block_max(mx, sm);
  ss = block_sum(ss, sm);
  cnt = block_sum(cnt, sm);
  if (tid == 0) {
    rec[1].max = mx;
    rec[1].sumsq = ss;
    rec[1].count = (long long)cnt;
  }
}

template <int D, int N>
constexpr size_t coarse_fast_smem() {
  return (size_t)CoarseGeo<D, N>::PS * 8 + (size_t)5 * Geo<D, N>::NI * 8 + 4 * 64 * 8 +
         Geo<D, N>::NI;
}

}  // namespace pmgdev
