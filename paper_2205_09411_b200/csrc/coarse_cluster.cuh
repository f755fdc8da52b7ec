// coarse_cluster.cuh -- K6 on a thread-block cluster (3D levels with N <= 16).
//
// Same algorithm and row arithmetic as coarse.cuh (a replica of
// detail::bicgstab, multigrid.hpp:208-280), distributed over a cluster of
// N/PPC CTAs: CTA r owns planes r*PPC .. r*PPC+PPC-1 of the root block, one
// cell per thread, every per-cell vector lives in registers.  The vectors the SpMV gathers (x, p^,
// s^) are kept as zero-padded planes in each CTA's shared memory; the z-1 and
// z+1 values are read from the neighbouring CTAs through distributed shared
// memory.  Each dot product is reduced inside the CTA by one warp, its partial
// pushed to every CTA of the cluster with st.async onto a per-stage mbarrier,
// and every CTA sums the N partials in rank order -- deterministic, and
// identical in every CTA, so all CTAs take the same branch at every
// breakdown/stopping test.  No cluster barrier inside the iteration loop.
#pragma once
#include <cooperative_groups.h>

#include "coarse.cuh"
#include "stream.cuh"  // mbarrier helpers

namespace pmgdev {

namespace cg = cooperative_groups;

template <int N, int PPC = 1>
struct CC {
  static constexpr int P = N + 2;           // padded plane extent
  static constexpr int PP = P * P;
  static constexpr int NC = N / PPC;        // CTAs in the cluster (PPC planes each)
  static constexpr int THR = PPC * N * N;   // one thread per cell of the CTA's planes
  static constexpr int NW = (THR + 31) / 32;
  static constexpr int NSTAGE = 6;          // reduction stages (0 setup; 1, 2, 4 per iteration)
};

template <int N>
__device__ __forceinline__ double cc_row(const CoarseFast& C, const double* __restrict__ G,
                                         const double* __restrict__ Gm,
                                         const double* __restrict__ Gp, uint8_t f, double dg,
                                         int pi, const double* sc) {
  // sorted column order: z-, y-, x-, diag, x+, y+, z+ (coarse.cuh); absent
  // terms are exact zeros (0*x with x finite) and change nothing.  `sc`: the
  // special row's six off-diagonals, held in registers by the caller.
  constexpr int P = N + 2;
  double s = 0;
  if (f & 0x80) {
    s += sc[4] * Gm[pi];
    s += sc[2] * G[pi - P];
    s += sc[0] * G[pi - 1];
    s += dg * G[pi];
    s += sc[1] * G[pi + 1];
    s += sc[3] * G[pi + P];
    s += sc[5] * Gp[pi];
    return s;
  }
  const double w = C.w;
  s += ((f & 16) ? w : 0.0) * Gm[pi];
  s += ((f & 4) ? w : 0.0) * G[pi - P];
  s += ((f & 1) ? w : 0.0) * G[pi - 1];
  s += dg * G[pi];
  s += ((f & 2) ? w : 0.0) * G[pi + 1];
  s += ((f & 8) ? w : 0.0) * G[pi + P];
  s += ((f & 32) ? w : 0.0) * Gp[pi];
  return s;
}

struct D3 {
  double x, y, z;
};

template <int N, int PPC>
__global__ void __launch_bounds__(CC<N, PPC>::THR, 1) k_coarse_cluster(LevelView L, CoarseFast C,
                                                                    const double* __restrict__ phi_b,
                                                                    Rec* rec, int* status,
                                                                    double* diag_out) {
  // programmatic dependent launch: the static per-cell operator data below is
  // loaded before waiting for the previous kernel (the FAS of level 1); PHI,
  // the right-hand side and phi_b are read only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  using G = Geo<3, N>;
  using K = CC<N, PPC>;
  cg::cluster_group cl = cg::this_cluster();
  // own planes of the two gathered vectors: [0] x / p^, [1] s^
  __shared__ double Gx[2][PPC][K::PP];
  // partials of every warp of every CTA, per reduction stage
  __shared__ double part[K::NSTAGE][K::NC * K::NW][2];
  __shared__ double part3[K::NC * K::NW];  // third value of the (s, s) / (t, s) / (t, t) stage
  const int zr = (int)cl.block_rank();
  const int t = threadIdx.x;
  const int lane = t & 31, wid = t >> 5;
  const int x = t % N, y = (t / N) % N, lp = t / (N * N);
  const int z = zr * PPC + lp;  // plane of this thread's cell
  const int ii = x + N * (y + N * z);
  const int pi = (x + 1) + (y + 1) * K::P;
  // neighbour planes across the CTA's edge planes are pushed here by the
  // neighbouring CTAs (st.async, completing on gbar[k]); out-of-block planes
  // alias our own (coefficient 0)
  __shared__ double gh[2][2][K::PP];
  __shared__ __align__(8) uint64_t gbar[2];
  double* Gs0 = Gx[0][lp];
  double* Gs1 = Gx[1][lp];
  const double* Gm0 = lp > 0 ? Gx[0][lp - 1] : (zr > 0 ? gh[0][0] : Gs0);
  const double* Gp0 = lp < PPC - 1 ? Gx[0][lp + 1] : (zr < K::NC - 1 ? gh[0][1] : Gs0);
  const double* Gm1 = lp > 0 ? Gx[1][lp - 1] : (zr > 0 ? gh[1][0] : Gs1);
  const double* Gp1 = lp < PPC - 1 ? Gx[1][lp + 1] : (zr < K::NC - 1 ? gh[1][1] : Gs1);
  for (int q = t; q < 4 * K::PP; q += K::THR) (&gh[0][0][0])[q] = 0.0;
  for (int q = t; q < 2 * PPC * K::PP; q += K::THR) (&Gx[0][0][0])[q] = 0.0;
  __syncthreads();
  // ---- per-cell data (multigrid.hpp:213-217, 445-453)
  const uint8_t f = C.flags[ii];
  const double dg = C.diag[ii];
  const double dinv = (dg != 0) ? 1.0 / dg : 1.0;
  const bool unk = (f & 0x40) != 0;
  double sc[6] = {0, 0, 0, 0, 0, 0};  // special-row off-diagonals, loaded once
  if (f & 0x80)
    for (int d = 0; d < 6; ++d) sc[d] = C.spec_c[(size_t)C.spec[ii] * 6 + d];
  const double c0v = C.c0[ii];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const size_t a = G::addr(0, x, y, z);
  double xv = unk ? L.phi[a] : 0.0;
  double bv = 0;
  if (unk) {
    bv = L.rhs[a] + c0v;
    for (int q = C.ob_start[ii]; q < C.ob_start[ii + 1]; ++q) bv += C.ob_val[q] * phi_b[C.ob_obj[q]];
  }
  // Cluster-wide deterministic sum of (a, b) plus the scalar recurrence that
  // consumes it, with no CTA or cluster barrier: every warp reduces its pair
  // (xor butterfly), lane r pushes it into part[stage][rank * NW + warp] of
  // CTA r with st.async, completing on that CTA's per-stage mbarrier; every
  // warp of every CTA waits for the NC * NW partials, sums them in one fixed
  // order (strided per lane, then the butterfly: every lane holds the same
  // bits) and evaluates the stage's scalars itself.  Identical inputs and
  // order everywhere, so every warp of every CTA takes the same branch.
  // Buffer reuse: a CTA pushes stage k of the next iteration only after every
  // warp of every CTA has pushed the later stages of this one, i.e. after
  // every warp has read stage k.
  __shared__ __align__(8) uint64_t sbar[K::NSTAGE];
  constexpr int NP = K::NC * K::NW;
  static_assert(K::NC <= 32, "one lane per destination CTA");
  unsigned uses = 0;  // bit k: parity of stage k's next phase
  auto csum3 = [&](int stage, double va, double vb, double vc, bool three, auto&& fn) -> D3 {
    va = warp_sum(va);
    vb = warp_sum(vb);
    if (three) vc = warp_sum(vc);
    if (t == 0) mbar_arrive_expect_tx(&sbar[stage], NP * (three ? 24u : 16u));
    if (lane < K::NC) {  // lane r pushes this warp's partial to rank r
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                   : "=r"(ra)
                   : "r"(smem_u32(&part[stage][zr * K::NW + wid][0])), "r"(lane));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&sbar[stage])), "r"(lane));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                   "d"(va), "d"(vb), "r"(rb)
                   : "memory");
      if (three) {
        uint32_t rc;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rc) : "r"(smem_u32(&part3[zr * K::NW + wid])), "r"(lane));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(rc), "d"(vc),
                     "r"(rb)
                     : "memory");
      }
    }
    mbar_wait(&sbar[stage], (uses >> stage) & 1u);
    uses ^= 1u << stage;
    double ta = 0, tb = 0, tc = 0;
#pragma unroll
    for (int k = lane; k < NP; k += 32) {
      ta += part[stage][k][0];
      tb += part[stage][k][1];
      if (three) tc += part3[k];
    }
    ta = warp_sum(ta);
    tb = warp_sum(tb);
    if (three) tc = warp_sum(tc);
    return fn(ta, tb, tc);
  };
  auto csum = [&](int stage, double va, double vb, auto&& fn) -> D3 {
    return csum3(stage, va, vb, 0.0, false, [&](double a2, double b2, double) { return fn(a2, b2); });
  };
  static_assert(K::THR % 32 == 0, "whole warps");
  if (t == 0) {
    for (int k = 0; k < K::NSTAGE; ++k) mbar_init(&sbar[k], 1);
    mbar_init(&gbar[0], 1);
    mbar_init(&gbar[1], 1);
    fence_mbar_init();
  }
  cl.sync();  // every CTA's barriers initialised, ghost planes zeroed
  // publish a vector's plane values: own planes in shared memory, edge planes
  // pushed into the neighbouring CTAs' ghost planes (k: which vector)
  const uint32_t gbytes = (uint32_t)(((zr > 0) + (zr < K::NC - 1)) * N * N * 8);
  unsigned guses = 0;
  auto push = [&](int k, double val) {
    (k ? Gs1 : Gs0)[pi] = val;
    if (t == 0) mbar_arrive_expect_tx(&gbar[k], gbytes);
    if (lp == 0 && zr > 0) {
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&gh[k][1][pi])), "r"(zr - 1));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&gbar[k])), "r"(zr - 1));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(val),
                   "r"(rb)
                   : "memory");
    }
    if (lp == PPC - 1 && zr < K::NC - 1) {
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&gh[k][0][pi])), "r"(zr + 1));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&gbar[k])), "r"(zr + 1));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(val),
                   "r"(rb)
                   : "memory");
    }
  };
  // wait for vector k's ghost planes, then a CTA barrier for the own planes
  auto land = [&](int k) {
    if (wid == 0) mbar_wait(&gbar[k], (guses >> k) & 1u);
    guses ^= 1u << k;
    __syncthreads();
  };
  push(0, xv);  // x planes
  land(0);
  double r = 0;
  if (unk) r = bv - cc_row<N>(C, Gs0, Gm0, Gp0, f, dg, pi, sc);
  const double r0 = r;
  // setup: n2 = (r, r), rho1 = (r0, r); norm0 = sqrt(n2)
  D3 o = csum(0, unk ? r * r : 0.0, unk ? r0 * r : 0.0, [](double a2, double b2) { return D3{a2, b2, sqrt(a2)}; });
  double rho1 = o.y;
  const double norm0 = o.z;
  bool converged = false;
  double rel = 1.0;
  int iters = 0;
  double p = 0, v = 0, s = 0, tv = 0;
  if (norm0 == 0 || norm0 < 1e-300) {
    converged = true;
    rel = 0;
  } else {
    const double target = C.rel_tol * norm0;
    const double rtol = C.rel_tol;
    double alpha = 1, omega = 1, beta = 0;
    for (int it = 0; it < C.max_iters; ++it) {
      if (rho1 == 0) break;
      if (unk) p = it == 0 ? r : r + beta * (p - omega * v);
      const double ph = unk ? dinv * p : 0.0;
      // p^ planes: every warp has passed the last reduction, so nobody in
      // this CTA or the neighbours still reads the previous p^
      push(0, ph);
      land(0);
      v = unk ? cc_row<N>(C, Gs0, Gm0, Gp0, f, dg, pi, sc) : 0.0;
      // (r0, v); alpha = rho1 / (r0, v)
      o = csum(1, unk ? r0 * v : 0.0, 0.0,
               [rho1](double a2, double) { return D3{a2, a2 == 0 ? 0.0 : rho1 / a2, 0.0}; });
      if (o.x == 0) break;
      alpha = o.y;
      s = unk ? r - alpha * v : 0.0;
      const double sh = unk ? dinv * s : 0.0;  // s^
      // s^ planes (s^ of the previous iteration was consumed before the
      // (r0, v) reduction everyone has passed); t = A s^ is formed before
      // ||s|| is known, so (s, s), (t, s) and (t, t) share one reduction --
      // on the early exit (||s|| <= tol ||r0||) t is simply not used
      push(1, sh);
      land(1);
      tv = unk ? cc_row<N>(C, Gs1, Gm1, Gp1, f, dg, pi, sc) : 0.0;
      o = csum3(2, s * s, tv * s, tv * tv, true,
                [](double a2, double b2, double c2) { return D3{sqrt(a2), c2, c2 == 0 ? 0.0 : b2 / c2}; });
      const double ns = o.x;
      if (ns <= target) {
        if (unk) xv += alpha * ph;
        converged = true;
        iters = it + 1;
        rel = ns / norm0;
        break;
      }
      if (o.y == 0) break;  // (t, t) = 0
      omega = o.z;  // (t, s) / (t, t)
      if (unk) {
        xv += alpha * ph + omega * sh;
        r = s - omega * tv;
      }
      // (r, r), (r0, r); rel = ||r|| / ||r0||; the next beta
      o = csum(4, unk ? r * r : 0.0, unk ? r0 * r : 0.0, [norm0, rho1, alpha, omega](double a2, double b2) {
        return D3{sqrt(a2) / norm0, b2, (b2 / rho1) * (alpha / omega)};
      });
      iters = it + 1;
      rel = o.x;
      if (rel <= rtol) {
        converged = true;
        break;
      }
      if (omega == 0) break;
      rho1 = o.y;
      beta = o.z;  // (rho1 / rho) * (alpha / omega), multigrid.hpp:236
    }
  }
  const bool wb = converged || C.fallback_ok;
  if (unk && wb) L.phi[a] = xv;
  // apply_pins(1) (multigrid.hpp:469): inside cells are not unknowns, so the
  // write-back never touched them; re-pinning is spread over the cluster
  for (int q = zr * K::THR + t; q < C.n_pins; q += K::NC * K::THR) L.phi[C.pins[q].x] = phi_b[C.pins[q].y];
  cl.sync();  // write-back complete in every plane before the tail
  if (zr != 0) return;
  // ---- tail on rank 0 (whole root block): fallback, pins, level-1 record
  __shared__ double sm[72];
  if (t == 0) {
    status[0] = wb ? 0 : 3;
    diag_out[0] = rel;
    diag_out[1] = (double)iters;
  }
  if (!converged && C.fallback_ok) {
    double r0m = -1;
    bool ok = false;
    for (int it = 0; it < 20000 && !ok; ++it) {
      for (int par = 0; par < 2; ++par) {
        __threadfence_block();
        for (int e = t; e < G::H; e += blockDim.x) gs_cell<3, N>(L, L, phi_b, 0, par, e);
        __syncthreads();
      }
      if (it % 50 == 0) {
        double m = 0;
        for (int ce = t; ce < G::NI; ce += blockDim.x) {
          bool ins;
          const double rr = resid_cell<3, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
          if (!ins) m = fmax(m, fabs(rr));
        }
        m = block_max(m, sm);
        if (r0m < 0) r0m = m;
        if (m <= C.rel_tol * r0m || m < 1e-300) ok = true;
      }
    }
    if (!ok && t == 0) status[0] = 4;
    __syncthreads();
  }
  if (!converged && C.fallback_ok && L.srow[0] >= 0) {  // the fallback sweeps skip inside cells; re-pin anyway
    for (int q = t; q < C.n_pins; q += blockDim.x) L.phi[C.pins[q].x] = phi_b[C.pins[q].y];
    __syncthreads();
  }
  if (!L.leaf[0]) return;  // level 1 has no leaves: its record stays zero
  double mx = 0, ss = 0, cnt = 0;
  {
    for (int ce = t; ce < G::NI; ce += blockDim.x) {
      bool ins;
      const double rr = resid_cell<3, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
      if (ins) continue;
      mx = fmax(mx, fabs(rr));
      ss += rr * rr;
      cnt += 1;
    }
  }
  mx = block_max(mx, sm);
  ss = block_sum(ss, sm);
  cnt = block_sum(cnt, sm);
  if (t == 0) {
    rec[1].max = mx;
    rec[1].sumsq = ss;
    rec[1].count = (long long)cnt;
  }
}

}  // namespace pmgdev
