// ops_impl.cuh -- kernel launchers (OpsImpl<Dim,N>); instantiated once per
// (Dim, N) in ops_<D>_<N>.cu so the variants compile in parallel.
#pragma once
#include <algorithm>
#include <type_traits>
#include "ctx.h"
#include "stencil_build.cuh"
#include "tile_kernels.cuh"
#include "coarse.cuh"
#include "coarse_cluster.cuh"
#include "stream.cuh"
#include "brick.cuh"
#include "coop.cuh"
#include "small.cuh"
#include "fields.cuh"

namespace pmghost {

using namespace pmgdev;

// streaming GS pipeline depth and residency (stream.cuh)
constexpr int kStreamStages = 2;
constexpr int kStreamCtasPerSm = 2;
constexpr int kFoldThreads = 512;  // k_record_fold: ~1500 partials at most on the large levels

static inline unsigned grid_for(long long n, int threads = kThreads) {
  return (unsigned)((n + threads - 1) / threads);
}

template <int D, int N>
struct OpsImpl final : Ops {
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  // shared-memory tiles fit the static 48 KB limit (3D N=32 keeps the per-cell kernels)
  static constexpr bool TILE = 2 * TT::SIZE * 8 + 1024 <= 48 * 1024;
  static constexpr bool FASTC = G::NI <= 4096;
  const LevelView& V(Ctx& c, int l) { return c.lev[(size_t)l]->view; }
  const LevelView& Vc(Ctx& c, int l) { return c.lev[(size_t)(l > 1 ? l - 1 : l)]->view; }
  // level l's view with the cfc table (coarse parts of its coarse-fine ghosts)
  // attached, rebuilt first if level l-1 changed since
  LevelView Vt(Ctx& c, int l) {
    LevelDev& d = *c.lev[(size_t)l];
    LevelView v = d.view;
    if (d.n_cf > 0) {
      ensure_cfc(c, l);
      v.cfc = d.cfc.p;
    }
    return v;
  }
  bool cf_table() const override { return TILE; }
  void cfc_build(Ctx& c, int l) override { cfc_build_on(c, l, c.stream); }
  void cfc_build_on(Ctx& c, int l, cudaStream_t s) {
    const LevelDev& d = *c.lev[(size_t)l];
    pdl_launch_on(k_cfc_build<D, N>, grid_for((long long)d.n_cf * G::NT, 256), 256, 0, s, V(c, l), Vc(c, l),
               (const int4*)d.cf_desc.p, d.n_cf, d.cfc.p);
    check();
  }
  // Level l's stale cfc table rebuilt on the forked stream, beside a kernel
  // that neither writes level l-1 nor reads the table (the caller forks
  // before and joins after): off the main stream's chain of launches.
  bool cfc_stale(Ctx& c, int l) {
    if (l < 2 || l > c.mesh.L) return false;
    const LevelDev& d = *c.lev[(size_t)l];
    return d.n_cf > 0 && d.cfc_dirty;
  }
  void cfc_build_side(Ctx& c, int l) {
    cfc_build_on(c, l, c.side);
    c.lev[(size_t)l]->cfc_dirty = false;
  }

  void check() { PMG_CUDA(cudaGetLastError()); }
  // k_resid_stream with coarse-fine support (MODE 0 restriction, 1 record) over `plan`
  template <int ST, int MINB, int MODE, int TTH>
  void launch_qs(Ctx& c, int grid, const LevelView& Lf, const LevelView& Lp, const int32_t* plan, int n) {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      using Q = QStream3<N, TTH>;
      constexpr size_t smem = (size_t)ST * (Q::STAGE + 12 * Q::FH) * sizeof(double);
      set_smem_attr(c, (const void*)k_resid_stream<N, ST, MINB, MODE, TTH, true>, smem);
      // programmatic dependent launch for the restriction (96.7 -> 85.5 us on cfg3's finest level;
      // the record measured slower with it there)
      if (MODE == 0)
        pdl_launch_on(k_resid_stream<N, ST, MINB, MODE, TTH, true>, grid, Q::THR, smem, c.stream, Lf, Lp, c.phi_b.p,
                      (const int4*)plan, n, (Rec*)nullptr, (Rec*)nullptr, (unsigned int*)nullptr);
      else
        pdl_launch(k_resid_stream<N, ST, MINB, MODE, TTH, true>, grid, Q::THR, smem, c.stream, Lf, Lp, c.phi_b.p,
                   (const int4*)plan, n, MODE == 1 ? c.partial.p : (Rec*)nullptr, MODE == 1 ? c.rec.p : (Rec*)nullptr,
                   (unsigned int*)nullptr);
    }
  }

  void gs(Ctx& c, int l, int parity) override {
    const LevelView& L = V(c, l);
    phi_written(c, l);
    if (L.nb <= kSmallLevel) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (d.has_tab)
        pdl_launch_on(k_gs_tab<D, N>, grid_for((long long)L.nb * G::H), 256, 0, c.stream, L, c.phi_b.p,
                      (const int4*)d.tab.p, (const double*)d.tgbc.p, parity);
      else
        pdl_launch(k_gs<D, N>, grid_for((long long)L.nb * G::H), kThreads, 0, c.stream, L, Vc(c, l), c.phi_b.p,
                   parity);
      check();
      return;
    }
    if constexpr (TILE) {
      const LevelDev& d = *c.lev[(size_t)l];
      // The streaming kernel (3D, N = 8/16) covers every lean block, cut rows
      // included; otherwise k_gs_lean does the uniform rows and k_gs_fix the
      // cut rows.  The general blocks (coarse-fine faces) run on a forked
      // branch: all kernels write disjoint cells of colour `parity` and read
      // only the other colour (plus, in k_gs_fix, the cut cell's own value).
      bool stream = false;
      if constexpr (D == 3 && (N == 8 || N == 16))
        stream = d.n_gs > 0;
      const int nfix = stream ? 0 : d.n_fix[parity];
      const bool lean_work = stream || d.n_fast > 0;
      const int ncut = stream ? d.n_cut[parity] : 0;
      // streaming: blocks with coarse-fine faces are in the plan too (gs_cf),
      // except the few with a cut row near such a face (gs_slow)
      const int n_tile = stream ? d.n_gs_slow : d.n_slow;
      const int32_t* tile_list = stream ? d.gs_slow.p : d.slow_list.p;
      const int ncutcf = stream ? d.n_cutcf[parity] : 0;
      const bool fork = lean_work && (n_tile > 0 || nfix > 0 || ncut > 0 || ncutcf > 0);
      const LevelView Lt = d.n_cf > 0 ? Vt(c, l) : L;  // before the fork: a table rebuild runs on c.stream
      if (fork) {
        PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
      }
      cudaStream_t s2 = fork ? c.side : c.stream;
      if (n_tile > 0)
        pdl_launch(k_gs_tile<D, N>, n_tile, TT::THREADS, 0, s2, Lt, Vc(c, l), c.phi_b.p, parity, tile_list);
      if (nfix > 0)
        pdl_launch(k_gs_fix<D, N>, grid_for(nfix, 128), 128, 0, s2, L, Vc(c, l), c.phi_b.p, parity,
                                                           (const int2*)d.fix_list[parity].p, nfix);
      if (ncut > 0 && ncutcf > 0)  // both cut-row tables in one launch
        pdl_launch(k_gs_cut2<D>, grid_for(ncut + ncutcf, 128), 128, 0, s2, L, (const int32_t*)d.cut_ent[parity].p,
                   (const double*)d.cut_gbc[parity].p, (const double*)d.cut_coef[parity].p, ncut,
                   (const int32_t*)d.cutcf_ent[parity].p, (const double*)d.cutcf_gbc[parity].p,
                   (const double*)d.cutcf_coef[parity].p, ncutcf);
      else if (ncut > 0)  // cut rows: disjoint from the streaming kernel's cells and inputs
        pdl_launch(k_gs_cut<D>, grid_for(ncut, 128), 128, 0, s2, L, (const int32_t*)d.cut_ent[parity].p,
                   (const double*)d.cut_gbc[parity].p, (const double*)d.cut_coef[parity].p, ncut);
      else if (ncutcf > 0)
        pdl_launch(k_gs_cut<D>, grid_for(ncutcf, 128), 128, 0, s2, L, (const int32_t*)d.cutcf_ent[parity].p,
                   (const double*)d.cutcf_gbc[parity].p, (const double*)d.cutcf_coef[parity].p, ncutcf);
      if (stream) {
        if constexpr (D == 3 && (N == 8 || N == 16)) {
          constexpr int T256 = N == 16 ? 256 : 0;
          if (d.gs_cf) {
            // ten 128-thread CTAs per SM (20.6 us per finest cfg3 half-sweep; 21.3 with eight,
            // 21.9 with three stages, 25.9 with 256-thread CTAs, 27.0 with twelve 64-thread CTAs)
            if constexpr (N == 8) launch_gs_stream<2, 10, 128, true>(c, Lt, d, parity);
            else launch_gs_stream<kStreamStages, kStreamCtasPerSm, 0, true>(c, Lt, d, parity);
          }
          else if (T256 && d.n_gs <= c.sms * 4)  // one block per CTA, all resident at once
            launch_gs_stream<1, 4, T256>(c, L, d, parity);
          else if (N == 8)  // 512-cell blocks: 128-thread CTAs, eight per SM (40.0 vs 45.1 us per
            launch_gs_stream<2, 8, 128>(c, L, d, parity);  // half-sweep on cfg3's finest level with <2, 2, 256>)
          else if (d.n_gs <= 1024) launch_gs_stream<2, 3, T256>(c, L, d, parity);  // 7.7 vs 8.0 us at 512 blocks
          else launch_gs_stream<kStreamStages, kStreamCtasPerSm, 0>(c, L, d, parity);
        }

      } else if (d.n_fast > 0) {
        pdl_launch(k_gs_lean<D, N>, d.n_fast, Lean<D, N>::THR, 0, c.stream, L, parity, d.fast_list.p);
      }
      if (fork) {
        PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
        PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
      }
    }
    else
      pdl_launch(k_gs<D, N>, grid_for((long long)L.nb * G::H), kThreads, 0, c.stream, L, Vc(c, l),
                                                                             c.phi_b.p, parity);
    check();
  }
  // smooth(l, steps) in one cooperative launch (coop.cuh): 3D N = 8 / 16
  // levels whose blocks are all lean, one CTA per plan block, all co-resident
  bool smooth(Ctx& c, int l, int steps) override {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      LevelDev& d = *c.lev[(size_t)l];
      if (steps <= 0 || !kCoopEnabled) return false;
      if (d.coop < 0) {
        d.coop = 0;
        if (!d.has_cf && d.n_slow == 0 && d.n_gs > 0 && d.n_gs <= kCoopMaxBlocks) {
          constexpr size_t smem = (size_t)Coop3<N>::SMEM * sizeof(double);
          set_smem_attr(c, (const void*)k_gs_coop<N>, smem);
          int per_sm = 0;
          PMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs_coop<N>, kCoopThreads, smem));
          d.coop = (long long)per_sm * c.sms >= d.n_gs ? 1 : 0;
        }
      }
      if (!d.coop) return false;
      const LevelView& L = V(c, l);
      CutTabs cut;
      for (int cc = 0; cc < 2; ++cc) {
        cut.ent[cc] = (const int32_t*)d.cut_ent[cc].p;
        cut.gbc[cc] = (const double*)d.cut_gbc[cc].p;
        cut.coef[cc] = (const double*)d.cut_coef[cc].p;
        cut.off[cc] = (const int32_t*)d.cut_off[cc].p;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)d.n_gs);
      cfg.blockDim = dim3(kCoopThreads);
      cfg.dynamicSmemBytes = (size_t)Coop3<N>::SMEM * sizeof(double);
      cfg.stream = c.stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PMG_CUDA(cudaLaunchKernelEx(&cfg, k_gs_coop<N>, L, (const int4*)d.gs_plan.p, d.n_gs, 2 * steps, cut,
                                  c.gbar.p));
      phi_written(c, l);
      return true;
    }
    return false;
  }
  template <int ST, int MINB, int TH, bool CF = false>
  void launch_gs_stream(Ctx& c, const LevelView& L, const LevelDev& d, int parity) {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      using S = Stream3<N, TH>;
      constexpr size_t smem = (size_t)ST * (S::STAGE + (CF ? 6 * S::FH : 0)) * sizeof(double);
      set_smem_attr(c, (const void*)k_gs_stream<N, ST, MINB, TH, CF>, smem);
      const int grid = std::min(d.n_gs, c.sms * MINB);
      // PDL: the prologue overlaps the previous kernel's drain; parity 1 walks
      // the plan backwards (starts on the blocks the red half-sweep wrote last)
      pdl_launch_on(k_gs_stream<N, ST, MINB, TH, CF>, grid, S::THR, smem, c.stream, L, parity, c.phi_b.p,
                    (const int4*)d.gs_plan.p, d.n_gs, parity);
    }
  }
  // residual-streaming kernels: k_restrict_stream (one thread per parent) for
  // the restriction, k_resid_stream (column mapping) for the record and FAS
  template <int MODE, int ST, int MINB, int TT>
  void launch_resid_stream(Ctx& c, const LevelView& Lf, const LevelView& Lp, const LevelDev& d, Rec* partial,
                           Rec* rec) {
    if constexpr (D == 3 && N == 16) {
      using Q = QStream3<N, TT>;
      constexpr size_t smem = (size_t)ST * Q::STAGE * sizeof(double);
      set_smem_attr(c, (const void*)k_resid_stream<N, ST, MINB, MODE, TT>, smem);
      const int grid = std::min(d.n_rs, c.sms * MINB);
      pdl_launch(k_resid_stream<N, ST, MINB, MODE, TT>, grid, Q::THR, smem, c.stream, Lf, Lp, c.phi_b.p,
                 (const int4*)d.rs_plan.p, d.n_rs, partial, rec, (unsigned int*)nullptr);
    }
  }
  template <int MODE>
  void launch_rstream(Ctx& c, const LevelView& Lf, const LevelView& Lp, const LevelDev& d, Rec* partial, Rec* rec) {
    if constexpr (D == 3 && N == 16) {
      if (MODE == 1) {  // record: the 16-byte-access brick kernel (68 vs 85 us for the column kernel at 256^3)
        constexpr int ST = 2;
        constexpr size_t smem = (size_t)ST * QStream3<N, 512>::STAGE * sizeof(double);
        set_smem_attr(c, (const void*)k_record_brick<N, ST>, smem);
        pdl_launch(k_record_brick<N, ST>, rstream_grid(c, Lf, d), kBrickThreads, smem, c.stream, Lf,
                   (const int4*)d.rs_plan.p, d.n_rs, partial);
        return;
      }
      // restriction: the one-thread-per-parent kernel (85 us at 256^3 vs 93 us
      // for the column kernel); record / FAS: the column kernel
      if (MODE == 0) {
        constexpr int ST = 2, MINB = 1;
        constexpr size_t smem = (size_t)ST * RStream3<N>::STAGE * sizeof(double);
        set_smem_attr(c, (const void*)k_restrict_stream<N, ST, MINB, MODE>, smem);
        const int grid = std::min(d.n_rs, c.sms * MINB);
        pdl_launch_on(k_restrict_stream<N, ST, MINB, MODE>, grid, RStream3<N>::THR, smem, c.stream, Lf, Lp,
                      c.phi_b.p, (const int4*)d.rs_plan.p, d.n_rs, partial, rec, (unsigned int*)nullptr);
      } else {
        launch_resid_stream<MODE, 3, 1, 512>(c, Lf, Lp, d, partial, rec);
      }
    }
  }
  // number of CTAs launch_rstream uses (record partials): k_record_brick runs two per SM
  int rstream_grid(Ctx& c, const LevelView& Lf, const LevelDev& d) { return std::min(d.n_rs, c.sms * 2); }
  void residual(Ctx& c, int l) override {
    const LevelView& L = V(c, l);
    pdl_launch(k_residual<D, N>, grid_for((long long)L.nb * G::NI), kThreads, 0, c.stream, L, Vc(c, l),
                                                                                  c.phi_b.p);
    check();
  }
  void restrict_(Ctx& c, int l, int mode) override {
    restrict_impl(c, l, mode);
    phi_written(c, l - 1);  // after the launch: level l's own table (read above) is stale from here on
  }
  void restrict_impl(Ctx& c, int l, int mode) {
    const LevelView& Lf = V(c, l);
    const unsigned g = grid_for((long long)Lf.nb * G::NI);  // k_restrict: one thread per child cell
    // 3D N=16 levels of more than 8 blocks restrict with the streaming kernel
    // (one block per CTA there)
    const bool stream_small = D == 3 && N == 16 && Lf.nb > 8 && mode == RM_FUSED;
    if (Lf.nb <= kSmallLevel && !stream_small) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (d.has_tab) {
        const LevelView& Lp = V(c, l - 1);
        if (mode == RM_RES)
          pdl_launch_on(k_restrict_tab<D, N, RM_RES>, g, 256, 0, c.stream, Lf, Lp, c.phi_b.p, (const int4*)d.tab.p,
                     (const double*)d.tgbc.p);
        else if (mode == RM_RHS)
          pdl_launch_on(k_restrict_tab<D, N, RM_RHS>, g, 256, 0, c.stream, Lf, Lp, c.phi_b.p, (const int4*)d.tab.p,
                     (const double*)d.tgbc.p);
        else
          pdl_launch_on(k_restrict_tab<D, N, RM_FUSED>, g, 256, 0, c.stream, Lf, Lp, c.phi_b.p,
                     (const int4*)d.tab.p, (const double*)d.tgbc.p);
        check();
        return;
      }
      if (mode == RM_RES)
        pdl_launch(k_restrict<D, N, RM_RES>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p);
      else if (mode == RM_RHS)
        pdl_launch(k_restrict<D, N, RM_RHS>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p);
      else
        pdl_launch(k_restrict<D, N, RM_FUSED>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p);
      check();
      return;
    }
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (mode == RM_FUSED && (N == 8 || d.has_cf) && d.n_rr > 0) {
        // N = 8, or coarse-fine faces: the column kernel (k_resid_stream, MODE 0)
        // over rr_plan, coarse-fine ghosts from the staged cfc pages; parents
        // with a cut child by k_restrict_fix, blocks with a cut row near a
        // coarse-fine face by k_restrict_tile (both only read level l and
        // write other parent cells), then apply_pins(l-1)
        constexpr int MINB = N == 8 ? 8 : 1;
        const int grid = std::min(d.n_rr, c.sms * MINB);
        const LevelView Lt = Vt(c, l);
        // level l-1's own table (read next by its FAS pass) depends on level l-2 only
        const bool pre = cfc_stale(c, l - 1);
        const bool fork = d.n_rfix > 0 || d.n_rr_slow > 0 || pre;
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
          PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        }
        if (pre) cfc_build_side(c, l - 1);
        if (d.n_rr_slow > 0)
          pdl_launch(k_restrict_tile<D, N, RM_FUSED>, d.n_rr_slow, TT::THREADS, 0, c.side, Lt, Vc(c, l), V(c, l - 1),
                     c.phi_b.p, (const int32_t*)d.rr_slow.p);
        if (d.n_rfix > 0)
          pdl_launch_on(k_restrict_fix<D, N>, grid_for((long long)d.n_rfix * 8, 128), 128, 0, c.side, Lf, V(c, l - 1),
                        (const int2*)d.rfix_list.p, (const int32_t*)d.rfix_tab.p, (const double*)d.rfix_gbc.p,
                        d.n_rfix);
        // 128-thread CTAs, eight per SM, two stages (three stages or 64-thread CTAs measured slower)
        if constexpr (N == 8) launch_qs<2, 8, 0, 128>(c, grid, Lt, V(c, l - 1), d.rr_plan.p, d.n_rr);
        else launch_qs<3, 1, 0, 512>(c, grid, Lt, V(c, l - 1), d.rr_plan.p, d.n_rr);
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
          PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
        const LevelDev& dp = *c.lev[(size_t)(l - 1)];
        if (dp.n_pin > 0)  // apply_pins(l-1)
          pdl_launch_on(k_pin_list, grid_for(dp.n_pin, 256), 256, 0, c.stream, V(c, l - 1).phi, c.phi_b.p,
                        (const int2*)dp.pin_list.p, dp.n_pin);
        check();
        return;
      }
    }
    if constexpr (D == 3 && N == 16) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (mode == RM_FUSED && !d.has_cf && d.n_rs == d.n_own) {
        // parents with a cut child: k_restrict_fix on the forked stream (the
        // streaming kernel leaves them alone; both only read level l)
        const bool fix = d.n_rfix > 0;
        if (fix) {
          PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
          PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
          pdl_launch(k_restrict_fix<D, N>, grid_for((long long)d.n_rfix * 8, 128), 128, 0, c.side, Lf, V(c, l - 1),
                     (const int2*)d.rfix_list.p, (const int32_t*)d.rfix_tab.p, (const double*)d.rfix_gbc.p,
                     d.n_rfix);
        }
        launch_rstream<0>(c, Lf, V(c, l - 1), d, nullptr, nullptr);
        if (fix) {
          PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
          PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
        const LevelDev& dp = *c.lev[(size_t)(l - 1)];
        if (dp.n_pin > 0)  // apply_pins(l-1)
          pdl_launch_on(k_pin_list, grid_for(dp.n_pin, 256), 256, 0, c.stream, V(c, l - 1).phi, c.phi_b.p,
                                                                    (const int2*)dp.pin_list.p, dp.n_pin);
        check();
        return;
      }
    }
    if constexpr (TILE) {
      if (mode == RM_RES)
        pdl_launch(k_restrict_tile<D, N, RM_RES>, Lf.nb, TT::THREADS, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p,
                   (const int32_t*)nullptr);
      else if (mode == RM_RHS)
        pdl_launch(k_restrict_tile<D, N, RM_RHS>, Lf.nb, TT::THREADS, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p,
                   (const int32_t*)nullptr);
      else
        pdl_launch(k_restrict_tile<D, N, RM_FUSED>, Lf.nb, TT::THREADS, 0, c.stream, Vt(c, l), Vc(c, l), V(c, l - 1), c.phi_b.p,
                   (const int32_t*)nullptr);
      check();
      return;
    }
    if (mode == RM_RES)
      pdl_launch(k_restrict<D, N, RM_RES>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p);
    else if (mode == RM_RHS)
      pdl_launch(k_restrict<D, N, RM_RHS>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1), c.phi_b.p);
    else
      pdl_launch(k_restrict<D, N, RM_FUSED>, g, kThreads, 0, c.stream, Lf, Vc(c, l), V(c, l - 1),
                                                             c.phi_b.p);
    check();
  }
  void fas(Ctx& c, int lc, bool f) override {
    const LevelView& L = V(c, lc);
    const unsigned g = grid_for((long long)L.nb * G::NI);
    if constexpr (D == 3 && N == 16) {
      const LevelDev& d = *c.lev[(size_t)lc];
      if (f && L.nb > kSmallLevel && !d.has_cf && d.n_rs == d.n_own) {
        // streaming FAS (the residual kernel in FAS mode) and the cut rows
        // cut rows on the forked stream: the streaming kernel writes g only at
        // the other rows (and OLD everywhere), k_fas_fix reads phi and g of
        // the cut rows and writes g there
        const int ncut = d.n_cut[0] + d.n_cut[1];
        if (ncut > 0) {
          PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
          PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
          pdl_launch(k_fas_fix<D, N>, grid_for(ncut, 128), 128, 0, c.side, L, (const int32_t*)d.cut_ent[0].p,
                     (const double*)d.cut_gbc[0].p, d.n_cut[0], (const int32_t*)d.cut_ent[1].p,
                     (const double*)d.cut_gbc[1].p, d.n_cut[1]);
        }
        launch_rstream<2>(c, L, L, d, nullptr, nullptr);
        if (ncut > 0) {
          PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
          PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
        check();
        return;
      }
    }
    {
      const LevelDev& d = *c.lev[(size_t)lc];
      if (L.nb <= kSmallLevel && d.has_tab) {
        if (f)
          pdl_launch_on(k_fas_tab<D, N, true>, grid_for((long long)L.nb * G::NI, 256), 256, 0, c.stream, L, c.phi_b.p,
                     (const int4*)d.tab.p, (const double*)d.tgbc.p);
        else
          pdl_launch_on(k_fas_tab<D, N, false>, grid_for((long long)L.nb * G::NI, 256), 256, 0, c.stream, L,
                     c.phi_b.p, (const int4*)d.tab.p, (const double*)d.tgbc.p);
        check();
        return;
      }
    }
    if constexpr (TILE) {
      if (L.nb > kSmallLevel) {
        if (f)
          pdl_launch_on(k_fas_tile<D, N, true>, L.nb, TT::THREADS, 0, c.stream, Vt(c, lc), Vc(c, lc), c.phi_b.p,
                        (const int32_t*)nullptr);
        else
          pdl_launch(k_fas_tile<D, N, false>, L.nb, TT::THREADS, 0, c.stream, L, Vc(c, lc), c.phi_b.p,
                     (const int32_t*)nullptr);
        check();
        return;
      }
    }
    if (f)
      pdl_launch(k_fas<D, N, true>, g, kThreads, 0, c.stream, L, Vc(c, lc), c.phi_b.p);
    else
      pdl_launch(k_fas<D, N, false>, g, kThreads, 0, c.stream, L, Vc(c, lc), c.phi_b.p);
    check();
  }
  void cfold(Ctx& c, int lc) override { cfold_on(c, lc, c.stream); }
  void cfold_on(Ctx& c, int lc, cudaStream_t s) {
    const LevelDev& d = *c.lev[(size_t)lc];
    if (d.n_cf == 0) return;
    pdl_launch_on(k_cfold_list<D, N>, grid_for((long long)d.n_cf * G::NT, 256), 256, 0, s, Vt(c, lc), Vc(c, lc),
               (const int2*)d.cf_faces.p, d.n_cf);
    check();
  }
  void fas_cfold(Ctx& c, int lc, bool f) override {
    const LevelDev& d = *c.lev[(size_t)lc];
    if (d.n_cf == 0) {
      fas(c, lc, f);
      return;
    }
    ensure_cfc(c, lc);  // on the main stream, before the fork
    PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
    PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
    cfold_on(c, lc, c.side);
    fas(c, lc, f);  // may fork again: the forked stream is in order, its join then covers the snapshot too
    PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
    PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
  }
  template <bool FULL>
  void launch_prolong_stream(Ctx& c, int l) {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      const LevelDev& d = *c.lev[(size_t)l];
      const int dead = FULL ? -1 : c.prolong_dead;
      // N = 8: 128-thread CTAs, eight per SM; CF kernel: parents with coarse-fine
      // faces take their ghosts from level l-1's cfc / cfold pages
      auto run_cf = [&](auto st, auto minb, auto th) {
        constexpr int ST = decltype(st)::value, MINB = decltype(minb)::value, TH = decltype(th)::value;
        using P = PStream3<N, TH>;
        constexpr size_t smem = (size_t)ST * P::STAGE * sizeof(double);
        set_smem_attr(c, (const void*)k_prolong_stream<N, ST, MINB, FULL, TH, true>, smem);
        const int grid = std::min(d.n_pp, c.sms * MINB);
        pdl_launch_on(k_prolong_stream<N, ST, MINB, FULL, TH, true>, grid, P::THR, smem, c.stream, V(c, l),
                      Vt(c, l - 1), (const int4*)d.pp_plan.p, d.n_pp, dead, 1);
      };
      using I2 = std::integral_constant<int, 2>;
      if constexpr (N == 8) {
        run_cf(I2{}, std::integral_constant<int, 8>{}, std::integral_constant<int, 128>{});
      } else if (d.pp_cf) {
        run_cf(I2{}, I2{}, std::integral_constant<int, 0>{});
      } else {
        constexpr int ST = 2, MINB = 2;
        constexpr size_t smem = (size_t)ST * PStream3<N>::STAGE * sizeof(double);
        set_smem_attr(c, (const void*)k_prolong_stream<N, ST, MINB, FULL>, smem);
        const int grid = std::min(d.n_pp, c.sms * MINB);
        pdl_launch_on(k_prolong_stream<N, ST, MINB, FULL>, grid, PStream3<N>::THR, smem, c.stream,
                      V(c, l), V(c, l - 1), (const int4*)d.pp_plan.p, d.n_pp, dead, 1);
      }
      if (d.n_pin > 0)  // inside cells were interpolated too: restore their pins
        pdl_launch_on(k_pin_list, grid_for(d.n_pin, 256), 256, 0, c.stream, V(c, l).phi, c.phi_b.p,
                                                                  (const int2*)d.pin_list.p, d.n_pin);
    }
  }
  void prolong(Ctx& c, int l, bool full) override {
    // level l's table (read by the sweeps that follow) depends on level l-1,
    // which the prolongation only reads: rebuilt beside it
    const bool pre = TILE && cfc_stale(c, l);
    if (pre) {
      PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
      PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
      cfc_build_side(c, l);
    }
    prolong_impl(c, l, full);
    if (pre) {
      PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
      PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
    }
  }
  void prolong_impl(Ctx& c, int l, bool full) {
    const LevelView& Lf = V(c, l);
    phi_written(c, l);
    const LevelView& Lp = V(c, l - 1);
    const LevelView& Lpp = Vc(c, l - 1);
    const unsigned g = grid_for((long long)Lf.nb * G::NI);
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      const LevelDev& d = *c.lev[(size_t)l];
      // streaming down to 64-block levels too (one block per CTA: 6.9 vs 10.1 us
      // for the generic per-cell kernel's chain of ghost lookups at 64 blocks,
      // but slower at 8)
      if (Lf.nb > (N == 16 ? 16 : kSmallLevel) && d.n_pp > 0) {
        if (full) launch_prolong_stream<true>(c, l);
        else launch_prolong_stream<false>(c, l);
        check();
        return;
      }
    }
    if constexpr (TILE) {
      if (Lf.nb > kSmallLevel) {
        const LevelView Lpt = Vt(c, l - 1);  // the parents' coarse-fine ghosts
        if (full)
          pdl_launch(k_prolong_tile<D, N, true>, Lf.nb, TT::THREADS, 0, c.stream, Lf, Lpt, Lpp);
        else
          pdl_launch(k_prolong_tile<D, N, false>, Lf.nb, TT::THREADS, 0, c.stream, Lf, Lpt, Lpp);
        check();
        return;
      }
    }
    if (full)
      pdl_launch_on(k_prolong<D, N, true>, g, kThreads, 0, c.stream, Lf, Lp, Lpp);
    else
      pdl_launch_on(k_prolong<D, N, false>, g, kThreads, 0, c.stream, Lf, Lp, Lpp);
    check();
  }
  void record(Ctx& c, int l) override {
    const LevelView& L = V(c, l);
    // a level without leaves records zeros, which enq_reset_records left there
    if (c.lev[(size_t)l]->n_leaf == 0) return;
    {
      const LevelDev& d = *c.lev[(size_t)l];
      if (L.nb <= kSmallLevel && d.has_tab) {
        const int gr = (int)grid_for((long long)L.nb * G::NI, 256);
        pdl_launch(k_record_tab<D, N>, gr, 256, 0, c.stream, L, c.phi_b.p, (const int4*)d.tab.p,
                   (const double*)d.tgbc.p, c.partial.p);
        pdl_launch(k_record_fold, 1, kFoldThreads, 0, c.stream, (const Rec*)c.partial.p, gr, c.rec.p + L.level,
                   FinishArgs{});
        check();
        return;
      }
    }
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      const LevelDev& d = *c.lev[(size_t)l];
      if ((N == 8 || d.has_cf) && d.n_rc > 0 && L.nb > kSmallLevel) {
        // N = 8, or coarse-fine faces: the column kernel (k_resid_stream, MODE 1)
        // over the leaf blocks of rc_plan, coarse-fine ghosts from the staged cfc
        // pages; the cut rows from their two tables, leaf blocks with a cut row
        // on a coarse-fine face by k_record_tile.  Partials: [0, G) streaming
        // CTAs, [G, G + g1) / [.., + g2) the cut-row CTAs, then one per listed
        // block; folded in that order.
        constexpr int MINB = N == 8 ? 8 : 1;
        const int grid = std::min(d.n_rc, c.sms * MINB);
        const int nc1 = d.n_cut[0] + d.n_cut[1], nc2 = d.n_cutcf[0] + d.n_cutcf[1];
        const int g1 = nc1 > 0 ? (int)grid_for(nc1, 256) : 0, g2 = nc2 > 0 ? (int)grid_for(nc2, 256) : 0;
        const LevelView Lt = Vt(c, l);
        const bool fork = d.n_rc_slow > 0 || nc1 > 0 || nc2 > 0;
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
          PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        }
        if (d.n_rc_slow > 0)
          pdl_launch(k_record_tile<D, N>, d.n_rc_slow, TT::THREADS, 0, c.side, Lt, Vc(c, l), c.phi_b.p,
                     c.partial.p + grid + g1 + g2, c.rec.p, (unsigned int*)nullptr, d.rc_slow.p);
        if (nc1 > 0)
          pdl_launch(k_record_cut<D>, g1, 256, 0, c.side, L, c.phi_b.p, d.cut_ent[0].p, d.cut_gbc[0].p, d.n_cut[0],
                     d.cut_ent[1].p, d.cut_gbc[1].p, d.n_cut[1], G::NI, c.partial.p + grid);
        if (nc2 > 0)
          pdl_launch(k_record_cut<D>, g2, 256, 0, c.side, L, c.phi_b.p, d.cutcf_ent[0].p, d.cutcf_gbc[0].p,
                     d.n_cutcf[0], d.cutcf_ent[1].p, d.cutcf_gbc[1].p, d.n_cutcf[1], G::NI,
                     c.partial.p + grid + g1);
        // 128-thread CTAs, eight per SM, two stages (three stages or 64-thread CTAs measured slower)
        if constexpr (N == 8) launch_qs<2, 8, 1, 128>(c, grid, Lt, Lt, d.rc_plan.p, d.n_rc);
        else launch_qs<2, 1, 1, 512>(c, grid, Lt, Lt, d.rc_plan.p, d.n_rc);
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
          PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
        FinishArgs fin{};
        if (c.finish_level == l && c.h_out_dev) {
          fin = FinishArgs{c.rec.p, c.mesh.L, l, c.outbuf.p, c.h_out_dev};
          c.finished = true;
        }
        pdl_launch(k_record_fold, 1, kFoldThreads, 0, c.stream, (const Rec*)c.partial.p, grid + g1 + g2 + d.n_rc_slow,
                   c.rec.p + L.level, fin);
        check();
        return;
      }
    }
    if constexpr (D == 3 && N == 16) {
      const LevelDev& d = *c.lev[(size_t)l];
      if (d.n_rs > 0 && L.nb > kSmallLevel) {
        // streaming record of every block without coarse-fine faces (special
        // rows excluded), the cut rows from their table and the remaining
        // blocks by k_record_tile, each into its own partials: [0, G) per
        // streaming CTA, [G, G + gcut) per cut-row CTA, then one per block of
        // the slow list; folded in that order
        const int grid = rstream_grid(c, L, d);
        const int ncut = d.n_cut[0] + d.n_cut[1];
        const int gcut = ncut > 0 ? (int)grid_for(ncut, 256) : 0;
        const bool fork = d.n_slow > 0 || ncut > 0;
        const LevelView Lt = d.n_slow > 0 ? Vt(c, l) : L;
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
          PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        }
        if (d.n_slow > 0)
          pdl_launch(k_record_tile<D, N>, d.n_slow, TT::THREADS, 0, c.side, Lt, Vc(c, l), c.phi_b.p,
                     c.partial.p + grid + gcut, c.rec.p, (unsigned int*)nullptr, d.slow_list.p);
        if (ncut > 0)
          pdl_launch(k_record_cut<D>, gcut, 256, 0, c.side, L, c.phi_b.p, d.cut_ent[0].p, d.cut_gbc[0].p,
                     d.n_cut[0], d.cut_ent[1].p, d.cut_gbc[1].p, d.n_cut[1], G::NI, c.partial.p + grid);
        launch_rstream<1>(c, L, L, d, c.partial.p, c.rec.p);
        if (fork) {
          PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
          PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
        // the cycle's last record also writes the CycleStats and the host copy
        FinishArgs fin{};
        if (c.finish_level == l && c.h_out_dev) {
          fin = FinishArgs{c.rec.p, c.mesh.L, l, c.outbuf.p, c.h_out_dev};
          c.finished = true;
        }
        pdl_launch(k_record_fold, 1, kFoldThreads, 0, c.stream, (const Rec*)c.partial.p,
                   grid + gcut + d.n_slow, c.rec.p + L.level, fin);
        check();
        return;
      }
    }
    if constexpr (TILE) {
      const LevelDev& d = *c.lev[(size_t)l];
      const bool fork = d.n_ufast > 0 && d.n_uslow > 0;
      const LevelView Lt = d.n_uslow > 0 ? Vt(c, l) : L;
      if (fork) {
        PMG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        PMG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
      }
      // one partial per listed block ([0, n_uslow) general, then the lean
      // ones), folded in that order by k_record_fold: no atomic counter, and
      // the cycle's last record writes the CycleStats and the host copy
      if (d.n_uslow > 0)
        pdl_launch(k_record_tile<D, N>, d.n_uslow, TT::THREADS, 0, fork ? c.side : c.stream, 
            Lt, Vc(c, l), c.phi_b.p, c.partial.p, c.rec.p, (unsigned int*)nullptr, d.uslow_list.p);
      if (d.n_ufast > 0)
        pdl_launch(k_record_lean<D, N>, d.n_ufast, TT::THREADS, 0, c.stream, L, c.partial.p + d.n_uslow, c.rec.p,
                                                                     (unsigned int*)nullptr, d.ufast_list.p);
      if (fork) {
        PMG_CUDA(cudaEventRecord(c.ev_join, c.side));
        PMG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
      }
      FinishArgs fin{};
      if (c.finish_level == l && c.h_out_dev) {
        fin = FinishArgs{c.rec.p, c.mesh.L, l, c.outbuf.p, c.h_out_dev};
        c.finished = true;
      }
      pdl_launch(k_record_fold, 1, kFoldThreads, 0, c.stream, (const Rec*)c.partial.p, d.n_uslow + d.n_ufast,
                 c.rec.p + L.level, fin);
      check();
      return;
    }
    pdl_launch(k_record<D, N>, L.nb, kThreads, 0, c.stream, L, Vc(c, l), c.phi_b.p, c.partial.p, c.rec.p,
                                                    c.counter.p);
    check();
  }
  void pins(Ctx& c, int l) override {
    const LevelView& L = V(c, l);
    phi_written(c, l);
    pdl_launch(k_pins<D, N>, grid_for((long long)L.nb * G::NI), kThreads, 0, c.stream, L, c.phi_b.p);
    check();
  }
  // can a 16-CTA cluster of k_coarse_cluster<N, 1> be scheduled on this device?
  bool coarse_cluster16_ok(Ctx& c) {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      using K = CC<N, 1>;
      if (K::NC <= 8) return true;
      if (c.cluster16 < 0) {
        set_cluster_attr(c, (const void*)k_coarse_cluster<N, 1>);
        cudaLaunchConfig_t cfgl = {};
        cfgl.gridDim = dim3(K::NC, 1, 1);
        cfgl.blockDim = dim3(K::THR, 1, 1);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = K::NC;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfgl.attrs = at;
        cfgl.numAttrs = 1;
        int n = 0;
        const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)k_coarse_cluster<N, 1>, &cfgl);
        if (e != cudaSuccess) (void)cudaGetLastError();
        c.cluster16 = (e == cudaSuccess && n > 0) ? 1 : 0;
      }
      return c.cluster16 == 1;
    }
    return false;
  }
  template <int PPC>
  void launch_coarse_cluster(Ctx& c, const CoarseFast& F) {
    if constexpr (D == 3 && (N == 8 || N == 16)) {
      using K = CC<N, PPC>;
      if (K::NC > 8) set_cluster_attr(c, (const void*)k_coarse_cluster<N, PPC>);
      cudaLaunchConfig_t cfgl = {};
      cfgl.gridDim = dim3(K::NC, 1, 1);
      cfgl.blockDim = dim3(K::THR, 1, 1);
      cfgl.dynamicSmemBytes = 0;
      cfgl.stream = c.stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = K::NC;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfgl.attrs = at;
      cfgl.numAttrs = 2;  // PDL: the static prologue overlaps the FAS of level 1
      PMG_CUDA(cudaLaunchKernelEx(&cfgl, k_coarse_cluster<N, PPC>, V(c, 1), F, (const double*)c.phi_b.p, c.rec.p,
                                  c.status.p, c.diag.p));
    }
  }
  void coarse(Ctx& c) override {
    phi_written(c, 1);
    if constexpr (FASTC) {
      CoarseFast F{};
      F.flags = c.cf_flags.p;
      F.diag = c.cf_diag.p;
      F.spec = c.cf_spec.p;
      F.spec_c = c.cf_spec_c.p;
      F.c0 = c.cf_c0.p;
      F.ob_start = c.cf_ob_start.p;
      F.ob_obj = c.cf_ob_obj.p;
      F.ob_val = c.cf_ob_val.p;
      F.w = c.cf_w;
      F.rel_tol = c.cfg.coarse_rel_tol;
      F.max_iters = c.cfg.coarse_max_iters;
      int lim = 1;
      for (int k = 0; k < D; ++k) lim *= 8;
      F.fallback_ok = c.coarse.n <= lim + 1;
      F.n_unknowns = c.coarse.n;
      F.pins = (const int2*)c.lev[1]->pin_list.p;
      F.n_pins = c.lev[1]->n_pin;
      if constexpr (D == 3 && (N == 8 || N == 16)) {
        // planes of the root block spread over a thread-block cluster, one
        // plane per CTA (N CTAs: a 16-CTA non-portable cluster at N=16; 786 vs
        // 796 us per V-cycle with two planes per CTA), or two planes per CTA on
        // the portable 8-CTA cluster where 16 co-resident CTAs cannot be placed
        // (MPS / green-context SM limits, partitioned devices)
        if (coarse_cluster16_ok(c)) launch_coarse_cluster<1>(c, F);
        else launch_coarse_cluster<2>(c, F);
        check();
        return;
      }
      constexpr size_t smem = coarse_fast_smem<D, N>();
      set_smem_attr(c, (const void*)k_coarse_fast<D, N>, smem);
      pdl_launch(k_coarse_fast<D, N>, 1, kCoarseThreads, smem, c.stream, V(c, 1), F, c.phi_b.p, c.rec.p,
                                                                   c.status.p, c.diag.p);
      check();
      return;
    }
    CoarseDev C{};
    C.n = c.coarse.n;
    C.nnz = (int)c.coarse.val.size();
    C.n_obj = (int)c.st.phi_b.size();
    C.rp = c.c_rp.p;
    C.ci = c.c_ci.p;
    C.val = c.c_val.p;
    C.dinv = c.c_dinv.p;
    C.c0 = c.c_c0.p;
    C.cobj = c.c_cobj.p;
    C.uaddr = c.c_uaddr.p;
    C.scratch = c.c_scratch.p;
    C.rel_tol = c.cfg.coarse_rel_tol;
    C.max_iters = c.cfg.coarse_max_iters;
    int lim = 1;
    for (int k = 0; k < D; ++k) lim *= 8;
    C.fallback_ok = c.coarse.n <= lim + 1;
    pdl_launch(k_coarse<D, N>, 1, 1024, 0, c.stream, V(c, 1), C, c.phi_b.p, c.rec.p, c.status.p, c.diag.p);
    check();
  }
  void face_gradient(Ctx& c, int n_leaves, double* faces, double* mag) override {
    constexpr long long PA = (N + 1) * (D == 3 ? N * N : N);
    // the leaf table is level-major: one launch per level over its range
    std::vector<int2> tab((size_t)n_leaves);
    if (n_leaves > 0)
      PMG_CUDA(cudaMemcpy(tab.data(), c.leaf_tab.p, (size_t)n_leaves * sizeof(int2), cudaMemcpyDeviceToHost));
    for (int q0 = 0; q0 < n_leaves;) {
      const int l = tab[(size_t)q0].x;
      int q1 = q0;
      while (q1 < n_leaves && tab[(size_t)q1].x == l) ++q1;
      const int n = q1 - q0;
      const int2* lv = (const int2*)c.leaf_tab.p + q0;
      pdl_launch(k_face_gradient<D, N>, grid_for((long long)n * D * PA, 256), 256, 0, c.stream, V(c, l), Vc(c, l),
                 lv, n, (const double*)c.phi_b.p, faces + (size_t)q0 * D * PA);
      if (mag)
        pdl_launch(k_face_magnitude<D, N>, grid_for((long long)n * G::NI, 256), 256, 0, c.stream, V(c, l), lv, n,
                   (const double*)faces + (size_t)q0 * D * PA, mag + (size_t)q0 * G::NI);
      q0 = q1;
    }
    check();
  }
  int error_norms(Ctx& c, int n_leaves, const double* origin, int tag, double phi_b, double a, double R, int vw,
                  double* part, int* err) override {
    std::vector<int2> tab((size_t)n_leaves);
    if (n_leaves > 0)
      PMG_CUDA(cudaMemcpy(tab.data(), c.leaf_tab.p, (size_t)n_leaves * sizeof(int2), cudaMemcpyDeviceToHost));
    int nb = 0;
    for (int q0 = 0; q0 < n_leaves;) {
      const int l = tab[(size_t)q0].x;
      int q1 = q0;
      while (q1 < n_leaves && tab[(size_t)q1].x == l) ++q1;
      const int n = q1 - q0;
      const unsigned g = grid_for((long long)n * G::NI, 256);
      pdl_launch(k_error_norms<D, N>, g, 256, 0, c.stream, V(c, l), (const int2*)c.leaf_tab.p + q0,
                 origin + (size_t)q0 * 3, n, tag, phi_b, a, R, vw, part + (size_t)nb * 3, err);
      nb += (int)g;
      q0 = q1;
    }
    check();
    return nb;
  }
  void scatter(Ctx& c, int l, double* dst, const double* staging, const int32_t* slot_id,
               int layout) override {
    const LevelView& L = V(c, l);
    phi_written(c, l);
    pdl_launch(k_scatter<D, N>, grid_for((long long)L.nb * G::NI), kThreads, 0, c.stream, 
        L.nb, dst, staging, slot_id, layout, L.own);
    check();
  }
  void gather(Ctx& c, int l, int var, double* staging, const int32_t* slot_id,
              int layout) override {
    const LevelView& L = V(c, l);
    const long long per = layout == 0 ? c.S : G::NI;
    pdl_launch(k_gather<D, N>, grid_for((long long)L.nb * per), kThreads, 0, c.stream, 
        L, Vc(c, l), var, staging, slot_id, layout);
    check();
  }
  void build_stencils(Ctx& c, const pmg_lsf_t* lsf, int n_lsf,
                      const pmg_stencil_cfg_t* cfg) override {
    run_stencil_build<D, N>(c, lsf, n_lsf, cfg);
  }
};

}  // namespace pmghost
