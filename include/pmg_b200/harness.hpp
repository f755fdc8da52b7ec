// pmg_b200/harness.hpp -- the reference experiment harness on the B200.
//
//   #include "pmg/harness.hpp"
//   #include "pmg_b200/harness.hpp"
//   pmg::CaseReport rep = pmg::b200::run_case(cfg);   // was pmg::run_case(cfg)
//
// pmg::b200::run_case restates pmg::detail::run_case_t (harness.hpp:506-595)
// with the GPU doing the work: the case is built by the reference's own
// build_case (mesh, level set, boundary conditions, refinement) and RHS fill,
// the stencils by pmg::b200::build_stencils (bit-identical), the cycles by
// pmg::b200::MgSolver without a host copy of PHI per cycle.  The per-cycle
// error norms of the sphere cases (AnalyticSolution) are evaluated on the
// device; the manufactured case's product-of-sines solution has no device
// form, so PHI is copied back for it each cycle (as the drop-in solver's
// default would).  two_electrodes' face_gradient runs on the device.  The
// reports are written by the reference's own write_outputs_t, so
// residuals.csv, errors.csv, mesh_stats.txt, config_resolved.cfg and the dumps
// have the reference's formats (%.17g rows) -- the residual and error columns
// agree with the CPU run to the fp64 tolerance of SURVEY.md §8c, the seconds
// column is the GPU's.
#ifndef PMG_B200_HARNESS_HPP
#define PMG_B200_HARNESS_HPP

#include <chrono>
#include <cmath>
#include <string>

#include "pmg/harness.hpp"
#include "pmg_b200/solver.hpp"

namespace pmg {
namespace b200 {

namespace detail {

template <int Dim>
CaseReport run_case_t(CaseConfig cfg, const ProgressFn& progress, int device) {
  using clock = std::chrono::steady_clock;
  auto seconds_since = [](clock::time_point t0) {
    return std::chrono::duration<double>(clock::now() - t0).count();
  };
  // harness.hpp:515-516: the thin-boundary search skips the finest level
  if (cfg.w_min <= 0) cfg.w_min = 1.0 / (cfg.block_size * (1 << (cfg.max_level - 1)));

  pmg::detail::CaseSetup<Dim> setup = pmg::detail::build_case<Dim>(cfg);
  TreeMesh<Dim>& mesh = setup.mesh;
  if (setup.rhs) {  // harness.hpp:521-530
    IVec<Dim> zero{}, nn;
    nn.fill(mesh.block_size());
    for (int id = 0; id < mesh.n_blocks(); ++id) {
      double* g = mesh.field(id, VAR_RHS);
      for_box<Dim>(zero, nn, [&](const IVec<Dim>& i) { g[mesh.lin(i)] = setup.rhs(mesh.cell_center(id, i)); });
    }
  }

  StencilBuildConfig sc;
  sc.root = RootSearchConfig{cfg.eps_tol, cfg.max_bracket_iters, cfg.d_min};
  sc.w_min = cfg.w_min;
  sc.boundary_safety = cfg.boundary_safety;
  sc.thin_rescue = cfg.thin_rescue;

  CaseReport rep;
  auto t0 = clock::now();
  StencilSet<Dim> set = b200::build_stencils<Dim>(mesh, setup.lsf, sc, device);
  rep.stencil_build_seconds = seconds_since(t0);
  rep.stats = pmg::detail::collect_stats(mesh, set);

  MgConfig mg;
  mg.n_up = cfg.n_up;
  mg.n_down = cfg.n_down;
  mg.cycle = cfg.cycle_type == "v" ? CycleType::v : CycleType::fmg;
  mg.coarse_rel_tol = cfg.coarse_rel_tol;
  mg.max_cycles = cfg.cycles;
  mg.target_resid = cfg.target_resid;
  mg.threads = cfg.threads;

  // the sphere cases' exact solution (build_case, harness.hpp:341-346) on the device
  const bool sphere = cfg.case_id == "sphere_uniform" || cfg.case_id == "sphere_refined";
  AnalyticSolution sol;
  sol.tag = Dim == 2 ? AnalyticSolution::Case::sphere2d : AnalyticSolution::Case::sphere3d;
  sol.R = cfg.radius;

  try {
    b200::MgSolver<Dim> solver(mesh, set, mg, device);
    solver.set_sync_to_host(false);
    CycleStats s0 = solver.measure_residual();
    rep.initial_max_resid = s0.max_resid;
    rep.initial_l2_resid = s0.l2_resid;
    rep.has_errors = setup.has_analytic;
    for (int c = 1; c <= cfg.cycles; ++c) {
      auto tc = clock::now();
      CycleStats s = solver.run_cycle();
      rep.cycles.push_back(CycleRecord{s.max_resid, s.l2_resid, seconds_since(tc)});
      if (setup.has_analytic) {
        ErrorRecord e;
        if (sphere) {
          const ErrorNorms un = solver.error_norms(sol, false);
          e.linf = un.linf;
          e.l2 = un.l2;
          e.l2_vw = solver.error_norms(sol, true).l2;
        } else {  // a callable exact solution: evaluated on the host
          solver.sync_to_host();
          const ErrorNorms un = error_norms<Dim>(mesh, set, VAR_PHI, setup.exact, false);
          e.linf = un.linf;
          e.l2 = un.l2;
          e.l2_vw = error_norms<Dim>(mesh, set, VAR_PHI, setup.exact, true).l2;
        }
        rep.errors.push_back(e);
      }
      if (progress) progress(c, rep.cycles.back());
      if (!std::isfinite(s.max_resid)) throw std::runtime_error("residual diverged (non-finite)");
      if (cfg.target_resid > 0 && s.max_resid <= cfg.target_resid) break;
    }
    if (cfg.case_id == "two_electrodes") solver.face_gradient(VAR_AUX);
    solver.sync_to_host();  // the dumps below read the mesh
  } catch (const std::exception& e) {
    rep.fail_reason = e.what();
  }

  if (rep.fail_reason.empty() && !rep.cycles.empty()) {
    if (cfg.target_resid > 0)
      rep.converged = rep.cycles.back().max_resid <= cfg.target_resid;
    else
      rep.converged = rep.reduction() >= 1e6 || rep.final_max_resid() == 0;
  }
  if (!cfg.out_dir.empty()) pmg::detail::write_outputs_t(cfg, rep, mesh);
  return rep;
}

}  // namespace detail

/// pmg::run_case (harness.hpp:598-603) on the GPU `device`.
inline CaseReport run_case(const CaseConfig& cfg, const ProgressFn& progress = nullptr, int device = 0) {
  cfg.validate();
  return cfg.dim == 2 ? detail::run_case_t<2>(cfg, progress, device) : detail::run_case_t<3>(cfg, progress, device);
}

}  // namespace b200
}  // namespace pmg

#endif  // PMG_B200_HARNESS_HPP
