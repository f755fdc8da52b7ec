// harness_dropin.cpp -- TEST INFRASTRUCTURE: the experiment harness on the GPU.
//
// Runs every case the reference harness knows (harness.hpp:47-54) twice, at
// small sizes, with report files:
//   A: pmg::run_case           (the reference harness, CPU)
//   B: pmg::b200::run_case     (include/pmg_b200/harness.hpp, GPU)
// and compares the files the harness writes (write_outputs_t, harness.hpp:462-503):
//   * residuals.csv: same rows and cycle numbers; max_resid / l2_resid within
//     |dr| <= 1e-6 r + 16 eps (2D/dx^2) max|phi|;
//   * errors.csv (the analytic cases): within 1e-9 relative + 1e-13;
//   * mesh_stats.txt: identical except the stencil_build_seconds line;
//   * config_resolved.cfg: identical;
//   * solution.dump (and gradnorm.dump): identical headers, data within
//     1e-10 max|phi| (the gradient magnitude within 1e-8 relative).
// `--bench` instead times the drop-in solver's default host-synchronised
// cycle against set_sync_to_host(false) on a 3D sphere case (the reference
// caller's view of the GPU solver).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "pmg/harness.hpp"
#include "pmg/io.hpp"
#include "pmg_b200/harness.hpp"

using namespace pmg;

namespace {

int failures = 0;
void fail(const std::string& c, const std::string& what) {
  std::printf("FAIL %s: %s\n", c.c_str(), what.c_str());
  ++failures;
}

std::vector<std::string> lines(const std::string& path) {
  std::ifstream in(path);
  std::vector<std::string> v;
  std::string s;
  while (std::getline(in, s)) v.push_back(s);
  return v;
}

std::vector<std::vector<double>> csv(const std::string& path, std::string& header) {
  auto ls = lines(path);
  std::vector<std::vector<double>> rows;
  if (ls.empty()) return rows;
  header = ls[0];
  for (size_t i = 1; i < ls.size(); ++i) {
    std::vector<double> r;
    std::stringstream ss(ls[i]);
    std::string t;
    while (std::getline(ss, t, ',')) r.push_back(std::stod(t));
    rows.push_back(r);
  }
  return rows;
}

void compare_case(const CaseConfig& base) {
  const std::string name = base.case_id + "_" + std::to_string(base.dim) + "d";
  CaseConfig a = base, b = base;
  a.out_dir = "/tmp/pmg_harness/" + name + "_ref";
  b.out_dir = "/tmp/pmg_harness/" + name + "_b200";
  a.threads = 8;
  const CaseReport ra = run_case(a);
  const CaseReport rb = b200::run_case(b);
  if (!ra.fail_reason.empty() || !rb.fail_reason.empty()) {
    if (ra.fail_reason != rb.fail_reason) fail(name, "fail_reason '" + ra.fail_reason + "' vs '" + rb.fail_reason + "'");
    return;
  }
  // the floor of SURVEY.md §8c(iii): finest dx and max|phi| from the reference dump
  const DumpData da = read_dump(a.out_dir + "/solution.dump");
  const DumpData db = read_dump(b.out_dir + "/solution.dump");
  double maxphi = 0, dphi = 0;
  for (double v : da.data) maxphi = std::max(maxphi, std::abs(v));
  if (da.data.size() != db.data.size()) return fail(name, "dump sizes differ");
  for (size_t i = 0; i < da.data.size(); ++i) dphi = std::max(dphi, std::abs(da.data[i] - db.data[i]));
  const double dx = 1.0 / (base.block_size * (1 << (base.max_level - 1)));  // unit-extent domains
  const double floor = 16 * 2.2e-16 * (2 * base.dim / (dx * dx)) * maxphi;
  std::string ha, hb;
  const auto ca = csv(a.out_dir + "/residuals.csv", ha), cb = csv(b.out_dir + "/residuals.csv", hb);
  if (ha != hb || ca.size() != cb.size()) return fail(name, "residuals.csv shape");
  for (size_t r = 0; r < ca.size(); ++r) {
    if (ca[r][0] != cb[r][0]) return fail(name, "residuals.csv cycle column");
    for (int k = 1; k <= 2; ++k)
      if (std::abs(ca[r][k] - cb[r][k]) > 1e-6 * ca[r][k] + floor) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "residuals.csv row %zu col %d: %.17g vs %.17g", r, k, ca[r][k], cb[r][k]);
        return fail(name, buf);
      }
  }
  if (std::filesystem::exists(a.out_dir + "/errors.csv")) {
    const auto ea = csv(a.out_dir + "/errors.csv", ha), eb = csv(b.out_dir + "/errors.csv", hb);
    if (ha != hb || ea.size() != eb.size()) return fail(name, "errors.csv shape");
    for (size_t r = 0; r < ea.size(); ++r)
      for (size_t k = 1; k < ea[r].size(); ++k)
        if (std::abs(ea[r][k] - eb[r][k]) > 1e-9 * std::abs(ea[r][k]) + 1e-13) {
          char buf[160];
          std::snprintf(buf, sizeof buf, "errors.csv row %zu col %zu: %.17g vs %.17g", r, k, ea[r][k], eb[r][k]);
          return fail(name, buf);
        }
  } else if (std::filesystem::exists(b.out_dir + "/errors.csv")) {
    return fail(name, "errors.csv only on the GPU side");
  }
  auto sa = lines(a.out_dir + "/mesh_stats.txt"), sb = lines(b.out_dir + "/mesh_stats.txt");
  if (sa.size() != sb.size()) return fail(name, "mesh_stats.txt length");
  for (size_t i = 0; i < sa.size(); ++i)
    if (sa[i].rfind("stencil_build_seconds", 0) != 0 && sa[i] != sb[i])
      return fail(name, "mesh_stats.txt: '" + sa[i] + "' vs '" + sb[i] + "'");
  {  // the resolved configs differ only in out_dir and threads (the CPU run's pool)
    auto fa = lines(a.out_dir + "/config_resolved.cfg"), fb = lines(b.out_dir + "/config_resolved.cfg");
    if (fa.size() != fb.size()) return fail(name, "config_resolved.cfg length");
    for (size_t i = 0; i < fa.size(); ++i)
      if (fa[i].rfind("out_dir", 0) != 0 && fa[i].rfind("threads", 0) != 0 && fa[i] != fb[i])
        return fail(name, "config_resolved.cfg: '" + fa[i] + "' vs '" + fb[i] + "'");
  }
  if (da.block_size != db.block_size || da.blocks.size() != db.blocks.size() || da.field != db.field)
    return fail(name, "dump header");
  if (dphi > 1e-10 * maxphi) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "solution.dump max|dphi| %.3e of %.3e", dphi, maxphi);
    return fail(name, buf);
  }
  if (std::filesystem::exists(a.out_dir + "/gradnorm.dump")) {
    const DumpData ga = read_dump(a.out_dir + "/gradnorm.dump"), gb = read_dump(b.out_dir + "/gradnorm.dump");
    double m = 0, d = 0;
    for (size_t i = 0; i < ga.data.size(); ++i) {
      m = std::max(m, std::abs(ga.data[i]));
      d = std::max(d, std::abs(ga.data[i] - gb.data[i]));
    }
    if (ga.data.size() != gb.data.size() || d > 1e-8 * m) return fail(name, "gradnorm.dump");
  }
  std::printf("ok   %-24s cycles %zu  final max_resid %.3e / %.3e  max|dphi|/max|phi| %.1e  stencils %.3f s / %.3f s\n",
              name.c_str(), ca.size(), ra.final_max_resid(), rb.final_max_resid(), maxphi > 0 ? dphi / maxphi : 0.0,
              ra.stencil_build_seconds, rb.stencil_build_seconds);
}

int bench() {
  // the drop-in solver as a reference caller drives it: 3D sphere, 256^3
  CaseConfig cfg;
  cfg.case_id = "sphere_uniform";
  cfg.dim = 3;
  cfg.block_size = 16;
  cfg.max_level = 5;
  cfg.w_min = 1.0 / 256;
  auto setup = pmg::detail::build_case<3>(cfg);
  StencilBuildConfig sc;
  sc.w_min = cfg.w_min;
  StencilSet<3> set = b200::build_stencils<3>(setup.mesh, setup.lsf, sc);
  MgConfig mg;
  mg.threads = (int)std::max(1u, std::thread::hardware_concurrency());  // the host pool scatters the copy
  for (int sync = 1; sync >= 0; --sync) {
    b200::MgSolver<3> s(setup.mesh, set, mg);
    s.set_sync_to_host(sync != 0);
    s.fmg_cycle();
    for (int w = 0; w < 3; ++w) s.v_cycle();
    const int K = 20;
    auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < K; ++k) s.v_cycle();
    const double ms = 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / K;
    std::printf("BENCH sphere_uniform 3D 256^3 drop-in v_cycle %s: %.3f ms/cycle (%.3e unknowns/s)\n",
                sync ? "with the default PHI copy to the host" : "set_sync_to_host(false)", ms,
                16777216.0 / (ms * 1e-3));
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--bench") return bench();
  std::vector<CaseConfig> cases;
  auto add = [&](const std::string& id, int dim, int N, int L, int cycles, const std::string& type) {
    CaseConfig c;
    c.case_id = id;
    c.dim = dim;
    c.block_size = N;
    c.max_level = L;
    c.cycles = cycles;
    c.cycle_type = type;
    cases.push_back(c);
  };
  add("sphere_uniform", 2, 8, 5, 4, "fmg");
  add("sphere_uniform", 3, 8, 4, 3, "v");
  add("sphere_refined", 2, 8, 5, 3, "fmg");
  add("sphere_refined", 3, 8, 4, 3, "v");
  add("shape2d_spheroid", 2, 8, 5, 3, "v");
  add("shape2d_rhombus", 2, 8, 5, 3, "v");
  add("shape2d_heart", 2, 8, 5, 3, "fmg");
  add("shape2d_astroid", 2, 8, 5, 3, "v");
  add("shape3d_cyl_spheroid", 3, 8, 4, 3, "v");
  add("shape3d_cyl_rhombus", 3, 8, 4, 3, "v");
  add("shape3d_cyl_heart", 3, 8, 4, 3, "fmg");
  add("shape3d_cyl_astroid", 3, 8, 4, 3, "v");
  add("two_electrodes", 3, 8, 5, 3, "v");
  add("manufactured", 2, 8, 5, 3, "fmg");
  add("manufactured", 3, 8, 4, 3, "v");
  for (const auto& c : cases) {
    try {
      compare_case(c);
    } catch (const std::exception& e) {
      fail(c.case_id, e.what());
    }
  }
  std::printf(failures ? "%d FAILED\n" : "ALL OK\n", failures);
  return failures ? 1 : 0;
}
