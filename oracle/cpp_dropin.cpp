// cpp_dropin.cpp -- TEST INFRASTRUCTURE: the C++ drop-in check.
//
// Builds reference harness cases with the reference's own code
// (pmg::detail::build_case, harness.hpp:324-441; RHS as run_case_t,
// harness.hpp:521-530), then solves each case twice on identical mesh copies:
//   A: pmg::MgSolver<Dim>          (the reference, CPU)
//   B: pmg::b200::MgSolver<Dim>    (include/pmg_b200/solver.hpp, GPU)
// and checks
//   * pmg::b200::build_stencils == pmg::build_stencils, every field bit-exact;
//   * the residual history of an FMG cycle + 3 V-cycles within
//     |dr| <= 1e-6 r + 16 eps (2D/dx^2) max|phi|;
//   * final PHI (with ghosts) within 1e-10 max|phi|  (§8c(ii));
//   * the mesh of every case rebuilt on the device (pmg::b200::DeviceTree,
//     include/pmg_b200/tree.hpp: refine_all / refine_by_criterion with
//     build_case's criteria, harness.hpp:332-357, 384-419) is the reference's
//     TreeMesh: ids, geometry, level lists and neighbour tables identical.
// Prints one line per case and exits non-zero on the first mismatch.
// Built by `make -C oracle dropin` into oracle/_ref/ (needs /root/reference);
// run on the GPU box by tests/test_gpu_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#include "pmg/harness.hpp"
#include "pmg/io.hpp"
#include "pmg_b200/solver.hpp"
#include "pmg_b200/tree.hpp"

using namespace pmg;

namespace {

int failures = 0;

void fail(const std::string& c, const std::string& what) {
  std::printf("FAIL %s: %s\n", c.c_str(), what.c_str());
  ++failures;
}

template <int Dim>
bool same_stencils(const StencilSet<Dim>& a, const StencilSet<Dim>& b, std::string& why) {
  if (a.by_block.size() != b.by_block.size()) return why = "block count", false;
  if (a.bv.phi_b != b.bv.phi_b) return why = "phi_b", false;
  for (size_t id = 0; id < a.by_block.size(); ++id) {
    const auto& x = a.by_block[id];
    const auto& y = b.by_block[id];
    if (x.boundary != y.boundary) return why = "boundary flag of block " + std::to_string(id), false;
    if (!x.boundary) continue;
    if (x.row_of != y.row_of) return why = "row_of of block " + std::to_string(id), false;
    if (x.rows.size() != y.rows.size()) return why = "row count of block " + std::to_string(id), false;
    for (size_t r = 0; r < x.rows.size(); ++r) {
      const auto& p = x.rows[r];
      const auto& q = y.rows[r];
      if (p.center != q.center || p.nb != q.nb || p.bc != q.bc || p.d != q.d || p.obj != q.obj ||
          p.mask != q.mask || p.pin_obj != q.pin_obj || p.lin != q.lin) {
        char b[160];
        std::snprintf(b, sizeof b, " (lin %d/%d mask %d/%d center %.17g/%.17g d0 %.17g/%.17g)", p.lin, q.lin,
                      p.mask, q.mask, p.center, q.center, p.d[0], q.d[0]);
        return why = "row " + std::to_string(r) + " of block " + std::to_string(id) + b, false;
      }
    }
  }
  return true;
}

// Op-by-op diagnosis (run when a case fails): the public MgSolver operators
// of an FMG-like sequence, comparing the interiors of PHI/RHS/RES/OLD after
// every operation; prints the first op whose result differs.
template <int Dim>
void diagnose(const std::string& name, TreeMesh<Dim> mesh, StencilSet<Dim> set) {
  TreeMesh<Dim> mesh_b = mesh;
  StencilSet<Dim> set_b = set;
  MgConfig mg;
  mg.threads = 8;
  MgSolver<Dim> a(mesh, set, mg);
  b200::MgSolver<Dim> b(mesh_b, set_b, mg);
  b.set_sync_to_host(false);
  const int L = mesh.n_levels(), N = mesh.block_size();
  const size_t S = mesh.var_stride();
  std::vector<double> buf((size_t)mesh.n_blocks() * S);
  // interior cells of every var, plus the face ghosts of PHI (corners are
  // never read, mesh.hpp:471-554)
  auto cmp = [&](const std::string& op) {
    for (int var : {VAR_PHI, VAR_RHS, VAR_OLD}) {  // RES: the GPU fuses it away
      b200::detail::check(b.context(), pmg_b200_download_field(b.context(), var, buf.data(), PMG_LAYOUT_PADDED));
      double m = 0, d = 0;
      int shown = 0;
      for (int id = 0; id < mesh.n_blocks(); ++id) {
        IVec<Dim> lo, hi;
        lo.fill(var == VAR_PHI ? -1 : 0);
        hi.fill(var == VAR_PHI ? N + 1 : N);
        for_box<Dim>(lo, hi, [&](const IVec<Dim>& i) {
          int outside = 0;
          for (int k = 0; k < Dim; ++k) outside += (i[k] < 0 || i[k] >= N);
          if (outside > 1) return;  // edge/corner ghosts
          const int l = mesh.lin(i);
          const double x = mesh.field(id, var)[l], y = buf[(size_t)id * S + (size_t)l];
          m = std::max(m, std::abs(x));
          d = std::max(d, std::abs(x - y));
          if (std::abs(x - y) > 1e-12 && shown < 6) {
            ++shown;
            int ii = 0;
            for (int k = Dim - 1; k >= 0; --k) ii = ii * N + std::min(std::max(i[k], 0), N - 1);
            const auto& st = set.by_block[(size_t)id];
            const int r = st.boundary ? st.row_of[(size_t)ii] : -1;
            std::printf("    var %d block %d (level %d coords %d,%d,%d) cell %d,%d,%d%s ref %.17g gpu %.17g row %d mask %d\n",
                        var, id, mesh.block(id).level, mesh.block(id).coords[0], mesh.block(id).coords[1],
                        Dim == 3 ? mesh.block(id).coords[Dim - 1] : 0, i[0], i[1], Dim == 3 ? i[Dim - 1] : 0,
                        outside ? " (ghost)" : "", x, y, r, r >= 0 ? st.rows[(size_t)r].mask : -1);
          }
        });
      }
      if (d > 1e-12 * std::max(m, 1.0)) {
        std::printf("  diverged after %s: var %d max|d| %.3e (max %.3e)\n", op.c_str(), var, d, m);
        return false;
      }
    }
    return true;
  };
  std::printf("  diagnose %s\n", name.c_str());
  if (!cmp("init")) return;
  auto smooth = [&](int l) {
    for (int p = 0; p < 2; ++p) {
      a.gsrb_sweep(l, p);
      mesh.fill_ghosts(l, VAR_PHI, &a.pool());
      b.gsrb_sweep(l, p);
      if (!cmp("gsrb level " + std::to_string(l) + " parity " + std::to_string(p))) return false;
    }
    return true;
  };
  for (int l = L; l >= 2; --l) {  // FMG descent: restrict g, phi
    a.restrict_level_no_guess(l);
    b.restrict_level_no_guess(l);
    if (!cmp("restrict_level_no_guess " + std::to_string(l))) return;
  }
  a.coarse_solve();
  b.coarse_solve();
  if (!cmp("coarse_solve (fmg)")) return;
  for (int l = 2; l <= L; ++l) {
    a.prolong_full(l);
    b.prolong_full(l);
    if (!cmp("prolong_full " + std::to_string(l))) return;
    if (!smooth(l)) return;
  }
  for (int l = L; l >= 2; --l) {  // V-cycle descent
    if (!smooth(l)) return;
    a.restrict_level(l);
    b.restrict_level(l);
    if (!cmp("restrict_level " + std::to_string(l))) return;
  }
  a.coarse_solve();
  b.coarse_solve();
  if (!cmp("coarse_solve")) return;
  for (int l = 2; l <= L; ++l) {
    a.prolong_correction(l);
    b.prolong_correction(l);
    if (!cmp("prolong_correction " + std::to_string(l))) return;
    if (!smooth(l)) return;
  }
  std::printf("  op sequence agrees\n");
}

// build_case's mesh (harness.hpp:324-441) rebuilt on the device
template <int Dim>
bool tree_matches(const CaseConfig& cfg, const TreeMesh<Dim>& mesh, std::string& why) {
  const std::string& id = cfg.case_id;
  b200::DeviceTree<Dim> tree(mesh.domain_lo(), mesh.domain_hi(), cfg.block_size);
  const double dx_min = mesh.level_dx(cfg.max_level);
  if (id == "sphere_refined") {  // harness.hpp:348-356
    tree.refine_radial(dx_min, cfg.radius, Vec<Dim>{}, cfg.max_level);
  } else if (id == "two_electrodes") {  // harness.hpp:384-419
    const int base = std::max(1, cfg.max_level - 2);
    tree.refine_all(base - 1, base);
    Vec<Dim> tip{};  // the reference sets the tip in 3D only (harness.hpp:398-403)
    if constexpr (Dim == 3) tip = Vec<Dim>{{0.5, 0.5, 0.8}};
    tree.refine_ball(dx_min, cfg.tip_refine_radius, tip, cfg.max_level);
  } else {  // build_uniform (mesh.hpp:565-572)
    tree.refine_all(cfg.max_level - 1, cfg.max_level);
  }
  return tree.same_as(mesh, &why);
}

template <int Dim>
void run(CaseConfig cfg) {
  const std::string name = cfg.case_id + "/" + std::to_string(Dim) + "D/L" + std::to_string(cfg.max_level);
  if (cfg.w_min <= 0) cfg.w_min = 1.0 / (cfg.block_size * (1 << (cfg.max_level - 1)));
  detail::CaseSetup<Dim> setup = detail::build_case<Dim>(cfg);
  TreeMesh<Dim>& mesh = setup.mesh;
  {
    std::string why;
    if (!tree_matches<Dim>(cfg, mesh, why)) return fail(name, "device tree differs: " + why);
  }
  if (setup.rhs) {
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
  ThreadPool pool(8);
  StencilSet<Dim> set_a = build_stencils(mesh, setup.lsf, sc, &pool);
  StencilSet<Dim> set_b = b200::build_stencils(mesh, setup.lsf, sc);
  std::string why;
  if (!same_stencils(set_a, set_b, why)) return fail(name, "stencils differ: " + why);

  const TreeMesh<Dim> mesh0 = mesh;
  const StencilSet<Dim> set0 = set_a;
  TreeMesh<Dim> mesh_b = mesh;  // identical copy for the GPU solver
  MgConfig mg;
  mg.threads = 8;
  MgSolver<Dim> a(mesh, set_a, mg);
  b200::MgSolver<Dim> b(mesh_b, set_b, mg);

  double maxphi = 0;
  std::vector<CycleStats> ha{a.measure_residual()}, hb{b.measure_residual()};
  ha.push_back(a.fmg_cycle());
  hb.push_back(b.fmg_cycle());
  for (int c = 0; c < 3; ++c) {
    ha.push_back(a.v_cycle());
    hb.push_back(b.v_cycle());
  }
  const size_t S = mesh.var_stride();
  for (int id = 0; id < mesh.n_blocks(); ++id)
    for (size_t k = 0; k < S; ++k) maxphi = std::max(maxphi, std::abs(mesh.field(id, VAR_PHI)[k]));
  const double dxf = mesh.level_dx(mesh.n_levels());
  const double eps = 2.220446049250313e-16;
  for (size_t k = 0; k < ha.size(); ++k) {
    const double tol_m = 1e-6 * ha[k].max_resid + 16 * eps * (2.0 * Dim / (dxf * dxf)) * maxphi;
    const double tol_2 = 1e-6 * ha[k].l2_resid + 16 * eps * (2.0 * Dim / (dxf * dxf)) * maxphi;
    if (std::abs(ha[k].max_resid - hb[k].max_resid) > tol_m ||
        std::abs(ha[k].l2_resid - hb[k].l2_resid) > tol_2) {
      char buf[200];
      std::snprintf(buf, sizeof buf, "residual %zu: ref %.17g/%.17g gpu %.17g/%.17g", k, ha[k].max_resid,
                    ha[k].l2_resid, hb[k].max_resid, hb[k].l2_resid);
      fail(name, buf);
      return diagnose<Dim>(name, mesh0, set0);
    }
  }
  // PHI with ghosts, as left in the host mesh by each solver
  double dmax = 0;
  for (int id = 0; id < mesh.n_blocks(); ++id)
    for (size_t k = 0; k < S; ++k)
      dmax = std::max(dmax, std::abs(mesh.field(id, VAR_PHI)[k] - mesh_b.field(id, VAR_PHI)[k]));
  if (dmax > 1e-10 * maxphi) {
    fail(name, "phi differs by " + std::to_string(dmax));
    return diagnose<Dim>(name, mesh0, set0);
  }
  // device-side dump (pmg_b200_write_dump) against the reference's write_dump
  // (io.hpp:23-71) of the same field: mesh_b holds the GPU's PHI after the sync
  {
    std::string tag = name;
    for (char& ch : tag)
      if (ch == '/' || ch == ' ') ch = '_';
    const std::string pa = "/tmp/pmg_dropin_ref_" + tag + ".dump", pb = "/tmp/pmg_dropin_gpu_" + tag + ".dump";
    write_dump<Dim>(mesh_b, VAR_PHI, pa, "phi");
    b200::detail::check(b.context(), pmg_b200_write_dump(b.context(), VAR_PHI, pb.c_str(), "phi"));
    std::ifstream fa(pa, std::ios::binary), fb(pb, std::ios::binary);
    const std::string da((std::istreambuf_iterator<char>(fa)), std::istreambuf_iterator<char>());
    const std::string db((std::istreambuf_iterator<char>(fb)), std::istreambuf_iterator<char>());
    std::remove(pa.c_str());
    std::remove(pb.c_str());
    if (da.empty() || da != db) return fail(name, "device dump differs from the reference's write_dump");
  }
  std::printf("ok   %-28s blocks %6d  resid %.3e -> %.3e (gpu %.3e)  max|dphi| %.2e\n", name.c_str(),
              mesh.n_blocks(), ha[0].max_resid, ha.back().max_resid, hb.back().max_resid, dmax);
}

CaseConfig make(const std::string& id, int dim, int N, int L) {
  CaseConfig c;
  c.case_id = id;
  c.dim = dim;
  c.block_size = N;
  c.max_level = L;
  c.threads = 8;
  return c;
}

}  // namespace

int main() {
  try {
    run<3>(make("sphere_uniform", 3, 16, 4));
    run<3>(make("sphere_refined", 3, 8, 5));
    run<2>(make("shape2d_heart", 2, 8, 6));
    run<2>(make("shape2d_astroid", 2, 16, 5));
    run<3>(make("shape3d_cyl_rhombus", 3, 8, 4));
    run<3>(make("two_electrodes", 3, 8, 5));
    run<2>(make("manufactured", 2, 16, 5));
    run<3>(make("manufactured", 3, 8, 4));
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 2;
  }
  std::printf(failures ? "FAILED %d\n" : "ALL OK\n", failures);
  return failures ? 1 : 0;
}
