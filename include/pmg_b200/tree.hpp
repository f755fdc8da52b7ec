// pmg_b200/tree.hpp -- the block tree on the device, in the reference's C++ vocabulary.
//
// pmg::b200::DeviceTree<Dim> holds the topology of a pmg::TreeMesh<Dim>
// (mesh.hpp:37-55, 60-150) in HBM and refines it there: the constructor,
// refine_all, adapt with refine flags and its 2:1 balancing
// (mesh.hpp:66-82, 157-175, 198, 206-216, 253-320), rebuild_topology
// (mesh.hpp:429-469) and refine_by_criterion (harness.hpp:295-321) with the
// criterion evaluated by a kernel.  Block ids, geometry, the level lists and
// both neighbour tables are the reference's, bit for bit; `same_as` checks a
// tree against a reference-built mesh, `attach` hands it to a solver context.
//
// Header-only over the C-ABI (pmg_b200_tree_*, include/pmg_b200.h); include
// after the reference's "pmg/mesh.hpp" / "pmg/levelset.hpp".
#ifndef PMG_B200_TREE_HPP
#define PMG_B200_TREE_HPP

#include <stdexcept>
#include <string>
#include <vector>

#include "pmg/levelset.hpp"
#include "pmg/mesh.hpp"
#include "pmg_b200.h"

namespace pmg {
namespace b200 {

template <int Dim>
class DeviceTree {
 public:
  /// TreeMesh(lo, hi, block_size) (mesh.hpp:66-82): the root block.
  DeviceTree(const Vec<Dim>& lo, const Vec<Dim>& hi, int block_size, int device = 0) {
    double l[3] = {0, 0, 0}, h[3] = {0, 0, 0};
    for (int k = 0; k < Dim; ++k) l[k] = lo[k], h[k] = hi[k];
    t_ = pmg_b200_tree_create(Dim, block_size, l, h, device);
    if (!t_) throw std::runtime_error("pmg_b200_tree_create: out of memory");
    const std::string e = pmg_b200_tree_last_error(t_);
    if (!e.empty()) {
      pmg_b200_tree_destroy(t_);
      throw std::runtime_error(e);
    }
  }
  ~DeviceTree() { pmg_b200_tree_destroy(t_); }
  DeviceTree(const DeviceTree&) = delete;
  DeviceTree& operator=(const DeviceTree&) = delete;

  int n_blocks() const { return pmg_b200_tree_n_blocks(t_); }
  int n_levels() const { return pmg_b200_tree_n_levels(t_); }

  /// TreeMesh::refine_all (mesh.hpp:206-216).
  void refine_all(int times, int max_level) { check(pmg_b200_tree_refine_all(t_, times, max_level)); }

  /// TreeMesh::adapt, refine flags (mesh.hpp:157-175, 198).  Coarsen flags
  /// are not supported on the device and are rejected.
  int adapt(const std::vector<RefineFlag>& flags, int max_level) {
    std::vector<uint8_t> f(flags.size());
    for (size_t i = 0; i < flags.size(); ++i) {
      if (flags[i] == RefineFlag::coarsen) throw std::runtime_error("device tree: coarsening is not supported");
      f[i] = flags[i] == RefineFlag::refine ? 1 : 0;
    }
    int n = 0;
    check(pmg_b200_tree_adapt(t_, f.data(), (int)f.size(), 0, max_level, &n));
    return n;
  }

  /// refine_by_criterion (harness.hpp:295-321) with want(b, x) = |f(x)| < band * b.dx.
  void refine_band(const LevelSetSpec<Dim>& lsf, double band, int max_level) {
    std::vector<pmg_lsf_t> d;
    auto one = [&](const LevelSetSpec<Dim>& s) {
      pmg_lsf_t x{};
      x.shape = (int32_t)s.shape;
      x.cylindrical = s.cylindrical ? 1 : 0;
      for (int k = 0; k < Dim; ++k) {
        x.center[k] = s.center[k];
        x.seg_a[k] = s.seg_a[k];
        x.seg_b[k] = s.seg_b[k];
      }
      x.radius = s.radius;
      x.boundary_value = s.boundary_value;
      x.shift_p = s.shift_p;
      x.shift_q = s.shift_q;
      x.scale = s.scale;
      d.push_back(x);
    };
    one(lsf);
    if (lsf.shape == Shape::composite_min)
      for (const auto& c : lsf.children) one(c);
    check(pmg_b200_tree_refine_by_criterion(t_, 0, d.data(), (int)d.size(), band, 0.0, nullptr, max_level));
  }
  /// ... with want(b, x) = b.dx > dx_min * max(1, |x - centre| / R)  (harness.hpp:351-355).
  void refine_radial(double dx_min, double R, const Vec<Dim>& centre, int max_level) {
    double c[3] = {0, 0, 0};
    for (int k = 0; k < Dim; ++k) c[k] = centre[k];
    check(pmg_b200_tree_refine_by_criterion(t_, 1, nullptr, 0, dx_min, R, c, max_level));
  }
  /// ... with want(b, x) = b.dx > dx_tip && |x - tip| < r_tip  (harness.hpp:413-418).
  void refine_ball(double dx_tip, double r_tip, const Vec<Dim>& tip, int max_level) {
    double c[3] = {0, 0, 0};
    for (int k = 0; k < Dim; ++k) c[k] = tip[k];
    check(pmg_b200_tree_refine_by_criterion(t_, 2, nullptr, 0, dx_tip, r_tip, c, max_level));
  }

  /// TreeMesh::level_blocks (mesh.hpp:102-105).
  std::vector<int> level_blocks(int level) const {
    int n = 0;
    check(pmg_b200_tree_level_blocks(t_, level, nullptr, &n));
    std::vector<int32_t> ids((size_t)(n > 0 ? n : 1));
    check(pmg_b200_tree_level_blocks(t_, level, ids.data(), &n));
    return std::vector<int>(ids.begin(), ids.begin() + n);
  }

  /// True when `mesh` has exactly this tree: ids, geometry (bitwise), parent /
  /// children, level lists and both neighbour tables.
  bool same_as(const TreeMesh<Dim>& mesh, std::string* why = nullptr) const {
    auto no = [&](const std::string& w) {
      if (why) *why = w;
      return false;
    };
    const int nb = n_blocks();
    if (nb != mesh.n_blocks()) return no("block count " + std::to_string(nb) + " vs " + std::to_string(mesh.n_blocks()));
    if (n_levels() != mesh.n_levels()) return no("level count");
    std::vector<int32_t> level(nb), coords((size_t)nb * 3), parent(nb), children((size_t)nb * 8), nbr((size_t)nb * 6),
        cnbr((size_t)nb * 6);
    std::vector<double> origin((size_t)nb * 3), dx(nb);
    check(pmg_b200_tree_get(t_, level.data(), coords.data(), origin.data(), dx.data(), parent.data(),
                            children.data(), nbr.data(), cnbr.data()));
    for (int id = 0; id < nb; ++id) {
      const Block<Dim>& b = mesh.block(id);
      const std::string at = " of block " + std::to_string(id);
      if (b.level != level[id]) return no("level" + at);
      if (b.dx != dx[id]) return no("dx" + at);
      if (b.parent != parent[id]) return no("parent" + at);
      for (int k = 0; k < Dim; ++k) {
        if (b.coords[k] != coords[(size_t)id * 3 + k]) return no("coords" + at);
        if (b.origin[k] != origin[(size_t)id * 3 + k]) return no("origin" + at);
      }
      for (int c = 0; c < (1 << Dim); ++c)
        if (b.children[c] != children[(size_t)id * 8 + c]) return no("children" + at);
      for (int f = 0; f < 2 * Dim; ++f) {
        if (b.nbr[f] != nbr[(size_t)id * 6 + f]) return no("nbr" + at);
        if (b.coarse_nbr[f] != cnbr[(size_t)id * 6 + f]) return no("coarse_nbr" + at);
      }
    }
    for (int l = 1; l <= n_levels(); ++l)
      if (level_blocks(l) != mesh.level_blocks(l)) return no("level list " + std::to_string(l));
    return true;
  }

  /// pmg_b200_set_mesh from the device tables.
  void attach(pmg_b200_ctx* ctx) const {
    const int rc = pmg_b200_set_mesh_from_tree(ctx, t_);
    if (rc != PMG_OK) throw std::runtime_error(pmg_b200_last_error(ctx));
  }
  pmg_b200_tree* handle() const { return t_; }

 private:
  void check(int rc) const {
    if (rc == PMG_OK) return;
    const std::string msg = pmg_b200_tree_last_error(t_);
    if (rc == PMG_ERR_TOPOLOGY) throw std::logic_error(msg);
    throw std::runtime_error(msg);
  }
  pmg_b200_tree* t_ = nullptr;
};

}  // namespace b200
}  // namespace pmg

#endif  // PMG_B200_TREE_HPP
