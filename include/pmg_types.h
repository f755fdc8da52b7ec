/*
 * pmg_types.h -- plain-old-data descriptors shared by the B200 C-ABI
 * (include/pmg_b200.h) and the CPU oracles (oracle/oc_api.h).
 *
 * Every struct here is the ABI-safe image of a reference C++ type that cannot
 * cross a C boundary (std::function, std::vector, templates on Dim):
 *
 *   pmg_lsf_t          <- pmg::LevelSetSpec<Dim>   (proj/include/pmg/levelset.hpp:31-52)
 *   pmg_stencil_cfg_t  <- pmg::StencilBuildConfig  (proj/include/pmg/stencil.hpp:115-120)
 *                         + pmg::RootSearchConfig   (proj/include/pmg/levelset.hpp:170-183)
 *   pmg_mg_cfg_t       <- pmg::MgConfig            (proj/include/pmg/multigrid.hpp:12-28)
 *   pmg_cycle_stats_t  <- pmg::CycleStats          (proj/include/pmg/multigrid.hpp:31-34)
 *
 * A composite level set (Shape::composite_min, levelset.hpp:42) is passed as
 * an array: element 0 is the composite itself, elements 1..n its children
 * (the reference forbids nesting).
 */
#ifndef PMG_TYPES_H
#define PMG_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* pmg::Shape (levelset.hpp:13-22), same order */
enum pmg_shape {
  PMG_SHAPE_NONE = 0,
  PMG_SHAPE_SPHERE = 1,
  PMG_SHAPE_SPHEROID = 2,
  PMG_SHAPE_RHOMBUS = 3,
  PMG_SHAPE_HEART = 4,
  PMG_SHAPE_ASTROID = 5,
  PMG_SHAPE_ROD = 6,
  PMG_SHAPE_COMPOSITE_MIN = 7
};

typedef struct pmg_lsf {
  int32_t shape;       /* enum pmg_shape */
  int32_t cylindrical; /* 3D revolved variant of the sharp shapes */
  double center[3];
  double radius;
  double seg_a[3], seg_b[3];
  double boundary_value;
  double shift_p, shift_q, scale;
} pmg_lsf_t;

typedef struct pmg_stencil_cfg {
  double eps_tol;        /* RootSearchConfig::eps_tol (1e-8) */
  int32_t max_bracket_iters; /* RootSearchConfig::max_bracket_iters (45) */
  double d_min;          /* RootSearchConfig::d_min (1e-4) */
  double w_min;          /* StencilBuildConfig::w_min (1e-3) */
  double boundary_safety;/* StencilBuildConfig::boundary_safety (1.5) */
  int32_t thin_rescue;   /* StencilBuildConfig::thin_rescue (1) */
} pmg_stencil_cfg_t;

typedef struct pmg_mg_cfg {
  int32_t n_down;          /* 2 */
  int32_t n_up;            /* 2 */
  double coarse_rel_tol;   /* 1e-6 */
  int32_t coarse_max_iters;/* 2000 */
  int32_t threads;         /* host threads (oracle only; ignored on the GPU) */
} pmg_mg_cfg_t;

typedef struct pmg_cycle_stats {
  double max_resid;
  double l2_resid;
} pmg_cycle_stats_t;

/* pmg::FaceBcType (mesh.hpp:22) */
enum pmg_face_bc_type { PMG_BC_DIRICHLET = 0, PMG_BC_NEUMANN_ZERO = 1 };

/* Var slots (mesh.hpp:13-20) */
enum pmg_var { PMG_VAR_PHI = 0, PMG_VAR_RHS = 1, PMG_VAR_RES = 2, PMG_VAR_OLD = 3, PMG_VAR_AUX = 4 };

/* Stencil-row masks (stencil.hpp:20-21) */
enum { PMG_SOLVED = 0, PMG_INSIDE = 1 };

/* Status codes returned by every C entry point. */
enum pmg_status {
  PMG_OK = 0,
  PMG_ERR_INVALID_ARG = 1, /* std::runtime_error from require() */
  PMG_ERR_CUDA = 2,
  PMG_ERR_COARSE_STALL = 3, /* multigrid.hpp:461-464 / :600 */
  PMG_ERR_NONFINITE = 4,
  PMG_ERR_STATE = 5,        /* call order (e.g. cycle before init) */
  PMG_ERR_TOPOLOGY = 6      /* std::logic_error (mesh.hpp:464) */
};

#ifdef __cplusplus
}
#endif

#endif /* PMG_TYPES_H */
