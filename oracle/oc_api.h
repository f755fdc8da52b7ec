/*
 * oc_api.h -- C interface of the CPU ORACLES (test infrastructure only).
 *
 * Two shared libraries implement exactly this interface:
 *   oracle/_ref/libpmgref.so   the reference itself: oracle/ref_capi.cpp
 *                              #includes /root/reference/proj/include/pmg/*.hpp
 *                              and forwards to pmg::TreeMesh / build_stencils /
 *                              MgSolver (compiled here, travels to the GPU box)
 *   oracle/_ref/libpmgport.so  our own CPU restatement, oracle/pmg_oracle.cpp
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load these libraries, and only as the checker or as
 * the timed CPU baseline.  The product path never links them.
 *
 * Conventions (all from the reference):
 *   - block ids are creation order (mesh.hpp:292-320); levels are 1-based;
 *   - a "padded field" is n_blocks x (N+2)^D doubles, lin(i) = sum (i_k+1)(N+2)^k
 *     (mesh.hpp:128-137);
 *   - dir = 2*axis + side, side 0 = -, 1 = + (core.hpp:79-83).
 * Every function returns 0 on success, else a pmg_status and oc_last_error()
 * holds the reference's exception text.
 */
#ifndef PMG_OC_API_H
#define PMG_OC_API_H

#include <stdint.h>
#include "../include/pmg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oc_ctx oc_ctx;

oc_ctx* oc_create(int dim, int N, const double* lo, const double* hi);
void oc_destroy(oc_ctx* h);
const char* oc_last_error(oc_ctx* h);

/* mesh (mesh.hpp:565-572 build_uniform; harness.hpp:295-321 refine_by_criterion
 * with want(b, x) = |lsf(x)| < band * b.dx) */
int oc_build_uniform(oc_ctx* h, int levels);
int oc_refine_band(oc_ctx* h, const pmg_lsf_t* lsf, int n_lsf, double band, int max_level);
/* refine_by_criterion with build_case's criteria: kind 1 b.dx > p0 max(1, |x - c| / p1)
 * (harness.hpp:351-355), kind 2 b.dx > p0 && |x - c| < p1 (harness.hpp:413-418) */
int oc_refine_crit(oc_ctx* h, int kind, double p0, double p1, const double* centre, int max_level);
/* TreeMesh::adapt with refine flags (mesh.hpp:157-175,198): flags[id] == 1 refines leaf id */
int oc_adapt(oc_ctx* h, const uint8_t* flags, int n, int max_level);
int oc_n_blocks(oc_ctx* h);
int oc_n_levels(oc_ctx* h);
/* per block: level[nb], coords[nb*3], origin[nb*3], dx[nb], parent[nb],
 * children[nb*8], nbr[nb*6], cnbr[nb*6] (unused trailing slots = -1) */
int oc_get_topology(oc_ctx* h, int32_t* level, int32_t* coords, double* origin, double* dx,
                    int32_t* parent, int32_t* children, int32_t* nbr, int32_t* cnbr);
int oc_level_blocks(oc_ctx* h, int level, int32_t* ids); /* returns count (>=0) */

/* physical BC per domain face: Dirichlet value(x) = c + sum_k g[k]*x[k] (in k order) */
int oc_set_face_bc(oc_ctx* h, int dir, int type, double c, const double* g);

int oc_set_field(oc_ctx* h, int var, const double* buf);
int oc_get_field(oc_ctx* h, int var, double* buf);

/* stencils (stencil.hpp:207-222) */
int oc_build_stencils(oc_ctx* h, const pmg_lsf_t* lsf, int n_lsf, const pmg_stencil_cfg_t* cfg);
/* boundary[nb] flags, row_count[nb]; returns total rows */
int oc_stencil_summary(oc_ctx* h, int32_t* boundary, int32_t* row_count);
/* row_of[nb*N^D] (-1 everywhere for uniform blocks); rows concatenated in
 * block-id order: center[R], nb[R*2D], bc[R*2D], d[R*2D], obj[R*2D], mask[R],
 * pin_obj[R], lin[R] */
int oc_get_stencils(oc_ctx* h, int32_t* row_of, double* center, double* nb, double* bc,
                    double* d, int8_t* obj, uint8_t* mask, int8_t* pin_obj, int32_t* lin);
/* replace all stencils (hand-built rows, KATs); same layout; n_obj phi_b values */
int oc_set_stencils(oc_ctx* h, const int32_t* boundary, const int32_t* row_count,
                    const int32_t* row_of, const double* center, const double* nb,
                    const double* bc, const double* d, const int8_t* obj,
                    const uint8_t* mask, const int8_t* pin_obj, const int32_t* lin,
                    int n_obj, const double* phi_b);
int oc_set_boundary_value(oc_ctx* h, int obj, double v);

/* solver (multigrid.hpp:292-792) */
int oc_solver_create(oc_ctx* h, const pmg_mg_cfg_t* cfg); /* ctor: validate + init() */
int oc_init(oc_ctx* h);
int oc_v_cycle(oc_ctx* h, pmg_cycle_stats_t* out);
int oc_fmg_cycle(oc_ctx* h, pmg_cycle_stats_t* out);
int oc_measure_residual(oc_ctx* h, pmg_cycle_stats_t* out);
int oc_gsrb_sweep(oc_ctx* h, int level, int parity);
int oc_fill_ghosts(oc_ctx* h, int level, int var);
int oc_apply_pins(oc_ctx* h, int level);
int oc_residual_level(oc_ctx* h, int level); /* residual_block on every block */
int oc_restrict_level(oc_ctx* h, int level);
int oc_restrict_level_no_guess(oc_ctx* h, int level);
int oc_prolong_correction(oc_ctx* h, int level);
int oc_prolong_full(oc_ctx* h, int level);
int oc_coarse_solve(oc_ctx* h);
int oc_set_have_guess(oc_ctx* h, int v);
/* assembled level-1 system (multigrid.hpp:41-57): sizes then arrays */
int oc_coarse_sizes(oc_ctx* h, int32_t* n, int32_t* nnz, int32_t* n_obj);
int oc_coarse_get(oc_ctx* h, int32_t* rp, int32_t* ci, double* val, double* c0,
                  double* cobj, int32_t* unk_block, int32_t* unk_lin);
/* KrylovResult of the BiCGStab that coarse_solve() would run on the current
 * state (b and x0 assembled as in multigrid.hpp:443-453), without changing it */
int oc_bicgstab_probe(oc_ctx* h, int32_t* converged, int32_t* iters, double* rel);

/* post-solve fields, REFERENCE BUILD ONLY (libpmgref.so): pmg::face_gradient
 * (fields.hpp:149-232) with var_out; faces[n_leaves][dim][(N+1) N^(dim-1)] in
 * FaceField order, leaf_ids[n_leaves]; either may be NULL.  Returns the
 * number of leaves, or < 0 on error. */
int oc_face_gradient(oc_ctx* h, int var, int var_out, double* faces, int32_t* leaf_ids);
/* REFERENCE BUILD ONLY: pmg::error_norms with AnalyticSolution{tag (0 sphere2d,
 * 1 sphere3d), phi_b, a, R} (fields.hpp:9-69); out = {linf, l2} */
int oc_error_norms(oc_ctx* h, int var, int tag, double phi_b, double a, double R, int vw, double* out);


#ifdef __cplusplus
}
#endif

#endif /* PMG_OC_API_H */
