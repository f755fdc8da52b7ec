/*
 * pmg_b200.h -- C-ABI of libpmg_b200.so, the B200 (sm_100a) V-cycle / FMG
 * hot path of the level-set geometric multigrid Poisson solver
 * (arXiv 2205.09411; reference C++ implementation "poissonmg").
 *
 * Plain pointers and sizes only; no C++ or torch types.  Every entry point
 * returns a pmg_status (include/pmg_types.h); pmg_b200_last_error() holds the
 * message, which for solver failures is the reference's exception text.
 *
 * Conventions follow the reference exactly: 1-based levels, block ids in the
 * caller's mesh order, dir = 2*axis + side (core.hpp:79-83), padded field
 * slices of (N+2)^D doubles with lin(i) = sum_k (i_k+1)(N+2)^k
 * (mesh.hpp:128-137), interior slices of N^D doubles x-fastest.
 *
 * Each function cites the reference interface it replaces.  A maintainer binds
 * these from the reference's C++ through include/pmg_b200/solver.hpp (a
 * header-only pmg::b200::MgSolver<D> with MgSolver's exact public surface) and
 * from Python through paper_2205_09411_b200/_lib.py (ctypes); see INTEGRATION.md.
 */
#ifndef PMG_B200_H
#define PMG_B200_H

#include <stddef.h>
#include <stdint.h>

#include "pmg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmg_b200_ctx pmg_b200_ctx;

/* Field layouts for upload/download. */
enum pmg_layout {
  PMG_LAYOUT_PADDED = 0,   /* (N+2)^D per block, Block::data var slice (mesh.hpp:47,118-125) */
  PMG_LAYOUT_INTERIOR = 1  /* N^D per block, x fastest (for_box order, core.hpp:85-97) */
};

/* ---- context ------------------------------------------------------------ */
/* replaces: TreeMesh<Dim>::TreeMesh(lo, hi, block_size) (mesh.hpp:66-82) for the
 * parts the solver reads; binds CUDA device `device`. Returns NULL only on OOM;
 * check pmg_b200_last_error(ctx) for argument errors. */
pmg_b200_ctx* pmg_b200_create(int dim, int N, const double* lo, const double* hi, int device);
void pmg_b200_destroy(pmg_b200_ctx* ctx);
const char* pmg_b200_last_error(pmg_b200_ctx* ctx);
/* cudaStream_t the context launches on (for events / interop) */
void* pmg_b200_stream(pmg_b200_ctx* ctx);

/* ---- mesh ----------------------------------------------------------------- */
/* replaces: the Block table of TreeMesh (mesh.hpp:37-55) + rebuild_topology
 * neighbour tables (mesh.hpp:429-469).  Arrays are indexed by block id:
 * level[nb], coords[nb*3], origin[nb*3], dx[nb], parent[nb], children[nb*8],
 * nbr[nb*6], cnbr[nb*6] (trailing unused entries ignored). */
int pmg_b200_set_mesh(pmg_b200_ctx* ctx, int n_blocks, const int32_t* level,
                      const int32_t* coords, const double* origin, const double* dx,
                      const int32_t* parent, const int32_t* children, const int32_t* nbr,
                      const int32_t* cnbr);
/* replaces: TreeMesh::face_bc[dir] (mesh.hpp:148, FaceBc mesh.hpp:22-32).
 * values: NULL (value 0) or, for every block with a physical face `dir`
 * (nbr == cnbr == -1) in increasing block id, N^(D-1) values bc(x_f) at the
 * face centres x_f = cell_center(b, i1) + 0.5 dx sign(dir) e_axis
 * (mesh.hpp:540-550), transverse index lower axis fastest. */
int pmg_b200_set_face_bc(pmg_b200_ctx* ctx, int dir, int type, const double* values);

/* ---- stencils ------------------------------------------------------------- */
/* replaces: StencilSet<Dim> (stencil.hpp:196-205) handed to MgSolver's ctor.
 * boundary[nb], row_count[nb]; row_of[nb*N^D] (entries of non-boundary blocks
 * ignored); rows concatenated in block-id order as SoA:
 * center[R], nb[R*2D], bc[R*2D], d[R*2D], obj[R*2D], mask[R], pin_obj[R], lin[R];
 * phi_b[n_obj] = BoundaryValues::phi_b (stencil.hpp:12-18). */
int pmg_b200_set_stencils(pmg_b200_ctx* ctx, const int32_t* boundary, const int32_t* row_count,
                          const int32_t* row_of, const double* center, const double* nb,
                          const double* bc, const double* d, const int8_t* obj,
                          const uint8_t* mask, const int8_t* pin_obj, const int32_t* lin,
                          int n_obj, const double* phi_b);
/* replaces: build_stencils(mesh, lsf, cfg) (stencil.hpp:207-222) -- runs on the
 * GPU (level-set line searches + thin-object rescue, levelset.hpp:151-382). */
int pmg_b200_build_stencils(pmg_b200_ctx* ctx, const pmg_lsf_t* lsf, int n_lsf,
                            const pmg_stencil_cfg_t* cfg);
/* read back the current StencilSet; summary returns total rows R (>= 0) */
int pmg_b200_stencil_summary(pmg_b200_ctx* ctx, int32_t* boundary, int32_t* row_count);
int pmg_b200_get_stencils(pmg_b200_ctx* ctx, int32_t* row_of, double* center, double* nb,
                          double* bc, double* d, int8_t* obj, uint8_t* mask, int8_t* pin_obj,
                          int32_t* lin);
/* replaces: StencilSet::set_boundary_value (stencil.hpp:201-204) */
int pmg_b200_set_boundary_value(pmg_b200_ctx* ctx, int obj, double value);

/* ---- fields --------------------------------------------------------------- */
/* replaces: writes/reads through TreeMesh::field(id, var) (mesh.hpp:118-125).
 * All blocks, block-id order.  Ghost values on download are the filled ghosts
 * (PHI, OLD); other vars report 0 in ghost slots. */
int pmg_b200_upload_field(pmg_b200_ctx* ctx, int var, const double* host, int layout);
int pmg_b200_download_field(pmg_b200_ctx* ctx, int var, double* host, int layout);
/* one level only, blocks in TreeMesh::level_blocks(level) order (mesh.hpp:101-105) */
int pmg_b200_upload_level_field(pmg_b200_ctx* ctx, int var, int level, const double* host,
                                int layout);
int pmg_b200_download_level_field(pmg_b200_ctx* ctx, int var, int level, double* host,
                                  int layout);
/* double-buffered upload (a new right-hand side per solve step, as in a
 * time-stepping caller): stage_field_async starts the host->device copy of
 * `host` (pinned for overlap; level 0 = all blocks, else level_blocks order)
 * on the context's copy stream and returns at once -- it overlaps whatever the
 * solver is running; commit_staged_field makes the solver stream wait for it
 * and scatters it into field `var`.  The host buffer must stay valid until the
 * commit has been issued. */
int pmg_b200_stage_field_async(pmg_b200_ctx* ctx, int var, int level, const double* host, int layout);
int pmg_b200_commit_staged_field(pmg_b200_ctx* ctx);

/* ---- solver (MgSolver<Dim>, multigrid.hpp:292-792) ------------------------ */
/* replaces: MgSolver(mesh, stencils, cfg) -- cfg.validate() then init() (:295-299) */
int pmg_b200_solver_create(pmg_b200_ctx* ctx, const pmg_mg_cfg_t* cfg);
/* replaces: MgSolver::init (:304-311) */
int pmg_b200_init(pmg_b200_ctx* ctx);
/* replaces: v_cycle (:318-323), fmg_cycle (:325-350), measure_residual (:353-360) */
int pmg_b200_v_cycle(pmg_b200_ctx* ctx, pmg_cycle_stats_t* out);
int pmg_b200_fmg_cycle(pmg_b200_ctx* ctx, pmg_cycle_stats_t* out);
int pmg_b200_measure_residual(pmg_b200_ctx* ctx, pmg_cycle_stats_t* out);
/* asynchronous variants: enqueue on pmg_b200_stream(); pmg_b200_cycle_result
 * waits and returns the stats (and the coarse-solve status) of the last one */
int pmg_b200_v_cycle_async(pmg_b200_ctx* ctx);
int pmg_b200_fmg_cycle_async(pmg_b200_ctx* ctx);
int pmg_b200_cycle_result(pmg_b200_ctx* ctx, pmg_cycle_stats_t* out);
/* op-level API (public MgSolver members) */
int pmg_b200_gsrb_sweep(pmg_b200_ctx* ctx, int level, int parity);       /* :365-370 */
int pmg_b200_fill_ghosts(pmg_b200_ctx* ctx, int level, int var);          /* mesh.hpp:217-221 (ghosts are always current: no-op) */
int pmg_b200_apply_pins(pmg_b200_ctx* ctx, int level);                     /* stencil.hpp:225-237 */
int pmg_b200_residual_level(pmg_b200_ctx* ctx, int level);                 /* :510-517 -> VAR_RES */
int pmg_b200_restrict_level(pmg_b200_ctx* ctx, int level);                 /* :374-398 (residual fused) */
int pmg_b200_restrict_level_no_guess(pmg_b200_ctx* ctx, int level);        /* :403-418 */
int pmg_b200_prolong_correction(pmg_b200_ctx* ctx, int level);             /* :422-428 */
int pmg_b200_prolong_full(pmg_b200_ctx* ctx, int level);                   /* :432-438 */
int pmg_b200_coarse_solve(pmg_b200_ctx* ctx);                              /* :442-472 */
int pmg_b200_set_have_guess(pmg_b200_ctx* ctx, int v);                     /* :480 */
/* replaces: coarse_system() (:474) -- CoarseSystem (:41-57) of level 1 */
int pmg_b200_coarse_sizes(pmg_b200_ctx* ctx, int32_t* n, int32_t* nnz, int32_t* n_obj);
int pmg_b200_coarse_get(pmg_b200_ctx* ctx, int32_t* rp, int32_t* ci, double* val, double* c0,
                        double* cobj, int32_t* unk_block, int32_t* unk_lin);

/* ---- introspection -------------------------------------------------------- */
/* kernels launched by one cycle of the given kind (0 = V, 1 = FMG, 2 = measure) */
int pmg_b200_cycle_kernel_count(pmg_b200_ctx* ctx, int kind);
/* number of refinement levels and blocks per level (after set_mesh) */
int pmg_b200_n_levels(pmg_b200_ctx* ctx);
int pmg_b200_level_size(pmg_b200_ctx* ctx, int level);
/* how the kernels split the blocks of `level` (after the stencils are set):
 * out[0] blocks, out[1] coarse-fine faces, out[2] blocks of the streaming
 * GS plan, out[3] blocks left to the block-per-CTA GS kernel (a cut row within two cells of a
 * coarse-fine face), out[4] / out[5] the same for the leaf record, out[6] /
 * out[7] for residual + restriction.  Diagnostics (tests, profiles). */
int pmg_b200_level_classes(pmg_b200_ctx* ctx, int level, int32_t* out8);
int pmg_b200_synchronize(pmg_b200_ctx* ctx);
/* a page-locked host buffer of at least `bytes`, owned by the context and
 * reused (the C++ drop-in's PHI copies to the host go through it) */
void* pmg_b200_host_buffer(pmg_b200_ctx* ctx, size_t bytes);
/* BiCGStab iterations and final relative residual of the most recent coarse
 * solve (KrylovResult, multigrid.hpp:200-204; the reference discards it) */
int pmg_b200_coarse_info(pmg_b200_ctx* ctx, int32_t* iters, double* rel);
/* ---- multi-GPU hooks (driven by paper_2205_09411_b200/distributed.py) ----
 * set_owned: the blocks of `level` this rank computes, one byte per block in
 * device slot order (Morton order of the block coordinates; NULL = all).  Every
 * kernel then skips the other blocks; their storage keeps whatever the halo
 * exchange copies in.
 * level_field_ptr: device pointer to the level's PHI / RHS / RES / OLD array
 * (n_blocks * N^D doubles, colour-split block layout) for the exchange.
 * restrict_only / fas_level: the two halves of restrict_level (multigrid.hpp:374-398)
 * -- residual + restriction into level-1, then FAS g = L(phi) + r and OLD on `level`.
 * level_record: record_leaf_residual(level) (:529-562) of the owned blocks:
 * out3 = {max |r|, sum r^2, count}. */
int pmg_b200_set_owned(pmg_b200_ctx* ctx, int level, const uint8_t* owned_by_slot);
void* pmg_b200_level_field_ptr(pmg_b200_ctx* ctx, int var, int level);
int pmg_b200_restrict_only(pmg_b200_ctx* ctx, int level);
int pmg_b200_fas_level(pmg_b200_ctx* ctx, int level);
int pmg_b200_level_record(pmg_b200_ctx* ctx, int level, double* out3);

/* ---- the Morton-partitioned V-cycle (csrc/dist.h) ----------
 * The reference has no multi-process path: this is the B200 decomposition of
 * MgSolver::v_cycle (multigrid.hpp:483-499) over one context per GPU.
 * set_partition: this context is rank `rank` of `world`; owner_of_block gives
 *   the rank of every block id on the levels >= split_level (paper_2205_09411_b200
 *   partition.morton_partition: Morton ranges of the split level, subtrees
 *   follow); the levels below belong to rank 0.  Restricts every kernel to the
 *   owned blocks and builds the device-resident halo plans (per level, per
 *   peer, per colour).  Call after set_mesh and the stencils, before
 *   solver_create.
 * nccl_unique_id: 128 bytes for ncclCommInitRank, made on rank 0 and passed
 *   to every rank by the caller.  dist_init_nccl: the NCCL transport (libnccl
 *   resolved at run time); the whole cycle -- halo pack / unpack kernels and
 *   grouped ncclSend / ncclRecv, the coarse-tail gather and broadcast, the
 *   record all-gather -- is captured into one CUDA graph.
 * dist_local_group: the in-process transport: ctxs[r] is rank r; each context
 *   must then be driven by its own host thread (device copies between the
 *   contexts, ordered by events; used to check the decomposition on one GPU).
 * dist_v_cycle: one partitioned V-cycle; the stats are every rank's records
 *   combined in rank order (the same on every rank).
 * dist_info: out6 = {world, split level, transport (0 none, 1 NCCL,
 *   2 in-process), halo cells received per sweep of every partitioned level
 *   (both colours), kernels in the captured cycle graph, graph captured (0/1)}. */
int pmg_b200_set_partition(pmg_b200_ctx* ctx, int world, int rank, int split_level, const int32_t* owner_of_block);
int pmg_b200_nccl_unique_id(unsigned char* out128);
int pmg_b200_dist_init_nccl(pmg_b200_ctx* ctx, const unsigned char* id128);
int pmg_b200_dist_local_group(int n, pmg_b200_ctx* const* ctxs);
int pmg_b200_dist_v_cycle(pmg_b200_ctx* ctx, pmg_cycle_stats_t* out);
int pmg_b200_dist_v_cycle_async(pmg_b200_ctx* ctx);
int pmg_b200_dist_info(pmg_b200_ctx* ctx, int32_t* out6);
/* device bytes held by the solution / rhs / OLD / residual arrays of every
 * level: the whole mesh on one context; on a partitioned rank only its blocks
 * and their halo blocks are backed (CUDA virtual memory), the coarse tail and
 * levels of at most 64 blocks stay whole */
int pmg_b200_field_bytes(pmg_b200_ctx* ctx, double* out);

/* ---- post-solve fields -------------------------
 * pmg::face_gradient (proj/include/pmg/fields.hpp:149-232): the staggered
 * gradient of PHI on the faces of every leaf cell -- centred difference on
 * regular faces, (phi_b - phi)/(d dx) from the solved side on faces cut by a
 * boundary, 0 inside objects -- with ghosts filled as the reference's
 * fill_ghosts would.  Leaves in dump order (level-major, x-major inside a
 * level; mesh.hpp:229-235).  faces: n_leaves x dim x (N+1) N^(dim-1) doubles,
 * per axis in FaceField::face_index order (fields.hpp:80-89).  magnitude
 * (optional): the cell-centred |grad| the reference writes to var_out,
 * n_leaves x N^dim, x-fastest.  leaf_ids (optional): the leaves' block ids.
 * var must be 0 (VAR_PHI). */
int pmg_b200_n_leaves(pmg_b200_ctx* ctx);
/* pmg::write_dump (proj/include/pmg/io.hpp:23-71): the "pmg dump 1" file of
 * field `var` over the leaf blocks, byte-identical to the reference's; the
 * field streams from the device one level at a time. */
int pmg_b200_write_dump(pmg_b200_ctx* ctx, int var, const char* path, const char* field_name);
/* pmg::error_norms with an AnalyticSolution (fields.hpp:9-69): PHI on every
 * solved leaf cell against phi_b + a log(r/R) (tag 0, sphere2d) or
 * phi_b + a (1 - R/r) (tag 1, sphere3d), r = |cell centre|; linf = max |d|,
 * l2 = RMS (cells weighted by dx^dim when volume_weighted).  A solved cell
 * with r < R fails with the reference's "analytic solution undefined inside". */
int pmg_b200_error_norms(pmg_b200_ctx* ctx, int var, int tag, double phi_b, double a, double R,
                         int volume_weighted, double* linf, double* l2);
int pmg_b200_face_gradient(pmg_b200_ctx* ctx, int var, double* faces, double* magnitude, int32_t* leaf_ids);

/* Average device time (CUDA events on pmg_b200_stream) of `reps` back-to-back
 * launches of one phase, after one untimed launch:
 *   op 0: GS-RB half-sweep on `level` (parities alternate)
 *   op 1: residual+restriction of `level` (+ FAS/OLD on level-1), as in the V-cycle
 *   op 2: prolong_correction of `level`
 *   op 3: leaf-residual record of `level`
 *   op 4: coarse solve
 *   op 5: one V-cycle (graph)        op 6: one FMG cycle (graph, with guess)
 *   op 7: residual+restriction of `level` alone   op 8: FAS/OLD of `level`-1 alone
 *   op + 100 (ops 0-4, 7, 8): the reps are captured into one CUDA graph and
 *   replayed, so launch gaps are those inside the cycle graphs
 * Ops 1-8 modify the solution exactly as the solver would. */
int pmg_b200_time_op(pmg_b200_ctx* ctx, int op, int level, int reps, double* ms_avg);

/* ---- the block tree on the device ------------------------------------------- */
/* replaces: TreeMesh<Dim>'s topology and its refinement (mesh.hpp:66-82,
 * 157-175, 198, 206-216, 253-320, 429-469) and refine_by_criterion
 * (harness.hpp:295-321).  The tree lives in HBM; flags are evaluated, the 2:1
 * balance closure is formed, new blocks are numbered and the level lists and
 * neighbour tables are rebuilt by kernels (csrc/tree.cu).  Block ids, level
 * lists and neighbour tables are identical to the reference's. */
typedef struct pmg_b200_tree pmg_b200_tree;
/* TreeMesh(lo, hi, block_size): the root block (mesh.hpp:66-82) */
pmg_b200_tree* pmg_b200_tree_create(int dim, int N, const double* lo, const double* hi, int device);
void pmg_b200_tree_destroy(pmg_b200_tree* tree);
const char* pmg_b200_tree_last_error(pmg_b200_tree* tree);
int pmg_b200_tree_n_blocks(pmg_b200_tree* tree);  /* TreeMesh::n_blocks (mesh.hpp:94) */
int pmg_b200_tree_n_levels(pmg_b200_tree* tree);  /* TreeMesh::n_levels (mesh.hpp:100) */
int pmg_b200_tree_adapt_passes(pmg_b200_tree* tree);
/* TreeMesh::refine_all(times, max_level) (mesh.hpp:206-216); build_uniform = create + refine_all(levels-1) */
int pmg_b200_tree_refine_all(pmg_b200_tree* tree, int times, int max_level);
/* TreeMesh::adapt(flags, max_level), refine flags (mesh.hpp:157-175,198): flags[id] == 1
 * (RefineFlag::refine) on a leaf refines it; the 2:1 balance forces more.
 * flags may be a host or a device pointer (flags_on_device). */
int pmg_b200_tree_adapt(pmg_b200_tree* tree, const uint8_t* flags, int n_flags, int flags_on_device,
                        int max_level, int* n_refined);
/* refine_by_criterion(mesh, max_level, want) (harness.hpp:295-321) with `want` evaluated on
 * the device at every cell centre of every leaf below max_level:
 *   kind 0  |f(x)| < p0 * b.dx, f the level set (lsf, n_lsf as in pmg_b200_build_stencils)
 *   kind 1  b.dx > p0 * max(1, ||x - centre|| / p1)   (harness.hpp:351-355, sphere_refined)
 *   kind 2  b.dx > p0 && ||x - centre|| < p1          (harness.hpp:413-418, two_electrodes) */
int pmg_b200_tree_refine_by_criterion(pmg_b200_tree* tree, int kind, const pmg_lsf_t* lsf, int n_lsf,
                                      double p0, double p1, const double* centre, int max_level);
/* the Block table (mesh.hpp:37-55) in the layout of pmg_b200_set_mesh; NULL outputs are skipped */
int pmg_b200_tree_get(pmg_b200_tree* tree, int32_t* level, int32_t* coords, double* origin, double* dx,
                      int32_t* parent, int32_t* children, int32_t* nbr, int32_t* cnbr);
/* TreeMesh::level_blocks(level) (mesh.hpp:102-105): ids sorted by coords */
int pmg_b200_tree_level_blocks(pmg_b200_tree* tree, int level, int32_t* ids, int* n);
/* device pointers of the table: level, coords, origin, dx, parent, children, nbr, cnbr */
int pmg_b200_tree_device_arrays(pmg_b200_tree* tree, const void** out8);
/* pmg_b200_set_mesh from the device tree */
int pmg_b200_set_mesh_from_tree(pmg_b200_ctx* ctx, pmg_b200_tree* tree);

#ifdef __cplusplus
}
#endif

#endif /* PMG_B200_H */
