/*
 * dpvslam_b200.h — C-ABI of the B200-native DPV-SLAM hot path.
 *
 * The drop-in boundary: plain pointers, sizes and an opaque problem handle;
 * no torch or C++ types cross it.  Every entry point returns an int status
 * (DPV_OK / DPV_SINGULAR / DPV_BAD_ARGS / DPV_CUDA_ERROR) and never throws.
 * Device pointers are CUDA global-memory addresses; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  All work is
 * enqueued on `stream`; functions that return host scalars synchronise it.
 *
 * Each entry point names the reference interface it replaces
 * (paths under /root/reference/pkg/src/patchslam).  The Python host mirror
 * (paper_2408_01654_b200/) binds them with ctypes exactly as a maintainer
 * would bind them from the reference.
 *
 * Layouts (row-major, float64 unless noted):
 *   quaternion (x, y, z, w); pose = world-from-camera, x_w = R x_c + t;
 *   tangent (rho, phi) = (translation, rotation); m = p*p patch cells,
 *   cell order row-major x-fastest (geometry.py:398-407).
 */
#ifndef DPVSLAM_B200_H
#define DPVSLAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPV_OK 0
#define DPV_SINGULAR 1   /* maps to patchslam.errors.SingularSystem (errors.py:28-29) */
#define DPV_BAD_ARGS 2   /* maps to ValueError (ba.py:63-66) */
#define DPV_CUDA_ERROR 3

#define DPV_ABI_VERSION 1

/* Library identity / diagnostics. */
int32_t dpv_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char* dpv_last_error(void);
/* Device properties (SM count, cc) probed on the current device. */
int32_t dpv_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);
/* Number of kernels this library has launched in the process (monotone counter). */
int64_t dpv_launch_count(void);

/* Per-kernel CUDA-event timing (used by bench.py for the roofline numbers):
 * enable, run, then collect = synchronise + aggregate per kernel name
 * ('\n'-separated names, summed ms, launch counts) and reset. */
int32_t dpv_timing_enable(int32_t on);
int32_t dpv_timing_collect(char* names, int64_t names_cap, double* total_ms, int64_t* counts,
                           int32_t cap, int32_t* n_out);

/* ------------------------------------------------------------------------
 * Geometry (K2 standalone).
 * ---------------------------------------------------------------------- */

/* geometry.quat_to_matrix (geometry.py:70-86): q (n,4) -> R (n,3,3). */
int32_t dpv_quat_to_matrix(const double* q, int64_t n, double* rot, void* stream);

/* geometry.reproject_grid (geometry.py:478-529).
 *   rays (E,m,3), inv_depth (E), rot_i/rot_j (E,3,3), t_i/t_j (E,3), intr = (fx,fy,cx,cy)
 *   -> pix (E,m,2), valid (E,m) uint8; if j_pose != NULL also
 *      j_pose (E,m,2,6) (source-pose tangent; target = negation) and j_depth (E,m,2). */
int32_t dpv_reproject_grid(const double* rays, const double* inv_depth,
                           const double* rot_i, const double* t_i,
                           const double* rot_j, const double* t_j,
                           const double* intr4, int64_t n_edges, int32_t cells,
                           double* pix, uint8_t* valid, double* j_pose, double* j_depth,
                           void* stream);

/* ------------------------------------------------------------------------
 * Bundle-adjustment problem (ba.BAProblem + _structure + _assembly_maps).
 * ---------------------------------------------------------------------- */

/* Device view of the patch graph (graph.PatchGraph, graph.py:82-136) in SoA form. */
typedef struct dpv_graph {
    int32_t n_frames;
    int32_t cells;              /* p*p (9 for the reference default p=3)            */
    int64_t n_patches;          /* total patches over all frames                   */
    int64_t n_edges;
    const double* patch_grid;   /* (n_patches, cells, 2) pixel grids                */
    const int32_t* edge_src;    /* (n_edges) source frame                          */
    const int32_t* edge_gpatch; /* (n_edges) global patch id = offset[src] + patch */
    const int32_t* edge_dst;    /* (n_edges) target frame                          */
    const double* edge_target;  /* (n_edges, cells, 2) flow targets                */
    const double* edge_conf;    /* (n_edges, 2) confidences                        */
    double intr[4];             /* fx, fy, cx, cy                                  */
} dpv_graph;

typedef struct dpv_problem dpv_problem;

typedef struct dpv_problem_info {
    int64_t n_edges;      /* E: problem edges                                 */
    int64_t n_depths;     /* P: free inverse depths (depth_keys)              */
    int64_t n_free;       /* n: free poses                                    */
    int64_t n_keys;       /* W: union_keys (pose-pair blocks)                 */
    int64_t n_inc;        /* I: (pose var, depth row) incidences              */
    int64_t n_pairs;      /* Schur incidence pairs                            */
    int64_t n_segments;   /* edge segments (src,dst) chunks                   */
    int64_t n_touched;    /* touched fixed frames                             */
    int32_t first_free, last_free;
    int32_t scale_degenerate;
    int32_t touched_fixed0; /* first touched fixed frame or -1                */
    int64_t device_bytes;   /* bytes the handle holds on the device           */
} dpv_problem_info;

/* BAProblem(graph, (first, last), edge_indices) (ba.py:60-98) plus the
 * state-independent structure and normal-equation index (ba.py:124-216).
 * edge_indices: device int64 array or NULL (select edges touching the range,
 * ba.py:72-77).  Copies what it needs; the graph view may be freed after. */
int32_t dpv_problem_create(const dpv_graph* graph, int32_t first_free, int32_t last_free,
                           const int64_t* edge_indices, int64_t n_edge_indices,
                           void* stream, dpv_problem** out);
/* Same, for one shard of an edge-partitioned global BA: extra_keys (device
 * int64, folded a*n+b) are merged into the shard's block pattern so every
 * shard's pose/Schur blocks line up with the global union_keys (the
 * all-reduce of SURVEY 8(e)). */
int32_t dpv_problem_create_ex(const dpv_graph* graph, int32_t first_free, int32_t last_free,
                              const int64_t* edge_indices, int64_t n_edge_indices,
                              const int64_t* extra_keys, int64_t n_extra_keys, void* stream,
                              dpv_problem** out);
/* Override the gauge (scale_degenerate, first touched fixed frame) with the
 * global problem's values (a shard sees only part of the touched frames). */
int32_t dpv_problem_set_gauge(dpv_problem* prob, int32_t scale_degenerate,
                              int32_t touched_fixed0);
int32_t dpv_problem_destroy(dpv_problem* prob);
/* Factor plan of the reduced-system Cholesky (after the first dense solve):
 * dense flag, 64-row tiles, planned trailing-update tiles and their flops. */
int32_t dpv_problem_plan_info(const dpv_problem* prob, int32_t* dense, int64_t* tiles,
                              int64_t* update_tiles, double* update_flops);
/* Sparse band+border factor plan of the reduced camera system (spd.cu):
 * v9 = [n, chains, band tiles, tile bandwidth, border poses, border rows,
 *       level-2 tiles, factor CTAs, modelled us]. */
int32_t dpv_problem_spd_info(const dpv_problem* prob, int64_t* v9);
int32_t dpv_problem_get_info(const dpv_problem* prob, dpv_problem_info* info);

/* Device pointer + element count + dtype code (0=f64, 1=i32, 2=i64, 3=u8) of a
 * named internal array (index arrays, assembled system, per-edge terms); see
 * DESIGN.md for the name list.  For parity tests and zero-copy host mirrors. */
int32_t dpv_problem_array(const dpv_problem* prob, const char* name,
                          void** ptr, int64_t* count, int32_t* dtype);

/* BAProblem.state depth gather (ba.py:110-115): d[r] = patch_depth[depth_patch[r]]. */
int32_t dpv_gather_depths(const dpv_problem* prob, const double* patch_depth, double* d,
                          void* stream);
/* BAProblem.write_back depth scatter (ba.py:117-122). */
int32_t dpv_scatter_depths(const dpv_problem* prob, const double* d, double* patch_depth,
                           void* stream);
/* active_patch_count (ba.py:143-145, graph.py:232-241); host int result. */
int32_t dpv_active_patch_count(dpv_problem* prob, double gate, int64_t* count, void* stream);

/* ------------------------------------------------------------------------
 * Hot path.  q (F,4), t (F,3) over ALL graph frames, d (P) over depth rows.
 * ---------------------------------------------------------------------- */

/* ba.residuals (ba.py:219-245): res (E,m,2), valid (E,m) in problem-edge order. */
int32_t dpv_residuals(dpv_problem* prob, const double* q, const double* t, const double* d,
                      double* res, uint8_t* valid, void* stream);
/* ba.objective (ba.py:248-253): deterministic sum written to out_dev[0] (device). */
int32_t dpv_objective(dpv_problem* prob, const double* q, const double* t, const double* d,
                      double* out_dev, void* stream);
/* ba.assemble (ba.py:328-440): fused reprojection + whitened Gram + segmented
 * reductions + Schur elimination into the handle's system arrays. */
int32_t dpv_assemble(dpv_problem* prob, const double* q, const double* t, const double* d,
                     void* stream);
/* dpv_assemble in two halves (the native LM's speculative assembly):
 * the per-edge pass at (q, t, d) - K2+K3 terms and per-segment sums, plus the
 * objective at that state into objective_out (DEVICE f64, may be NULL) - and
 * the rest (depth rows, incidences, Schur blocks, rhs, gauge pin) from the
 * last edge pass.  dpv_assemble == dpv_assemble_edges + dpv_assemble_rest. */
int32_t dpv_assemble_edges(dpv_problem* prob, const double* q, const double* t, const double* d,
                           double* objective_out, void* stream);
int32_t dpv_assemble_rest(dpv_problem* prob, const double* t, void* stream);
/* BlockSparseSystem.reduced_system(lam) (ba.py:303-319). Any output may be NULL. */
int32_t dpv_reduced_system(dpv_problem* prob, double lam, double* blocks, double* rhs,
                           double* cinv, void* stream);
/* solve_dense / solve_block_sparse numerics (ba.py:451-487): S(lam) dense
 * Cholesky on FP64 tensor cores + back-substitution (ba.py:321-325).
 * dp (n,6), dd (P).  *status_dev (device int32) = 0 ok / 1 not positive definite. */
int32_t dpv_solve(dpv_problem* prob, double lam, double* dp, double* dd, int32_t* status_dev,
                  void* stream);
/* The same solve with an explicit backend (ba.py:490 _BACKENDS): 0 = auto
 * (the fastest: single-CTA dense solve for 6n <= 162, else the banded +
 * border sparse factorisation), 1 = dense (solve_dense, ba.py:451-472: S in
 * a dense matrix, every-tile Cholesky on the FP64 tensor cores), 2 = block
 * sparse (solve_block_sparse, ba.py:475-487: the spd.cu factorisation at
 * every size). */
int32_t dpv_solve_backend(dpv_problem* p, double lam, int32_t backend, double* dp, double* dd,
                          int32_t* status_dev, void* stream);
/* K2 pixels of every problem edge times `scale` (problem order, (E,m,2)):
 * the reprojected coordinates P' that feed the correlation lookup (pass 0.25
 * for 1/4-resolution feature maps).  Same arithmetic as reproject_grid. */
int32_t dpv_reproject_coords(dpv_problem* prob, const double* q, const double* t,
                             const double* d, double scale, double* coords, void* stream);
/* K2 pixels (scaled) of a selection of problem edges (DEVICE int64 problem
 * edge indices) -> coords_out (n_sel, p*p, 2) in selection order: the
 * correlation edges' coordinates without reprojecting every BA edge. */
int32_t dpv_reproject_coords_sel(dpv_problem* prob, const double* q, const double* t,
                                 const double* d, double scale, const int64_t* sel,
                                 int64_t n_sel, double* coords_out, void* stream);
/* Replace the flow targets (E,m,2) and confidences (E,2) (problem order, conf
 * may be NULL) without rebuilding the index: the per-iteration update-operator
 * output of DPVO or a re-run flow oracle. */
int32_t dpv_update_targets(dpv_problem* prob, const double* target, const double* conf,
                           void* stream);
/* BlockSparseSystem.back_substitute(dp, lam) (ba.py:321-325): dd (P). */
int32_t dpv_back_substitute(dpv_problem* prob, double lam, const double* dp, double* dd,
                            void* stream);
/* ba._apply_step (ba.py:521-531). */
int32_t dpv_apply_step(dpv_problem* prob, const double* q, const double* t, const double* d,
                       const double* dp, const double* dd, double* q2, double* t2, double* d2,
                       void* stream);

typedef struct dpv_lm_params {
    int32_t max_iterations;   /* ba.solve max_iterations */
    double tolerance;         /* ba.solve tolerance      */
    double lambda0;           /* problem.damping         */
} dpv_lm_params;

typedef struct dpv_lm_report {  /* ba.BAReport (ba.py:497-518) */
    int32_t iterations;
    int32_t converged;
    double initial_objective;
    double final_objective;
    double gradient_norm;
    int64_t unconstrained_depths;
    double final_damping;
    double step_norm;
    int32_t n_attempts;       /* total lambda attempts (solves) */
    int32_t times_len;
    double iteration_times[64];
} dpv_lm_report;

/* ba.solve LM driver (ba.py:534-605) run natively; q/t/d (device) updated in
 * place with the accepted state.  Returns DPV_SINGULAR when the reference
 * would raise SingularSystem. */
int32_t dpv_lm_solve(dpv_problem* prob, double* q, double* t, double* d,
                     const dpv_lm_params* params, dpv_lm_report* report, void* stream);

/* Batched replicas: `count` independent problems,
 * each on its own stream, driven concurrently by up to `threads` host workers
 * (<= 0: one per hardware thread).  Element i of every array belongs to
 * problem i; status[i] is that problem's own return code (a singular problem
 * does not stop the others).  Returns DPV_OK, or the first failing problem's
 * code with dpv_last_error() naming it.  No reference counterpart: the
 * reference solves one problem per ba.solve call (ba.py:534-605), and these
 * are exactly `count` such calls. */
int32_t dpv_problem_create_batch(int32_t count, const dpv_graph* graphs,
                                 const int32_t* first_free, const int32_t* last_free,
                                 void* const* streams, int32_t threads, dpv_problem** out,
                                 int32_t* status);
int32_t dpv_lm_solve_batch(int32_t count, dpv_problem* const* probs, double* const* q,
                           double* const* t, double* const* d, const dpv_lm_params* params,
                           dpv_lm_report* reports, void* const* streams, int32_t threads,
                           int32_t* status);

/* Block-sparse SPD solve (the block-sparse backend, block_cholesky.py:48-111
 * + BlockCholeskyFactor.solve 31-45): keys (n_keys, 2) HOST int64 upper
 * pattern a <= b of 6x6 blocks; blocks (n_keys, 6, 6) and rhs (6n) DEVICE
 * f64; x (6n) DEVICE out.  Banded + border plan, one dataflow factor kernel
 * (spd.cu).  status_dev[0] = 1 if not positive definite (SingularSystem). */
int32_t dpv_block_sparse_solve(const int64_t* keys, int64_t n_keys, int64_t n,
                               const double* blocks, const double* rhs, double* x,
                               int32_t* status_dev, void* stream);
/* ------------------------------------------------------------------------
 * Dense SPD solve (the K4c engine, usable standalone).
 * A: (N,N) row-major, lower triangle read, overwritten by L; b (N) -> x.
 * ---------------------------------------------------------------------- */
int32_t dpv_cholesky_solve(double* a, double* b, int64_t n, int32_t* status_dev, void* stream);

/* block_cholesky symbolic fill (block_cholesky.py:48-111): number of
 * diagonal + strictly-lower blocks of the natural-order factor of the
 * upper-triangle block pattern keys (w,2) (host int64).  Host-only. */
int32_t dpv_block_fill_count(const int64_t* keys, int64_t n_keys, int64_t n, int64_t* count);

/* ------------------------------------------------------------------------
 * Synthetic inputs on the device.
 * dpv_fill_flow: the flow oracle fill_flow (synthetic.py:222-287) for the
 * n edges sel (DEVICE int64, NULL = edges 0..n-1): ground-truth reprojection
 * of each source patch grid (rot (F,9) row-major / trans (F,3) ground-truth
 * poses, landmarks (L,3), patch_landmark (n_patches) int64), plus the host
 * generator's draws shift (n,2), outlier (n) uint8, gross (n,2); writes
 * target (n, cells, 2) and conf (n, 2).  Bit-identical to the reference's
 * numpy expressions.  All arrays DEVICE.
 * dpv_reproject_exact: initial targets = reprojection at the current state
 * (graph.py:152-164) with patch inverse depths patch_depth (n_patches). */
int32_t dpv_fill_flow(const dpv_graph* g, const double* rot, const double* trans,
                      const double* landmarks, const int64_t* patch_landmark, const int64_t* sel,
                      int64_t n, const double* shift, const uint8_t* outlier, const double* gross,
                      double low_confidence, double width, double height, double* target,
                      double* conf, void* stream);
int32_t dpv_reproject_exact(const dpv_graph* g, const double* rot, const double* trans,
                            const double* patch_depth, const int64_t* sel, int64_t n, double* pix,
                            void* stream);
/* visible_landmarks (synthetic.py:68-79) of every frame: inverse ground-truth
 * poses inv_q (F,4) / inv_t (F,3), landmarks (L,3), intr HOST [fx fy cx cy];
 * flags (F, L) uint8 = in front (z > 0.5) and inside the image by `margin`
 * (u in [margin, u_max], v in [margin, v_max]).  Bit-identical tests. */
int32_t dpv_visible_landmarks(int64_t n_frames, int64_t n_landmarks, const double* inv_q,
                              const double* inv_t, const double* landmarks, const double* intr,
                              double margin, double u_max, double v_max, uint8_t* flags,
                              void* stream);

/* ------------------------------------------------------------------------
 * Sim(3) pose-graph optimisation (posegraph.py:121-196, optimize; SURVEY
 * 8(f) rank 4).  Similarities as 8 doubles [tx ty tz qx qy qz qw s]
 * (x -> s R x + t; the g2o field order, posegraph.py:12-14).  Constraint c:
 * nodes (a_c, b_c) and constant M_c, residual r = log(M S_a^-1 S_b) in the
 * tangent (rho, phi, sigma) (posegraph.py:91-104).
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t iterations;
    int32_t converged;
    double initial_objective;
    double final_objective;
    double max_residual_norm;    /* of the last linearisation */
    double final_damping;
} dpv_pgo_report;

/* optimize(): Levenberg-Marquardt over node tangents, node 0 the gauge.
 * nodes (n_nodes, 8) DEVICE, overwritten by the solution; ca_h / cb_h HOST
 * and ca / cb DEVICE copies of the constraint node indices (int32, the host
 * copy builds the block pattern); cm (n_cons, 8) DEVICE.  DPV_SINGULAR when
 * the damped normal equations stay singular (SingularSystem). */
int32_t dpv_pgo_optimize(int64_t n_nodes, double* nodes, int64_t n_cons, const int32_t* ca_h,
                         const int32_t* cb_h, const int32_t* ca, const int32_t* cb,
                         const double* cm, int32_t max_iterations, double tolerance,
                         double damping, dpv_pgo_report* report, void* stream);
/* residual_and_jacobian / objective (posegraph.py:91-104): r (n_cons, 7),
 * J (n_cons, 7, 7) d r / d (left tangent of S_b) or NULL, objective (device
 * scalar, sum r.r) or NULL.  All DEVICE. */
int32_t dpv_pgo_linearize(int64_t n_nodes, const double* nodes, int64_t n_cons,
                          const int32_t* ca, const int32_t* cb, const double* cm, double* r,
                          double* J, double* objective, void* stream);
/* sim3_exp / sim3_log (geometry.py:303-321), n items, DEVICE arrays. */
int32_t dpv_sim3_exp(int64_t n, const double* tangents, double* sims, void* stream);
int32_t dpv_sim3_log(int64_t n, const double* sims, double* tangents, void* stream);

/* ------------------------------------------------------------------------
 * K1: per-edge correlation lookup (Eq. 4; no reference code).
 *   gmap  (n_src_patches, p*p, C)       patch features, channels-last
 *   fmap_l (n_frames, H_l, W_l, C)      level-l frame features, channels-last
 *                                       (level 1 = dpv_avg_pool4 of level 0)
 *   coords (E, p*p, 2) level-0 coordinates (feature resolution); level 1 uses /4
 *   ii (E) patch index into gmap, jj (E) frame index into fmaps
 *   out (E, L, p*p, 2r+1, 2r+1) float32.  dtype: 0 = float32 features, 1 = bf16.
 *   p = 3, C % 4 == 0, r <= 3.  OOB taps contribute 0 (bilinear, zero padding).
 * ---------------------------------------------------------------------- */
int32_t dpv_corr(const void* gmap, const void* fmap0, const void* fmap1,
                 const double* coords, const int32_t* ii, const int32_t* jj,
                 int64_t n_edges, int32_t channels, int32_t h0, int32_t w0,
                 int32_t h1, int32_t w1, int32_t n_levels, int32_t radius,
                 int32_t dtype, float* out, void* stream);

/* Same, with the sizes of gmap (n_patches) and the fmaps (n_frames): bf16
 * features with r = 3 and C in {64, 128, 256} take the TMA + tensor-core
 * kernel (corr_tma.cu; 10x10 tap windows, hardware zero fill outside the
 * image), everything else the corr.cu kernels. */
int32_t dpv_corr_ex(const void* gmap, int64_t n_patches, const void* fmap0, const void* fmap1,
                    int64_t n_frames, const double* coords, const int32_t* ii, const int32_t* jj,
                    int64_t n_edges, int32_t channels, int32_t h0, int32_t w0, int32_t h1,
                    int32_t w1, int32_t n_levels, int32_t radius, int32_t dtype, float* out,
                    void* stream);

/* dpv_corr_ex with a CTA work size: items_per_cta = 0 runs one persistent
 * CTA per SM (fastest alone); > 0 cuts each SM's share of (edge, level)
 * items into CTAs of that many items, so when the lookup runs on a
 * low-priority stream beside a higher-priority one (the correlation beside
 * the BA solve) the scheduler hands SMs back at CTA granularity and the
 * lookup fills the SMs the latency-bound solve leaves idle.  Same results. */
int32_t dpv_corr_ex2(const void* gmap, int64_t n_patches, const void* fmap0, const void* fmap1,
                     int64_t n_frames, const double* coords, const int32_t* ii, const int32_t* jj,
                     int64_t n_edges, int32_t channels, int32_t h0, int32_t w0, int32_t h1,
                     int32_t w1, int32_t n_levels, int32_t radius, int32_t dtype,
                     int64_t items_per_cta, float* out, void* stream);

/* Proximity loop-closure candidates (loop.py:64-85): centers (n_frames, 3)
 * DEVICE f64 camera centres; pairs (capacity, 2) DEVICE int64 (old, recent),
 * sorted by centre distance (ties: recent, then old ascending) exactly as the
 * reference; *count (HOST) = number of pairs.  Pass pairs = NULL to query
 * the count only.  Candidates: recent - old >= min_gap, distance < threshold. */
int32_t dpv_proximity_detect(const double* centers, int64_t n_frames, int64_t min_gap,
                             double threshold, int64_t* pairs, int64_t capacity, int64_t* count,
                             void* stream);

/* Level-1 pyramid: 4x4 average pool of channels-last fmap (F,H,W,C) -> (F,H/4,W/4,C). */
int32_t dpv_avg_pool4(const void* fmap, int64_t n_frames, int32_t h, int32_t w, int32_t channels,
                      int32_t dtype, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
