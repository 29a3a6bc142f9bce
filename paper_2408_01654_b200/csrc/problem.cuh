// Device-resident BA problem: state-independent index (ba.py:60-216) and the
// assembled system arrays (ba.py:272-440).  One handle per BAProblem.
#pragma once

#include <thread>
#include <vector>

#include "common.cuh"

namespace dpv {
// Which 64x64 tiles the Cholesky touches (dense or symbolic tile fill); see cholesky.cu.
struct FactorPlan {
    int64_t N = -1;
    int T = 0;                        // 64-row tiles over [0, N); tile T = the rhs row N
    int ng = 0;                       // panel groups (2 panels each)
    bool dense = true;
    int* d_rows = nullptr;            // trsm row tiles, per panel
    std::vector<int> rows_off;        // T + 1
    int* d_rows_off = nullptr;        // device copy of rows_off
    int2* d_pairs = nullptr;          // syrk (row tile, col tile), per group: intra|next|rest
    std::vector<int> intra_off, next_off, rest_off, rest_end;
    int64_t pair_count = 0;
    double syrk_flops = 0.0;          // algorithmic flops of the planned updates
    ~FactorPlan() {
        if (d_rows) cudaFree(d_rows);
        if (d_rows_off) cudaFree(d_rows_off);
        if (d_pairs) cudaFree(d_pairs);
    }
};
int32_t build_factor_plan(int64_t N, const std::vector<char>* tile_pattern, FactorPlan& pl);

// Banded + border sparse SPD solver of the reduced camera system (spd.cu).
struct SpdPlan;
int32_t spd_plan_build(const int32_t* ka, const int32_t* kb, int64_t W, int64_t n, SpdPlan** out,
                       cudaStream_t st);
void spd_plan_free(SpdPlan* p);
void spd_plan_set_stream(SpdPlan* p, cudaStream_t st);
int64_t spd_plan_bytes(const SpdPlan* p);
void spd_plan_describe(const SpdPlan* p, int64_t* v);
double spd_plan_flops(const SpdPlan* p);
// S(lam) from the assembled system instead of precomputed blocks / rhs: the
// scatter into the solver's storage forms each entry itself (no separate
// reduced-system pass)
struct SpdSysInput {
    const double* pose = nullptr;       // (W, 36) pose blocks
    const double* schur = nullptr;      // (W, 36) Schur blocks
    const double* rhs_pose = nullptr;   // (n, 6)
    const double* rhs_schur = nullptr;  // (n, 6)
    const double* scal = nullptr;       // gauge pin (scal[1] flag, scal[2..4] u)
    double lam = 0.0;
};
int32_t spd_factor_solve(SpdPlan* pl, const int32_t* ka, const int32_t* kb, const double* blocks,
                         const double* rhs, double* dp, int32_t* status, cudaStream_t st,
                         const SpdSysInput* sys = nullptr);

// S(lam) block value at entry (i, j) of key w (ba.py:305-309)
__device__ __forceinline__ double reduced_entry(const double* pose, const double* schur,
                                                int64_t w, int idx, bool diag, double lam) {
    double v = pose[w * 36 + idx] - schur[w * 36 + idx] / (1.0 + lam);
    if (diag && (idx / 6 == idx % 6)) v += lam * pose[w * 36 + idx];
    return v;
}
// ... plus the scale-gauge pin on the first free pose's block (ba.py:311-319)
__device__ __forceinline__ double reduced_pinned_entry(const double* pose, const double* schur,
                                                       const int32_t* ka, int64_t w, int idx,
                                                       bool diag, double lam, const double* scal) {
    double v = reduced_entry(pose, schur, w, idx, diag, lam);
    if (w == 0 && scal[1] != 0.0 && diag && ka[0] == 0) {
        const int i = idx / 6, j = idx % 6;
        if (i < 3 && j < 3) {
            double mx = 0.0;
            for (int k = 0; k < 6; ++k)
                mx = fmax(mx, fabs(reduced_entry(pose, schur, 0, k * 7, true, lam)));
            const double mu = 1e6 * fmax(1.0, mx);
            v += mu * scal[2 + i] * scal[2 + j];
        }
    }
    return v;
}
}  // namespace dpv

namespace dpv {
// 16-double pinned host slots from a process-wide pool: cudaMallocHost /
// cudaFreeHost cost milliseconds and cudaFreeHost synchronises the device,
// which would serialise concurrently built / destroyed problems
double* pinned_slot_get();
void pinned_slot_put(double* p);
}  // namespace dpv

struct dpv_problem {
    // ---- sizes -------------------------------------------------------------
    int32_t F = 0;      // graph frames
    int32_t m = 9;      // cells per patch
    int64_t E = 0;      // problem edges
    int64_t P = 0;      // depth rows
    int64_t n = 0;      // free poses
    int64_t W = 0;      // union keys
    int64_t I = 0;      // incidences
    int64_t NP = 0;     // Schur pairs
    int64_t S = 0;      // edge segments
    int64_t NC = 0;     // incidence contributions
    int64_t T = 0;      // touched fixed frames
    int64_t KS = 0;     // key->segment entries
    int64_t VS = 0;     // var->segment entries
    int32_t first = 0, last = 0;
    int32_t scale_degenerate = 0;
    int32_t touched0 = -1;
    double intr[4] = {0, 0, 0, 0};

    // ---- problem-order arrays ---------------------------------------------
    int64_t* edge_idx = nullptr;   // (E) graph edge index
    int32_t* p_row = nullptr;      // (E) depth row
    int32_t* p_pos = nullptr;      // (E) assembly position
    int32_t* p_vi = nullptr;       // (E) var of src or -1
    int32_t* p_vj = nullptr;       // (E) var of dst or -1
    double* p_conf_max = nullptr;  // (E) max confidence (active_patch_count)

    // ---- assembly-order (segment-sorted) SoA arrays -----------------------
    int32_t* a_src = nullptr;      // (E)
    int32_t* a_dst = nullptr;      // (E)
    int32_t* a_row = nullptr;      // (E)
    int32_t* a_pidx = nullptr;     // (E) problem index
    double* a_tgt = nullptr;       // (2m, E)
    double* a_w = nullptr;         // (2, E)

    // ---- depth rows ---------------------------------------------------------
    int32_t* depth_patch = nullptr;  // (P) global patch id, sorted
    double* r_ray = nullptr;         // (2m, P) ray x,y per cell (z = 1)
    int32_t* row_ptr = nullptr;      // (P+1) CSR over assembly positions
    int32_t* row_pos = nullptr;      // (E)

    // ---- segments (same (src,dst), <= kSegMax edges) ------------------------
    int32_t* seg_ptr = nullptr;    // (S+1)
    int32_t* seg_src = nullptr;    // (S)
    int32_t* seg_dst = nullptr;    // (S)

    // ---- incidences ---------------------------------------------------------
    int32_t* inc_var = nullptr;    // (I)  sorted by (var, row) (np.unique order)
    int32_t* inc_row = nullptr;    // (I)
    int32_t* inc_ptr = nullptr;    // (I+1) CSR over contributions
    int32_t* inc_con = nullptr;    // (NC) assembly position * 2 + (negative)
    int32_t* p_inc_inv = nullptr;  // (NC) reference inc_inv (contribution -> incidence)
    int32_t* var_inc_ptr = nullptr;  // (n+1) incidence range per var
    int32_t* rinc_ptr = nullptr;   // (P+1) incidences per row (ascending var)
    int32_t* rinc = nullptr;       // (I)

    // ---- pose-pair keys -------------------------------------------------------
    int64_t* union_keys = nullptr; // (W) a*n+b, a<=b
    int64_t* key_pair_ptr = nullptr;  // (W+1)
    int32_t* pair_l = nullptr;     // (NP) incidence index (left)
    int32_t* pair_r = nullptr;     // (NP) incidence index (right)
    int64_t NR = 0;                // pair runs
    int32_t* key_run_ptr = nullptr;   // (W+1) runs per key
    int32_t* run_l = nullptr;      // (NR) first left incidence of the run
    int32_t* run_r = nullptr;      // (NR) first right incidence
    int32_t* run_len = nullptr;    // (NR) pairs in the run
    // grouped Schur: rows with identical incidence-var lists, SYRK per chunk
    int32_t grouped = 0;
    int32_t* g_rows = nullptr;     // (P) rows sorted by group
    int4* g_chunks = nullptr;      // (n_chunks) {first sorted row, rows, vars m, block offset}
    int64_t n_chunks = 0;
    int64_t n_gblocks = 0;
    double* g_sbuf = nullptr;      // (n_gblocks, 36) chunk Schur blocks
    int32_t* key_blk_ptr = nullptr;   // (W+1)
    int32_t* key_blk = nullptr;    // (n_gblocks) chunk blocks of each key, chunk order
    int32_t* key_seg_ptr = nullptr;   // (W+1)
    int32_t* key_seg = nullptr;    // (KS) seg*2 + (negative)
    int32_t* var_seg_ptr = nullptr;   // (n+1)
    int32_t* var_seg = nullptr;    // (VS) seg*2 + (negative)
    int32_t* key_a = nullptr;      // (W) block row var
    int32_t* key_b = nullptr;      // (W) block col var
    int32_t* touched = nullptr;    // (T)

    // ---- assembled system -----------------------------------------------------
    double* frame_R = nullptr;     // (F, 9)
    double* e_terms = nullptr;     // [e_pd (E, 6) | (c_dd, g_d) (E, 2)]
    double* seg_h = nullptr;       // (S, 21) upper-triangular sum of J^T W J
    double* seg_g = nullptr;       // (S, 6)  sum of J^T W r
    double* seg_obj = nullptr;     // (S) sum of w r^2 (LM candidate objective)
    double* depth_diag = nullptr;  // (P)
    double* rhs_depth = nullptr;   // (P)
    uint8_t* active = nullptr;     // (P)
    double* cinv0 = nullptr;       // (P)
    double* inc_block = nullptr;   // (I, 6)
    double* uinc = nullptr;        // (I, 6) inc_block * cinv0[row]
    double* sysbuf = nullptr;      // one allocation: the four arrays below + red_tail
    double* red_tail = nullptr;    // (kRedTail) per-rank depth-gradient slots
    double* pose_blocks = nullptr; // (W, 36)
    double* schur_blocks = nullptr;// (W, 36)
    double* rhs_pose = nullptr;    // (n, 6)
    double* rhs_schur = nullptr;   // (n, 6)
    double* scal = nullptr;        // [0]=grad bits, [1]=pin flag, [2..4]=pin u, [5]=objective,
                                   // [6]=unconstrained count, [7]=depth-only grad bits
    double* obj_part = nullptr;    // (kObjBlocks)
    int64_t* count_buf = nullptr;  // (2) scratch counters

    // ---- solve workspace -----------------------------------------------------
    double* red_rhs = nullptr;     // (N)
    double* cinv = nullptr;        // (P)
    double* dense = nullptr;       // (N+1) x ld lower, lazily allocated
    int64_t dense_ld = 0;
    double* bsub_part = nullptr;   // back-substitution partials + diag inverses
    dpv::FactorPlan* plan = nullptr;  // tile plan of the reduced system (lazily built)
    int32_t* perm_pos = nullptr;   // (n) pose var -> permuted position in the dense solve
    dpv::SpdPlan* spd = nullptr;   // sparse band+border solver plan (lazily built)
    int32_t spd_failed = 0;        // plan impossible -> tile-plan factorisation
    // explicit backend of the next solve (dpv_solve_backend): 0 = auto (small
    // dense solve for 6n <= kSmallMax, else the sparse factorisation),
    // 1 = dense (ba.solve_dense: full dense Cholesky of S), 2 = block sparse
    int32_t solve_backend = 0;
    dpv::FactorPlan* dplan = nullptr;   // every-tile plan of the dense backend
    int32_t* ident_pos = nullptr;       // (n) identity pose order for it
    // the plan is host work (~1 ms at cfg3): built on a host thread started
    // by the index build, joined by the first sparse solve
    std::thread plan_thread;
    dpv::SpdPlan* spd_pending = nullptr;
    int32_t plan_status = 0;
    int32_t* status = nullptr;     // (4) device flags

    // ---- LM scratch ------------------------------------------------------------
    double* lm_q = nullptr; double* lm_t = nullptr; double* lm_d = nullptr;
    double* lm_dp = nullptr; double* lm_dd = nullptr;
    double* lm_wq = nullptr; double* lm_wt = nullptr; double* lm_wd = nullptr;
    uint8_t* row_flag = nullptr;   // (P) scratch for active_patch_count
    double* lm_host = nullptr;     // pinned host scalars

    std::vector<void*> allocs;     // everything above, freed by destroy
    int64_t bytes = 0;
    cudaStream_t alloc_stream = nullptr;   // stream-ordered pool allocations

    template <typename T>
    int32_t alloc(T** p, int64_t count) {
        size_t b = sizeof(T) * (size_t)(count > 0 ? count : 1);
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, b, alloc_stream);
        if (e != cudaSuccess) {
            dpv::set_error(std::string("cudaMalloc ") + std::to_string(b) + ": " +
                           cudaGetErrorString(e));
            return DPV_CUDA_ERROR;
        }
        allocs.push_back(q);
        bytes += (int64_t)b;
        *p = reinterpret_cast<T*>(q);
        return DPV_OK;
    }
    ~dpv_problem() {
        if (plan_thread.joinable()) plan_thread.join();
        dpv::spd_plan_free(spd_pending);
        // returned to the device pool (release threshold raised: see
        // dpv::configure_pool), so the next problem reuses the memory
        for (void* p : allocs) cudaFreeAsync(p, alloc_stream);
        if (lm_host) dpv::pinned_slot_put(lm_host);
        delete plan;
        delete dplan;
        dpv::spd_plan_free(spd);
    }
};

namespace dpv {
constexpr int kSegMax = 128;      // edges per segment chunk
constexpr int kRedTail = 64;      // ranks whose depth gradient rides in the packed all-reduce
constexpr int kSyrkMaxRows = 128;            // rows per grouped-Schur chunk
constexpr int kSyrkSmemDoubles = 12800;      // 100 KB of W_g staging per chunk (2 CTAs/SM)
int32_t configure_pool();
constexpr int kObjBlocks = 1184;  // 148 SMs x 8
int32_t build_problem(const dpv_graph* g, int32_t first, int32_t last, const int64_t* eidx,
                      int64_t n_eidx, const int64_t* extra_keys, int64_t n_extra,
                      cudaStream_t st, dpv_problem* P);
int32_t frame_rotations(dpv_problem* p, const double* q, cudaStream_t st);
int32_t objective(dpv_problem* p, const double* q, const double* t, const double* d,
                  double* out, cudaStream_t st);
int32_t residuals(dpv_problem* p, const double* q, const double* t, const double* d,
                  double* res, uint8_t* valid, cudaStream_t st);
int32_t assemble(dpv_problem* p, const double* q, const double* t, const double* d,
                 cudaStream_t st);
int32_t assemble_edges_pass(dpv_problem* p, const double* q, const double* t, const double* d,
                            double* obj, cudaStream_t st);
int32_t assemble_rest(dpv_problem* p, const double* t, cudaStream_t st);
int32_t coords(dpv_problem* p, const double* q, const double* t, const double* d, double scale,
               double* out, cudaStream_t st);
int32_t update_targets(dpv_problem* p, const double* tgt, const double* conf, cudaStream_t st);
int32_t corr_tma(const void* gmap, int64_t n_patches, const void* fmap0, const void* fmap1,
                 int64_t n_frames, const double* coords, const int32_t* ii, const int32_t* jj,
                 int64_t E, int C, int h0, int w0, int h1, int w1, int levels, float* out,
                 int64_t items_per_cta, cudaStream_t st);
int32_t corr(const void* gmap, const void* fmap0, const void* fmap1, const double* coords,
             const int32_t* ii, const int32_t* jj, int64_t E, int C, int h0, int w0, int h1,
             int w1, int levels, int radius, int dtype, float* out, cudaStream_t st);
int32_t proximity_detect(const double* centers, int64_t n, int64_t gap, double thr,
                         int64_t* pairs, int64_t cap, int64_t* count, cudaStream_t st);
int32_t ensure_pairs(dpv_problem* P);
int32_t coords_sel(dpv_problem* p, const double* q, const double* t, const double* d,
                   double scale, const int64_t* sel, int64_t n_sel, double* out,
                   cudaStream_t st);
int32_t reduced_system(dpv_problem* p, double lam, double* blocks, double* rhs, double* cinv,
                       cudaStream_t st);
void spd_plan_prefetch(dpv_problem* p);
int32_t solve(dpv_problem* p, double lam, double* dp, double* dd, int32_t* status,
              cudaStream_t st);
int32_t apply_step(dpv_problem* p, const double* q, const double* t, const double* d,
                   const double* dp, const double* dd, double* q2, double* t2, double* d2,
                   cudaStream_t st);
int32_t back_substitute(dpv_problem* p, double lam, const double* dp, double* dd,
                        cudaStream_t st);
int32_t cholesky_solve(double* a, int64_t lda, double* b, int64_t n, int32_t* status,
                       double* work, cudaStream_t st);
int64_t cholesky_work_doubles(int64_t n);
int64_t dense_workspace_doubles(int64_t N);
int32_t dense_factor_solve(double* A, int64_t ld, int64_t N, int32_t* status, double* x,
                           double* ws, const FactorPlan& pl, cudaStream_t st);
}  // namespace dpv
