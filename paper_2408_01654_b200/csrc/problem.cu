// Device index build for one BA problem: restates, bit-exactly, the
// reference's BAProblem edge/depth selection (ba.py:60-98), the per-edge
// structure (ba.py:124-141) and the normal-equation index
// _assembly_maps (ba.py:147-216), then adds the B200-specific layouts:
// segment-sorted SoA edge arrays and CSR lists for deterministic segmented
// reductions.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include <mutex>

#include "problem.cuh"

namespace dpv {
namespace {

// ---------------------------------------------------------------------------
// scratch allocations freed (stream-ordered) at scope exit

struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
    template <typename T>
    int32_t get(T** p, int64_t count) {
        void* q = nullptr;
        size_t b = sizeof(T) * (size_t)(count > 0 ? count : 1);
        DPV_CUDA(cudaMallocAsync(&q, b, st));
        ptrs.push_back(q);
        *p = reinterpret_cast<T*>(q);
        return DPV_OK;
    }
};

template <typename F>
int32_t cub_run(Scratch& sc, F f) {
    size_t bytes = 0;
    DPV_CUDA(f(nullptr, bytes));
    void* tmp = nullptr;
    DPV_TRY(sc.get(reinterpret_cast<char**>(&tmp), (int64_t)bytes + 16));
    DPV_CUDA(f(tmp, bytes));
    return DPV_OK;
}

template <typename T>
int32_t read_scalar(const T* dev, T* host, cudaStream_t st) {
    DPV_CUDA(cudaMemcpyAsync(host, dev, sizeof(T), cudaMemcpyDeviceToHost, st));
    DPV_CUDA(cudaStreamSynchronize(st));
    return DPV_OK;
}

int bits_for(uint64_t max_value) {
    int b = 1;
    while (b < 64 && (max_value >> b) != 0) ++b;
    return b;
}

// ---------------------------------------------------------------------------
// kernels

__global__ void k_select_flags(int64_t ne, const int32_t* src, const int32_t* dst, int32_t first,
                               int32_t last, uint8_t* flags) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t s = src[e], d = dst[e];
        flags[e] = ((s >= first && s <= last) || (d >= first && d <= last)) ? 1 : 0;
    }
}

__global__ void k_gather_edges(int64_t E, const int64_t* eidx, const int32_t* src,
                               const int32_t* dst, const int32_t* gp, const double* conf,
                               int32_t first, int32_t last, int32_t* p_src, int32_t* p_dst,
                               int32_t* p_gp, int32_t* p_vi, int32_t* p_vj, double* p_cmax) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t g = eidx[e];
        int32_t s = src[g], d = dst[g];
        p_src[e] = s;
        p_dst[e] = d;
        p_gp[e] = gp[g];
        p_vi[e] = (s >= first && s <= last) ? s - first : -1;
        p_vj[e] = (d >= first && d <= last) ? d - first : -1;
        p_cmax[e] = fmax(conf[2 * g], conf[2 * g + 1]);
    }
}

template <typename T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t n, T v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_rows(int64_t E, const int32_t* p_gp, const int32_t* depth_patch, int64_t P,
                       int32_t* p_row) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        p_row[e] = (int32_t)lower_bound_dev(depth_patch, P, p_gp[e]);
}

template <typename T>
__global__ void k_lower_bounds(int64_t nq, const T* sorted, int64_t n, int32_t* out) {
    // out[i] = lower_bound(sorted, i) for i in [0, nq]
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nq;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)lower_bound_dev(sorted, n, (T)i);
}

template <typename T, typename Q>
__global__ void k_lower_bounds_of(int64_t nq, const Q* queries, const T* sorted, int64_t n,
                                  int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = lower_bound_dev(sorted, n, (T)queries[i]);
}

__global__ void k_touch(int64_t E, const int32_t* p_src, const int32_t* p_dst,
                        const int32_t* p_vi, const int32_t* p_vj, int32_t* flags) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (p_vi[e] < 0) flags[p_src[e]] = 1;
        if (p_vj[e] < 0) flags[p_dst[e]] = 1;
    }
}

__global__ void k_seg_keys(int64_t E, const int32_t* p_src, const int32_t* p_dst, int64_t F,
                           uint64_t* key, int32_t* val) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        key[e] = (uint64_t)p_src[e] * (uint64_t)F + (uint64_t)p_dst[e];
        val[e] = (int32_t)e;
    }
}

__global__ void k_group_start(int64_t E, const uint64_t* key, int64_t* gstart) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x)
        gstart[i] = (i == 0 || key[i] != key[i - 1]) ? i : 0;
}

__global__ void k_seg_heads(int64_t E, const int64_t* gstart_max, uint8_t* head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x)
        head[i] = ((i - gstart_max[i]) % kSegMax) == 0 ? 1 : 0;
}

__global__ void k_gather_assembly(int64_t E, int m, const int32_t* perm, const int64_t* eidx,
                                  const int32_t* p_src, const int32_t* p_dst,
                                  const int32_t* p_row, const double* tgt, const double* conf,
                                  int32_t* a_src, int32_t* a_dst, int32_t* a_row,
                                  int32_t* a_pidx, int32_t* p_pos, double* a_tgt, double* a_w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t p = perm[i];
        int64_t g = eidx[p];
        a_src[i] = p_src[p];
        a_dst[i] = p_dst[p];
        a_row[i] = p_row[p];
        a_pidx[i] = p;
        p_pos[p] = (int32_t)i;
        for (int c = 0; c < 2 * m; ++c) a_tgt[(int64_t)c * E + i] = tgt[g * 2 * m + c];
        a_w[i] = conf[2 * g];
        a_w[E + i] = conf[2 * g + 1];
    }
}

__global__ void k_seg_ends(int64_t S, const int32_t* seg_ptr, const int32_t* a_src,
                           const int32_t* a_dst, int32_t* seg_src, int32_t* seg_dst) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
         s += (int64_t)gridDim.x * blockDim.x) {
        seg_src[s] = a_src[seg_ptr[s]];
        seg_dst[s] = a_dst[seg_ptr[s]];
    }
}

__global__ void k_rays(int64_t P, int m, const int32_t* depth_patch, const double* grid,
                       double fx, double fy, double cx, double cy, double* r_ray) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P;
         r += (int64_t)gridDim.x * blockDim.x) {
        const double* gp = grid + (int64_t)depth_patch[r] * 2 * m;
        for (int c = 0; c < m; ++c) {
            // pinhole_rays: IEEE division exactly as geometry.py:389-390
            r_ray[(int64_t)(2 * c) * P + r] = (gp[2 * c] - cx) / fx;
            r_ray[(int64_t)(2 * c + 1) * P + r] = (gp[2 * c + 1] - cy) / fy;
        }
    }
}

__global__ void k_iota(int64_t n, int32_t* v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

// incidence contributions, reference order: all source-side (rows_i) in
// problem order, then all target-side (rows_j) in problem order (ba.py:176-180)
__global__ void k_inc_contrib(int64_t E, const int32_t* p_vi, const int32_t* p_vj,
                              const int32_t* p_src, const int32_t* p_dst, const int32_t* p_row,
                              const int32_t* p_pos, const int64_t* off_i, const int64_t* off_j,
                              int64_t n_i, int64_t P, uint64_t* key, int32_t* code) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        bool distinct = p_src[e] != p_dst[e];
        if (distinct && p_vi[e] >= 0) {
            int64_t o = off_i[e];
            key[o] = (uint64_t)p_vi[e] * (uint64_t)P + (uint64_t)p_row[e];
            code[o] = p_pos[e] * 2;
        }
        if (distinct && p_vj[e] >= 0) {
            int64_t o = n_i + off_j[e];
            key[o] = (uint64_t)p_vj[e] * (uint64_t)P + (uint64_t)p_row[e];
            code[o] = p_pos[e] * 2 + 1;
        }
    }
}

__global__ void k_flags_ij(int64_t E, const int32_t* p_vi, const int32_t* p_vj,
                           const int32_t* p_src, const int32_t* p_dst, int64_t* fi,
                           int64_t* fj) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        bool distinct = p_src[e] != p_dst[e];
        fi[e] = (distinct && p_vi[e] >= 0) ? 1 : 0;
        fj[e] = (distinct && p_vj[e] >= 0) ? 1 : 0;
    }
}

__global__ void k_inc_split(int64_t I, const uint64_t* ukey, int64_t P, int32_t* inc_var,
                            int32_t* inc_row) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I;
         i += (int64_t)gridDim.x * blockDim.x) {
        inc_var[i] = (int32_t)(ukey[i] / (uint64_t)P);
        inc_row[i] = (int32_t)(ukey[i] % (uint64_t)P);
    }
}

__global__ void k_run_heads(int64_t n, const uint64_t* key, int32_t* head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void k_inc_inverse(int64_t n, const int32_t* run_incl, const int32_t* orig,
                              const int32_t* code_sorted_src, int32_t* inc_inv,
                              int32_t* inc_con) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t o = orig[i];
        inc_inv[o] = run_incl[i] - 1;
        inc_con[i] = code_sorted_src[o];
    }
}

__global__ void k_pair_counts(int64_t P, const int32_t* rinc_ptr, int64_t* npair) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t m = rinc_ptr[r + 1] - rinc_ptr[r];
        npair[r] = m * (m + 1) / 2;
    }
}

// ---- grouped Schur index: rows with identical incidence-var lists ---------
__global__ void k_row_hash(int64_t P, const int32_t* rinc_ptr, const int32_t* rinc,
                           const int32_t* inc_var, uint64_t* h, int32_t* idx) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P;
         r += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = 1469598103934665603ull ^ (uint64_t)(rinc_ptr[r + 1] - rinc_ptr[r]);
        for (int32_t k = rinc_ptr[r]; k < rinc_ptr[r + 1]; ++k) {
            x ^= (uint64_t)(uint32_t)inc_var[rinc[k]] + 0x9e3779b97f4a7c15ull;
            x *= 1099511628211ull;
            x ^= x >> 29;
        }
        h[r] = x;
        idx[r] = (int32_t)r;
    }
}

__global__ void k_group_flags(int64_t P, const uint64_t* hs, int32_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || hs[i] != hs[i - 1]) ? 1 : 0;
}

// group start positions (in sorted order) and a full check that every row's
// var list equals its group head's (hash collisions -> *bad)
__global__ void k_group_verify(int64_t P, const int32_t* flag, const int32_t* gid,
                               const int32_t* rows, const int32_t* rinc_ptr, const int32_t* rinc,
                               const int32_t* inc_var, int32_t* gstart, int32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) gstart[gid[i]] = (int32_t)i;
}

__global__ void k_group_verify2(int64_t P, const int32_t* gid, const int32_t* gstart,
                                const int32_t* rows, const int32_t* rinc_ptr, const int32_t* rinc,
                                const int32_t* inc_var, int32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[i], h = rows[gstart[gid[i]]];
        const int32_t m = rinc_ptr[r + 1] - rinc_ptr[r];
        bool ok = m == rinc_ptr[h + 1] - rinc_ptr[h];
        for (int32_t j = 0; ok && j < m; ++j)
            ok = inc_var[rinc[rinc_ptr[r] + j]] == inc_var[rinc[rinc_ptr[h] + j]];
        if (!ok) atomicExch(bad, 1);
    }
}

// per chunk (rows of one group) and local block (j1 <= j2): the union-key
// index of (var_j1, var_j2) and the block's slot in the chunk buffer
__global__ void k_chunk_contrib(int64_t n_chunks, const int4* chunks, const int32_t* rows,
                                const int32_t* rinc_ptr, const int32_t* rinc,
                                const int32_t* inc_var, const uint64_t* union_keys, int64_t W,
                                int64_t nfree, uint64_t* ckey, int32_t* cblk) {
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int4 ch = chunks[c];
        const int32_t head = rows[ch.x];
        const int m = ch.z;
        const int nb = m * (m + 1) / 2;
        for (int q = threadIdx.x; q < nb; q += blockDim.x) {
            int j1 = 0, rem = q;
            while (rem >= m - j1) {
                rem -= m - j1;
                ++j1;
            }
            const int j2 = j1 + rem;
            const uint64_t a = (uint64_t)inc_var[rinc[rinc_ptr[head] + j1]];
            const uint64_t b = (uint64_t)inc_var[rinc[rinc_ptr[head] + j2]];
            const uint64_t key = a * (uint64_t)nfree + b;
            const int64_t w = lower_bound_dev(union_keys, W, key);
            ckey[(int64_t)ch.w + q] = (uint64_t)w;
            cblk[(int64_t)ch.w + q] = ch.w + q;
        }
    }
}

__global__ void k_sub_one(int64_t n, int32_t* a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] -= 1;
}

// Schur pair runs without materialising the pairs.  Pair (il, ir) of a depth
// row continues a run iff (il-1, ir-1) is a pair of the same key: both
// incidences belong to the same vars and share a row.  MODE 0 counts the run
// heads per row, MODE 1 writes them in pair order (deterministic).  The
// row's incidences (index, var, and the row of the previous incidence of the
// same var, or -1) are staged in shared memory once, then the pairs
// (l, r >= l) are tested l-major with lanes over r: no triangular index
// decode and no per-pair gathers.  Rows with more than kPhMax incidences
// take a per-pair path.
constexpr int kPhMax = 128;

template <int MODE>
__global__ void __launch_bounds__(256) k_pair_heads_staged(
    int64_t P, const int32_t* rinc_ptr, const int32_t* rinc, const int32_t* inc_var,
    const int32_t* inc_row, int64_t nfree, int32_t* hcount, const int64_t* hoff, uint64_t* hkey,
    int32_t* hl, int32_t* hr) {
    __shared__ int32_t s_il[8][kPhMax], s_var[8][kPhMax], s_prev[8][kPhMax];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int32_t* il_s = s_il[wib];
    int32_t* var_s = s_var[wib];
    int32_t* prev_s = s_prev[wib];
    for (int64_t r = warp; r < P; r += nwarps) {
        const int32_t s = rinc_ptr[r];
        const int32_t m = rinc_ptr[r + 1] - s;
        int64_t base = MODE ? hoff[r] : 0;
        int32_t cnt = 0;
        if (m > kPhMax) {      // per-pair path
            const int64_t tot = (int64_t)m * (m + 1) / 2;
            for (int64_t k0 = 0; k0 < tot; k0 += 32) {
                const int64_t k = k0 + lane;
                bool head = false;
                int32_t il = 0, ir = 0;
                if (k < tot) {
                    int32_t l = 0;
                    int64_t rowlen = m, acc = 0;
                    while (acc + rowlen <= k) { acc += rowlen; --rowlen; ++l; }
                    const int32_t rr = l + (int32_t)(k - acc);
                    il = rinc[s + l];
                    ir = rinc[s + rr];
                    head = !(il > 0 && ir > 0 && inc_var[il - 1] == inc_var[il] &&
                             inc_var[ir - 1] == inc_var[ir] && inc_row[il - 1] == inc_row[ir - 1]);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, head);
                if (MODE == 1 && head) {
                    const int64_t pos = base + cnt + __popc(bal & ((1u << lane) - 1u));
                    hkey[pos] = (uint64_t)inc_var[il] * (uint64_t)nfree + (uint64_t)inc_var[ir];
                    hl[pos] = il;
                    hr[pos] = ir;
                }
                cnt += __popc(bal);
            }
        } else {
            __syncwarp();
            for (int j = lane; j < m; j += 32) {
                const int32_t il = rinc[s + j];
                const int32_t v = inc_var[il];
                il_s[j] = il;
                var_s[j] = v;
                prev_s[j] = (il > 0 && inc_var[il - 1] == v) ? inc_row[il - 1] : -1;
            }
            __syncwarp();
            for (int l = 0; l < m; ++l) {
                const int32_t pl = prev_s[l];
                for (int r0 = l; r0 < m; r0 += 32) {
                    const int rr = r0 + lane;
                    const bool act = rr < m;
                    const bool head = act && !(pl >= 0 && prev_s[rr] == pl);
                    const unsigned bal = __ballot_sync(0xffffffffu, head);
                    if (MODE == 1 && head) {
                        const int64_t pos = base + cnt + __popc(bal & ((1u << lane) - 1u));
                        hkey[pos] = (uint64_t)var_s[l] * (uint64_t)nfree + (uint64_t)var_s[rr];
                        hl[pos] = il_s[l];
                        hr[pos] = il_s[rr];
                    }
                    cnt += __popc(bal);
                }
            }
        }
        if (MODE == 0 && lane == 0) hcount[r] = cnt;
    }
}

// run length: warp per head, 32 offsets per probe
__global__ void k_run_extent(int64_t NR, int64_t I, const int32_t* run_l, const int32_t* run_r,
                             const int32_t* inc_var, const int32_t* inc_row, int32_t* run_len) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = warp; q < NR; q += nwarps) {
        const int32_t il = run_l[q], ir = run_r[q];
        const int32_t a = inc_var[il], b = inc_var[ir];
        int32_t len = 0;
        for (int32_t t0 = 0;; t0 += 32) {
            const int32_t t = t0 + lane;
            const bool ok = il + t < I && ir + t < I && inc_var[il + t] == a &&
                            inc_var[ir + t] == b && inc_row[il + t] == inc_row[ir + t];
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (bal != 0xffffffffu) {
                len = t0 + __ffs(~bal) - 1;
                break;
            }
        }
        if (lane == 0) run_len[q] = len;
    }
}

// lazily materialised pairs (parity export): run q -> pairs off[q] + t
__global__ void k_expand_runs(int64_t NR, const int64_t* off, const int32_t* run_l,
                              const int32_t* run_r, const int32_t* run_len, int32_t* pl,
                              int32_t* pr) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = warp; q < NR; q += nwarps)
        for (int32_t t = lane; t < run_len[q]; t += 32) {
            pl[off[q] + t] = run_l[q] + t;
            pr[off[q] + t] = run_r[q] + t;
        }
}

__global__ void k_key_pair_ptr(int64_t W, const int32_t* key_run_ptr, const int64_t* off,
                               int64_t* key_pair_ptr) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= W;
         w += (int64_t)gridDim.x * blockDim.x)
        key_pair_ptr[w] = off[key_run_ptr[w]];
}

__global__ void k_i32_to_i64(int64_t n, const int32_t* a, int64_t* b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

__global__ void k_i64_to_i32(int64_t n, const int64_t* a, int32_t* b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (int32_t)a[i];
}

__global__ void k_gather_i32(int64_t n, const int32_t* idx, const int32_t* src, int32_t* dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

// up to three folded Hessian keys per segment (ba.py:161-173): diagonal of the
// source var, diagonal of the target var, off-diagonal (min, max) negated
__global__ void k_seg_hkeys(int64_t S, const int32_t* seg_src, const int32_t* seg_dst,
                            int32_t first, int32_t last, int64_t nfree, uint64_t* key,
                            int32_t* code, uint64_t* vkey, int32_t* vcode) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t a = seg_src[s], b = seg_dst[s];
        int32_t vi = (a >= first && a <= last) ? a - first : -1;
        int32_t vj = (b >= first && b <= last) ? b - first : -1;
        bool distinct = a != b;
        const uint64_t none = ~0ull;
        key[3 * s] = (distinct && vi >= 0) ? (uint64_t)vi * (nfree + 1) : none;
        key[3 * s + 1] = (distinct && vj >= 0) ? (uint64_t)vj * (nfree + 1) : none;
        key[3 * s + 2] = (distinct && vi >= 0 && vj >= 0)
                             ? (uint64_t)min(vi, vj) * nfree + (uint64_t)max(vi, vj)
                             : none;
        code[3 * s] = (int32_t)s * 2;
        code[3 * s + 1] = (int32_t)s * 2;
        code[3 * s + 2] = (int32_t)s * 2 + 1;
        // rhs_pose: source side -g (ba.py:378), target side +g (ba.py:380)
        vkey[2 * s] = (distinct && vi >= 0) ? (uint64_t)vi : none;
        vkey[2 * s + 1] = (distinct && vj >= 0) ? (uint64_t)vj : none;
        vcode[2 * s] = (int32_t)s * 2 + 1;
        vcode[2 * s + 1] = (int32_t)s * 2;
    }
}

__global__ void k_diag_keys(int64_t nfree, uint64_t* key) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nfree;
         v += (int64_t)gridDim.x * blockDim.x)
        key[v] = (uint64_t)v * (nfree + 1);
}

__global__ void k_key_ab(int64_t W, const int64_t* keys, int64_t nfree, int32_t* ka,
                         int32_t* kb) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
         w += (int64_t)gridDim.x * blockDim.x) {
        ka[w] = (int32_t)(keys[w] / nfree);
        kb[w] = (int32_t)(keys[w] % nfree);
    }
}

__global__ void k_keys_to_union(int64_t n, const uint64_t* key, const int64_t* ukeys,
                                int64_t W, uint64_t* widx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[i];
        widx[i] = (k == ~0ull) ? ~0ull : (uint64_t)lower_bound_dev(ukeys, W, (int64_t)k);
    }
}

__global__ void k_frame_rot(int64_t F, const double* q, double* R) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F;
         f += (int64_t)gridDim.x * blockDim.x)
        quat_to_rot(q + 4 * f, R + 9 * f);
}

}  // namespace

int32_t frame_rotations(dpv_problem* p, const double* q, cudaStream_t st) {
    k_frame_rot<<<grid_for(p->F, 256), 256, 0, st>>>(p->F, q, p->frame_R);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

// ---------------------------------------------------------------------------

// DPV_BUILD_PROFILE=1: per-phase wall times of the index build (synchronising)
struct PhaseTimer {
    bool on = getenv("DPV_BUILD_PROFILE") != nullptr;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    explicit PhaseTimer(cudaStream_t s) : st(s) {}
    void lap(const char* name) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[dpv build] %-28s %8.3f ms\n", name,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

int32_t build_problem(const dpv_graph* g, int32_t first, int32_t last, const int64_t* eidx_in,
                      int64_t n_eidx, const int64_t* extra_keys, int64_t n_extra,
                      cudaStream_t st, dpv_problem* P) {
    DPV_ARG(g != nullptr, "graph is NULL");
    DPV_ARG(g->cells > 0 && g->cells <= 64, "cells out of range");
    DPV_ARG(0 <= first && first <= last && last < g->n_frames, "free range out of bounds");
    DPV_ARG(!(first == 0 && last == g->n_frames - 1),
            "at least one pose must stay fixed to anchor the gauge");
    Scratch sc(st);
    const int B = 256;
    P->F = g->n_frames;
    P->m = g->cells;
    P->first = first;
    P->last = last;
    P->n = last - first + 1;
    for (int i = 0; i < 4; ++i) P->intr[i] = g->intr[i];
    const int m = P->m;
    int64_t* dcount;
    DPV_TRY(P->alloc(&P->count_buf, 4));
    dcount = P->count_buf;

    PhaseTimer ptimer(st);
    // 1. edge selection (ba.py:72-77)
    if (eidx_in) {
        P->E = n_eidx;
        DPV_TRY(P->alloc(&P->edge_idx, P->E));
        DPV_CUDA(cudaMemcpyAsync(P->edge_idx, eidx_in, sizeof(int64_t) * P->E,
                                 cudaMemcpyDeviceToDevice, st));
    } else {
        const int64_t NE = g->n_edges;
        uint8_t* flags;
        DPV_TRY(sc.get(&flags, NE));
        k_select_flags<<<grid_for(NE, B), B, 0, st>>>(NE, g->edge_src, g->edge_dst, first, last,
                                                       flags);
        DPV_CHECK_LAUNCH();
        int64_t* sel;
        DPV_TRY(sc.get(&sel, NE));
        cub::CountingInputIterator<int64_t> it(0);
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, it, flags, sel, dcount, (int)NE, st);
        }));
        DPV_TRY(read_scalar(dcount, &P->E, st));
        DPV_TRY(P->alloc(&P->edge_idx, P->E));
        DPV_CUDA(cudaMemcpyAsync(P->edge_idx, sel, sizeof(int64_t) * P->E,
                                 cudaMemcpyDeviceToDevice, st));
    }
    const int64_t E = P->E;
    const int GE = grid_for(E, B);

    int32_t *p_src, *p_dst, *p_gp;
    DPV_TRY(sc.get(&p_src, E));
    DPV_TRY(sc.get(&p_dst, E));
    DPV_TRY(sc.get(&p_gp, E));
    DPV_TRY(P->alloc(&P->p_vi, E));
    DPV_TRY(P->alloc(&P->p_vj, E));
    DPV_TRY(P->alloc(&P->p_conf_max, E));
    DPV_TRY(P->alloc(&P->p_row, E));
    DPV_TRY(P->alloc(&P->p_pos, E));
    if (E > 0) {
        k_gather_edges<<<GE, B, 0, st>>>(E, P->edge_idx, g->edge_src, g->edge_dst, g->edge_gpatch,
                                         g->edge_conf, first, last, p_src, p_dst, p_gp, P->p_vi,
                                         P->p_vj, P->p_conf_max);
        DPV_CHECK_LAUNCH();
    }

    ptimer.lap("before 2. depth keys = sort");
    // 2. depth keys = sorted {(src_frame, src_patch)} (ba.py:80-83)
    {
        int32_t* sorted;
        DPV_TRY(sc.get(&sorted, E));
        int32_t* uniq;
        DPV_TRY(sc.get(&uniq, E));
        int eb = bits_for((uint64_t)std::max<int64_t>(g->n_patches, 1));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, p_gp, sorted, (int)E, 0, eb, st);
        }));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Unique(t, b, sorted, uniq, dcount, (int)E, st);
        }));
        DPV_TRY(read_scalar(dcount, &P->P, st));
        DPV_TRY(P->alloc(&P->depth_patch, P->P));
        DPV_CUDA(cudaMemcpyAsync(P->depth_patch, uniq, sizeof(int32_t) * P->P,
                                 cudaMemcpyDeviceToDevice, st));
    }
    const int64_t NPD = P->P;
    if (E > 0) {
        k_rows<<<GE, B, 0, st>>>(E, p_gp, P->depth_patch, NPD, P->p_row);
        DPV_CHECK_LAUNCH();
    }

    ptimer.lap("before 3. touched fixed fra");
    // 3. touched fixed frames (ba.py:89-95)
    {
        int32_t* fl;
        DPV_TRY(sc.get(&fl, P->F));
        DPV_CUDA(cudaMemsetAsync(fl, 0, sizeof(int32_t) * P->F, st));
        if (E > 0) {
            k_touch<<<GE, B, 0, st>>>(E, p_src, p_dst, P->p_vi, P->p_vj, fl);
            DPV_CHECK_LAUNCH();
        }
        int32_t* sel;
        DPV_TRY(sc.get(&sel, P->F));
        cub::CountingInputIterator<int32_t> it(0);
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, it, fl, sel, dcount, (int)P->F, st);
        }));
        DPV_TRY(read_scalar(dcount, &P->T, st));
        DPV_TRY(P->alloc(&P->touched, P->T));
        DPV_CUDA(cudaMemcpyAsync(P->touched, sel, sizeof(int32_t) * P->T,
                                 cudaMemcpyDeviceToDevice, st));
        P->scale_degenerate = P->T <= 1 ? 1 : 0;
        P->touched0 = -1;
        if (P->T > 0) {
            DPV_CUDA(cudaMemcpyAsync(&P->touched0, P->touched, sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, st));
            DPV_CUDA(cudaStreamSynchronize(st));
        }
    }

    ptimer.lap("before 4. segments: stable ");
    // 4. segments: stable sort by (src, dst), chunks of <= kSegMax edges
    int32_t* perm;
    DPV_TRY(sc.get(&perm, E));
    {
        uint64_t *k0, *k1;
        int32_t* v0;
        DPV_TRY(sc.get(&k0, E));
        DPV_TRY(sc.get(&k1, E));
        DPV_TRY(sc.get(&v0, E));
        if (E > 0) {
            k_seg_keys<<<GE, B, 0, st>>>(E, p_src, p_dst, P->F, k0, v0);
            DPV_CHECK_LAUNCH();
        }
        int eb = bits_for((uint64_t)P->F * (uint64_t)P->F);
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, k0, k1, v0, perm, (int)E, 0, eb, st);
        }));
        int64_t *gs, *gmax;
        DPV_TRY(sc.get(&gs, E));
        DPV_TRY(sc.get(&gmax, E));
        uint8_t* head;
        DPV_TRY(sc.get(&head, E));
        if (E > 0) {
            k_group_start<<<GE, B, 0, st>>>(E, k1, gs);
            DPV_CHECK_LAUNCH();
        }
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::InclusiveScan(t, b, gs, gmax, cub::Max(), (int)E, st);
        }));
        if (E > 0) {
            k_seg_heads<<<GE, B, 0, st>>>(E, gmax, head);
            DPV_CHECK_LAUNCH();
        }
        int32_t* heads;
        DPV_TRY(sc.get(&heads, E + 1));
        cub::CountingInputIterator<int32_t> it(0);
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, it, head, heads, dcount, (int)E, st);
        }));
        DPV_TRY(read_scalar(dcount, &P->S, st));
        DPV_TRY(P->alloc(&P->seg_ptr, P->S + 1));
        DPV_CUDA(cudaMemcpyAsync(P->seg_ptr, heads, sizeof(int32_t) * P->S,
                                 cudaMemcpyDeviceToDevice, st));
        int32_t e32 = (int32_t)E;
        DPV_CUDA(cudaMemcpyAsync(P->seg_ptr + P->S, &e32, sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
        DPV_CUDA(cudaStreamSynchronize(st));
    }

    ptimer.lap("before 5. assembly-order So");
    // 5. assembly-order SoA copies (ba.py:124-141 structure, permuted)
    DPV_TRY(P->alloc(&P->a_src, E));
    DPV_TRY(P->alloc(&P->a_dst, E));
    DPV_TRY(P->alloc(&P->a_row, E));
    DPV_TRY(P->alloc(&P->a_pidx, E));
    DPV_TRY(P->alloc(&P->a_tgt, E * 2 * m));
    DPV_TRY(P->alloc(&P->a_w, E * 2));
    if (E > 0) {
        k_gather_assembly<<<GE, B, 0, st>>>(E, m, perm, P->edge_idx, p_src, p_dst, P->p_row,
                                            g->edge_target, g->edge_conf, P->a_src, P->a_dst,
                                            P->a_row, P->a_pidx, P->p_pos, P->a_tgt, P->a_w);
        DPV_CHECK_LAUNCH();
    }
    DPV_TRY(P->alloc(&P->seg_src, P->S));
    DPV_TRY(P->alloc(&P->seg_dst, P->S));
    if (P->S > 0) {
        k_seg_ends<<<grid_for(P->S, B), B, 0, st>>>(P->S, P->seg_ptr, P->a_src, P->a_dst,
                                                    P->seg_src, P->seg_dst);
        DPV_CHECK_LAUNCH();
    }
    DPV_TRY(P->alloc(&P->r_ray, NPD * 2 * m));
    if (NPD > 0) {
        k_rays<<<grid_for(NPD, B), B, 0, st>>>(NPD, m, P->depth_patch, g->patch_grid, g->intr[0],
                                               g->intr[1], g->intr[2], g->intr[3], P->r_ray);
        DPV_CHECK_LAUNCH();
    }

    ptimer.lap("before 6. per-row CSR over ");
    // 6. per-row CSR over assembly positions
    DPV_TRY(P->alloc(&P->row_ptr, NPD + 1));
    DPV_TRY(P->alloc(&P->row_pos, E));
    {
        int32_t *iota, *rows_sorted;
        DPV_TRY(sc.get(&iota, E));
        DPV_TRY(sc.get(&rows_sorted, E));
        if (E > 0) {
            k_iota<<<GE, B, 0, st>>>(E, iota);
            DPV_CHECK_LAUNCH();
        }
        int eb = bits_for((uint64_t)std::max<int64_t>(NPD, 1));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, P->a_row, rows_sorted, iota, P->row_pos,
                                                   (int)E, 0, eb, st);
        }));
        k_lower_bounds<int32_t><<<grid_for(NPD + 1, B), B, 0, st>>>(NPD, rows_sorted, E,
                                                                     P->row_ptr);
        DPV_CHECK_LAUNCH();
    }

    ptimer.lap("before 7. incidences (ba.py");
    // 7. incidences (ba.py:175-182): unique (var, row) keys of the source- and
    //    target-side rows, with the contribution CSR and inc_inv
    int32_t* inc_inv_tmp = nullptr;
    {
        int64_t *fi, *fj, *oi, *oj;
        DPV_TRY(sc.get(&fi, E + 1));
        DPV_TRY(sc.get(&fj, E + 1));
        DPV_CUDA(cudaMemsetAsync(fi + E, 0, sizeof(int64_t), st));
        DPV_CUDA(cudaMemsetAsync(fj + E, 0, sizeof(int64_t), st));
        DPV_TRY(sc.get(&oi, E + 1));
        DPV_TRY(sc.get(&oj, E + 1));
        if (E > 0) {
            k_flags_ij<<<GE, B, 0, st>>>(E, P->p_vi, P->p_vj, p_src, p_dst, fi, fj);
            DPV_CHECK_LAUNCH();
        }
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, fi, oi, (int)E + 1, st);
        }));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, fj, oj, (int)E + 1, st);
        }));
        int64_t n_i = 0, n_j = 0;
        DPV_CUDA(cudaMemcpyAsync(&n_i, oi + E, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaMemcpyAsync(&n_j, oj + E, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        P->NC = n_i + n_j;
        const int64_t NC = P->NC;
        uint64_t *ck, *cks;
        int32_t *ccode, *corig, *corig_s;
        DPV_TRY(sc.get(&ck, NC));
        DPV_TRY(sc.get(&cks, NC));
        DPV_TRY(sc.get(&ccode, NC));
        DPV_TRY(sc.get(&corig, NC));
        DPV_TRY(sc.get(&corig_s, NC));
        if (E > 0) {
            k_inc_contrib<<<GE, B, 0, st>>>(E, P->p_vi, P->p_vj, p_src, p_dst, P->p_row, P->p_pos,
                                            oi, oj, n_i, NPD, ck, ccode);
            DPV_CHECK_LAUNCH();
        }
        if (NC > 0) {
            k_iota<<<grid_for(NC, B), B, 0, st>>>(NC, corig);
            DPV_CHECK_LAUNCH();
        }
        int eb = bits_for((uint64_t)P->n * (uint64_t)std::max<int64_t>(NPD, 1));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, ck, cks, corig, corig_s, (int)NC, 0, eb,
                                                   st);
        }));
        uint64_t* ukey;
        int32_t* counts;
        DPV_TRY(sc.get(&ukey, NC));
        DPV_TRY(sc.get(&counts, NC + 1));     // + the scan's terminating zero (I == NC possible)
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRunLengthEncode::Encode(t, b, cks, ukey, counts, dcount, (int)NC,
                                                      st);
        }));
        DPV_TRY(read_scalar(dcount, &P->I, st));
        const int64_t I = P->I;
        DPV_TRY(P->alloc(&P->inc_var, I));
        DPV_TRY(P->alloc(&P->inc_row, I));
        DPV_TRY(P->alloc(&P->inc_ptr, I + 1));
        DPV_TRY(P->alloc(&P->inc_con, NC));
        DPV_TRY(sc.get(&inc_inv_tmp, NC));
        if (I > 0) {
            k_inc_split<<<grid_for(I, B), B, 0, st>>>(I, ukey, NPD, P->inc_var, P->inc_row);
            DPV_CHECK_LAUNCH();
        }
        DPV_CUDA(cudaMemsetAsync(counts + I, 0, sizeof(int32_t), st));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, counts, P->inc_ptr, (int)I + 1, st);
        }));
        int32_t *heads, *runs;
        DPV_TRY(sc.get(&heads, NC));
        DPV_TRY(sc.get(&runs, NC));
        if (NC > 0) {
            k_run_heads<<<grid_for(NC, B), B, 0, st>>>(NC, cks, heads);
            DPV_CHECK_LAUNCH();
        }
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::InclusiveSum(t, b, heads, runs, (int)NC, st);
        }));
        if (NC > 0) {
            k_inc_inverse<<<grid_for(NC, B), B, 0, st>>>(NC, runs, corig_s, ccode, inc_inv_tmp,
                                                         P->inc_con);
            DPV_CHECK_LAUNCH();
        }
    }
    const int64_t I = P->I;
    // keep inc_inv for parity export
    {
        int32_t* keep;
        DPV_TRY(P->alloc(&keep, P->NC));
        DPV_CUDA(cudaMemcpyAsync(keep, inc_inv_tmp, sizeof(int32_t) * P->NC,
                                 cudaMemcpyDeviceToDevice, st));
        P->p_inc_inv = keep;
    }
    DPV_TRY(P->alloc(&P->var_inc_ptr, P->n + 1));
    k_lower_bounds<int32_t><<<grid_for(P->n + 1, B), B, 0, st>>>(P->n, P->inc_var, I,
                                                                  P->var_inc_ptr);
    DPV_CHECK_LAUNCH();

    ptimer.lap("before 8. incidences per de");
    // 8. incidences per depth row, ascending var (ba.py:185-189 `order`)
    DPV_TRY(P->alloc(&P->rinc_ptr, NPD + 1));
    DPV_TRY(P->alloc(&P->rinc, I));
    {
        int32_t *iota, *rows_sorted;
        DPV_TRY(sc.get(&iota, I));
        DPV_TRY(sc.get(&rows_sorted, I));
        if (I > 0) {
            k_iota<<<grid_for(I, B), B, 0, st>>>(I, iota);
            DPV_CHECK_LAUNCH();
        }
        int eb = bits_for((uint64_t)std::max<int64_t>(NPD, 1));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, P->inc_row, rows_sorted, iota, P->rinc,
                                                   (int)I, 0, eb, st);
        }));
        k_lower_bounds<int32_t><<<grid_for(NPD + 1, B), B, 0, st>>>(NPD, rows_sorted, I,
                                                                     P->rinc_ptr);
        DPV_CHECK_LAUNCH();
    }

    ptimer.lap("before 9. Schur pairs per r");
    // 9. Schur pairs per row (ba.py:190-199) in run-length form: only the run
    // heads are enumerated and sorted by folded key (stable -> row order); the
    // pair list itself is materialised lazily for the parity export
    uint64_t* hkey_s = nullptr;
    {
        int64_t *npair, *poff;
        DPV_TRY(sc.get(&npair, NPD + 1));
        DPV_TRY(sc.get(&poff, NPD + 1));
        if (NPD > 0) {
            k_pair_counts<<<grid_for(NPD, B), B, 0, st>>>(NPD, P->rinc_ptr, npair);
            DPV_CHECK_LAUNCH();
        }
        DPV_CUDA(cudaMemsetAsync(npair + NPD, 0, sizeof(int64_t), st));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, npair, poff, (int)NPD + 1, st);
        }));
        DPV_TRY(read_scalar(poff + NPD, &P->NP, st));
        int32_t* hcount;
        int64_t *hcount64, *hoff;
        DPV_TRY(sc.get(&hcount, NPD + 1));
        DPV_TRY(sc.get(&hcount64, NPD + 1));
        DPV_TRY(sc.get(&hoff, NPD + 1));
        if (NPD > 0) {
            k_pair_heads_staged<0><<<grid_for(NPD * 32, B), B, 0, st>>>(
                NPD, P->rinc_ptr, P->rinc, P->inc_var, P->inc_row, P->n, hcount, nullptr, nullptr,
                nullptr, nullptr);
            DPV_CHECK_LAUNCH();
            k_i32_to_i64<<<grid_for(NPD, B), B, 0, st>>>(NPD, hcount, hcount64);
            DPV_CHECK_LAUNCH();
        }
        DPV_CUDA(cudaMemsetAsync(hcount64 + NPD, 0, sizeof(int64_t), st));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, hcount64, hoff, (int)NPD + 1, st);
        }));
        int64_t nr = 0;
        DPV_TRY(read_scalar(hoff + NPD, &nr, st));
        P->NR = nr;
        uint64_t* hk;
        int32_t *hl, *hr, *hid, *hid_s;
        DPV_TRY(sc.get(&hk, nr));
        DPV_TRY(sc.get(&hkey_s, nr));
        DPV_TRY(sc.get(&hl, nr));
        DPV_TRY(sc.get(&hr, nr));
        DPV_TRY(sc.get(&hid, nr));
        DPV_TRY(sc.get(&hid_s, nr));
        if (NPD > 0) {
            k_pair_heads_staged<1><<<grid_for(NPD * 32, B), B, 0, st>>>(
                NPD, P->rinc_ptr, P->rinc, P->inc_var, P->inc_row, P->n, nullptr, hoff, hk, hl,
                hr);
            DPV_CHECK_LAUNCH();
        }
        if (nr > 0) {
            k_iota<<<grid_for(nr, B), B, 0, st>>>(nr, hid);
            DPV_CHECK_LAUNCH();
        }
        const int eb = bits_for((uint64_t)P->n * (uint64_t)P->n);
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, hk, hkey_s, hid, hid_s, (int)nr, 0, eb,
                                                   st);
        }));
        DPV_TRY(P->alloc(&P->run_l, nr));
        DPV_TRY(P->alloc(&P->run_r, nr));
        DPV_TRY(P->alloc(&P->run_len, nr));
        if (nr > 0) {
            k_gather_i32<<<grid_for(nr, B), B, 0, st>>>(nr, hid_s, hl, P->run_l);
            DPV_CHECK_LAUNCH();
            k_gather_i32<<<grid_for(nr, B), B, 0, st>>>(nr, hid_s, hr, P->run_r);
            DPV_CHECK_LAUNCH();
            k_run_extent<<<grid_for(nr * 32, B), B, 0, st>>>(nr, P->I, P->run_l, P->run_r,
                                                              P->inc_var, P->inc_row, P->run_len);
            DPV_CHECK_LAUNCH();
        }
    }
    const int64_t NRH = P->NR;

    ptimer.lap("before 10. union keys = uni");
    // 10. union keys = unique(hpp ∪ schur ∪ diagonal) (ba.py:201-203)
    uint64_t *hk, *vk;
    int32_t *hc, *vc;
    DPV_TRY(sc.get(&hk, 3 * P->S));
    DPV_TRY(sc.get(&hc, 3 * P->S));
    DPV_TRY(sc.get(&vk, 2 * P->S));
    DPV_TRY(sc.get(&vc, 2 * P->S));
    if (P->S > 0) {
        k_seg_hkeys<<<grid_for(P->S, B), B, 0, st>>>(P->S, P->seg_src, P->seg_dst, first, last,
                                                     P->n, hk, hc, vk, vc);
        DPV_CHECK_LAUNCH();
    }
    {
        // the run heads are sorted by key: unique them (every pair key has a
        // head), then sort only the short union with the other key sets
        uint64_t* pk_u;
        int64_t npu = 0;
        DPV_TRY(sc.get(&pk_u, std::max<int64_t>(NRH, 1)));
        if (NRH > 0) {
            DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
                return cub::DeviceSelect::Unique(t, b, hkey_s, pk_u, dcount, (int)NRH, st);
            }));
            DPV_TRY(read_scalar(dcount, &npu, st));
        }
        const int64_t tot = npu + P->n + 3 * P->S + n_extra;
        uint64_t *all, *alls, *uk;
        DPV_TRY(sc.get(&all, tot));
        DPV_TRY(sc.get(&alls, tot));
        DPV_TRY(sc.get(&uk, tot));
        if (npu > 0)
            DPV_CUDA(cudaMemcpyAsync(all, pk_u, sizeof(uint64_t) * npu, cudaMemcpyDeviceToDevice,
                                     st));
        if (P->n > 0) {
            k_diag_keys<<<grid_for(P->n, B), B, 0, st>>>(P->n, all + npu);
            DPV_CHECK_LAUNCH();
        }
        if (P->S > 0)
            DPV_CUDA(cudaMemcpyAsync(all + npu + P->n, hk, sizeof(uint64_t) * 3 * P->S,
                                     cudaMemcpyDeviceToDevice, st));
        // sharded global BA: every shard carries the global block pattern
        if (n_extra > 0)
            DPV_CUDA(cudaMemcpyAsync(all + npu + P->n + 3 * P->S, extra_keys,
                                     sizeof(uint64_t) * n_extra, cudaMemcpyDeviceToDevice, st));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, all, alls, (int)tot, 0, 64, st);
        }));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Unique(t, b, alls, uk, dcount, (int)tot, st);
        }));
        int64_t nu = 0;
        DPV_TRY(read_scalar(dcount, &nu, st));
        // drop the ~0 "absent" sentinel (sorts last)
        uint64_t lastkey = 0;
        if (nu > 0) {
            DPV_CUDA(cudaMemcpyAsync(&lastkey, uk + nu - 1, sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, st));
            DPV_CUDA(cudaStreamSynchronize(st));
            if (lastkey == ~0ull) --nu;
        }
        P->W = nu;
        DPV_TRY(P->alloc(&P->union_keys, P->W));
        DPV_CUDA(cudaMemcpyAsync(P->union_keys, uk, sizeof(int64_t) * P->W,
                                 cudaMemcpyDeviceToDevice, st));
    }
    const int64_t W = P->W;
    DPV_TRY(P->alloc(&P->key_a, W));
    DPV_TRY(P->alloc(&P->key_b, W));
    if (W > 0) {
        k_key_ab<<<grid_for(W, B), B, 0, st>>>(W, P->union_keys, P->n, P->key_a, P->key_b);
        DPV_CHECK_LAUNCH();
    }
    // key -> runs CSR (heads sorted by key)
    DPV_TRY(P->alloc(&P->key_run_ptr, W + 1));
    if (W > 0) {
        int64_t* krp;
        DPV_TRY(sc.get(&krp, W + 1));
        k_lower_bounds_of<uint64_t, int64_t><<<grid_for(W, B), B, 0, st>>>(
            W, P->union_keys, hkey_s, NRH, krp);
        DPV_CHECK_LAUNCH();
        k_i64_to_i32<<<grid_for(W, B), B, 0, st>>>(W, krp, P->key_run_ptr);
        DPV_CHECK_LAUNCH();
    }
    {
        const int32_t nr32 = (int32_t)NRH;
        DPV_CUDA(cudaMemcpyAsync(P->key_run_ptr + W, &nr32, sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
        DPV_CUDA(cudaStreamSynchronize(st));
    }

    ptimer.lap("before 10c. grouped Schur c");
    // 10c. grouped Schur complement: depth rows with identical incidence-var
    // lists (all patches of a frame on a banded graph) form a group whose
    // Schur contribution is one SYRK W_g W_g^T on the tensor cores; chunks of
    // <= rows_per_chunk rows; each key sums its chunk blocks in a fixed order
    P->grouped = 0;
    // Opt-in (DPV_SCHUR_GROUPED=1): at cfg3 the pair-run DMMA kernel is faster
    // (0.42 ms for its Schur part vs SYRK 0.37 + ordered chunk sum 0.11 ms:
    // the SYRK's per-chunk staging is a gather it cannot overlap, and every
    // chunk's blocks make a round trip through memory); it wins for dense
    // var sets.
    if (NPD > 0 && getenv("DPV_SCHUR_GROUPED") && atoi(getenv("DPV_SCHUR_GROUPED")) != 0) {
        uint64_t *rh, *rh_s;
        int32_t *ridx, *flag, *gid, *bad;
        DPV_TRY(sc.get(&rh, NPD));
        DPV_TRY(sc.get(&rh_s, NPD));
        DPV_TRY(sc.get(&ridx, NPD));
        DPV_TRY(P->alloc(&P->g_rows, NPD));
        DPV_TRY(sc.get(&flag, NPD));
        DPV_TRY(sc.get(&gid, NPD));
        DPV_TRY(sc.get(&bad, 1));
        k_row_hash<<<grid_for(NPD, B), B, 0, st>>>(NPD, P->rinc_ptr, P->rinc, P->inc_var, rh, ridx);
        DPV_CHECK_LAUNCH();
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, rh, rh_s, ridx, P->g_rows, (int)NPD, 0, 64,
                                                   st);
        }));
        k_group_flags<<<grid_for(NPD, B), B, 0, st>>>(NPD, rh_s, flag);
        DPV_CHECK_LAUNCH();
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceScan::InclusiveSum(t, b, flag, gid, (int)NPD, st);
        }));
        int32_t ng = 0;
        DPV_CUDA(cudaMemcpyAsync(&ng, gid + NPD - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        // gid is 1-based after the inclusive scan
        k_sub_one<<<grid_for(NPD, B), B, 0, st>>>(NPD, gid);
        DPV_CHECK_LAUNCH();
        int32_t* gstart;
        DPV_TRY(sc.get(&gstart, ng + 1));
        DPV_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
        k_group_verify<<<grid_for(NPD, B), B, 0, st>>>(NPD, flag, gid, P->g_rows, P->rinc_ptr,
                                                        P->rinc, P->inc_var, gstart, bad);
        DPV_CHECK_LAUNCH();
        k_group_verify2<<<grid_for(NPD, B), B, 0, st>>>(NPD, gid, gstart, P->g_rows, P->rinc_ptr,
                                                         P->rinc, P->inc_var, bad);
        DPV_CHECK_LAUNCH();
        // host: group sizes and var counts -> chunks
        std::vector<int32_t> h_gstart(ng), h_rows_head(ng), h_rp;
        DPV_CUDA(cudaMemcpyAsync(h_gstart.data(), gstart, sizeof(int32_t) * ng,
                                 cudaMemcpyDeviceToHost, st));
        int32_t h_bad = 0;
        DPV_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        std::vector<int32_t> h_rows(NPD), h_rinc_ptr(NPD + 1);
        DPV_CUDA(cudaMemcpyAsync(h_rows.data(), P->g_rows, sizeof(int32_t) * NPD,
                                 cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaMemcpyAsync(h_rinc_ptr.data(), P->rinc_ptr, sizeof(int32_t) * (NPD + 1),
                                 cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        if (!h_bad) {
            std::vector<int4> chunks;
            int64_t nblk = 0;
            for (int32_t g = 0; g < ng; ++g) {
                const int32_t b0 = h_gstart[g], b1 = g + 1 < ng ? h_gstart[g + 1] : (int32_t)NPD;
                const int32_t head = h_rows[b0];
                const int m = h_rinc_ptr[head + 1] - h_rinc_ptr[head];
                if (m == 0) continue;
                // staged W: 6m rows + zero rows to a whole 16-row block, x (rows
                // + <= 16 padding) doubles <= kSyrkSmemDoubles
                const int rpc = std::min(kSyrkMaxRows,
                                         ((int)(kSyrkSmemDoubles / (6 * m + 16)) - 16) & ~3);
                if (rpc < 4) { h_bad = 1; break; }
                for (int32_t r0 = b0; r0 < b1; r0 += rpc) {
                    chunks.push_back(make_int4(r0, std::min(rpc, b1 - r0), m, (int)nblk));
                    nblk += (int64_t)m * (m + 1) / 2;
                }
            }
            if (!h_bad && !chunks.empty() && nblk < (int64_t)1 << 30) {
                P->n_chunks = (int64_t)chunks.size();
                P->n_gblocks = nblk;
                DPV_TRY(P->alloc(&P->g_chunks, P->n_chunks));
                DPV_CUDA(cudaMemcpyAsync(P->g_chunks, chunks.data(), sizeof(int4) * chunks.size(),
                                         cudaMemcpyHostToDevice, st));
                uint64_t *ckey, *ckey_s;
                int32_t* cblk;
                DPV_TRY(sc.get(&ckey, nblk));
                DPV_TRY(sc.get(&ckey_s, nblk));
                DPV_TRY(sc.get(&cblk, nblk));
                DPV_TRY(P->alloc(&P->key_blk, nblk));
                k_chunk_contrib<<<(int)std::min<int64_t>(P->n_chunks, 65535), 128, 0, st>>>(
                    P->n_chunks, P->g_chunks, P->g_rows, P->rinc_ptr, P->rinc, P->inc_var,
                    reinterpret_cast<const uint64_t*>(P->union_keys), W, P->n, ckey, cblk);
                DPV_CHECK_LAUNCH();
                DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
                    return cub::DeviceRadixSort::SortPairs(t, b, ckey, ckey_s, cblk, P->key_blk,
                                                           (int)nblk, 0, bits_for(W + 1), st);
                }));
                DPV_TRY(P->alloc(&P->key_blk_ptr, W + 1));
                k_lower_bounds<uint64_t><<<grid_for(W + 1, B), B, 0, st>>>(W, ckey_s, nblk,
                                                                             P->key_blk_ptr);
                DPV_CHECK_LAUNCH();
                DPV_TRY(P->alloc(&P->g_sbuf, nblk * 36));
                P->grouped = 1;
            }
        }
    }

    ptimer.lap("before 11. key -> segment C");
    // 11. key -> segment CSR (pose blocks) and var -> segment CSR (rhs_pose)
    {
        const int64_t n3 = 3 * P->S;
        uint64_t *widx, *widx_s;
        int32_t* hc_s;
        DPV_TRY(sc.get(&widx, n3));
        DPV_TRY(sc.get(&widx_s, n3));
        DPV_TRY(sc.get(&hc_s, n3));
        if (n3 > 0) {
            k_keys_to_union<<<grid_for(n3, B), B, 0, st>>>(n3, hk, P->union_keys, W, widx);
            DPV_CHECK_LAUNCH();
        }
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, widx, widx_s, hc, hc_s, (int)n3, 0, 64,
                                                   st);
        }));
        DPV_TRY(P->alloc(&P->key_seg_ptr, W + 1));
        k_lower_bounds<uint64_t><<<grid_for(W + 1, B), B, 0, st>>>(W, widx_s, n3,
                                                                     P->key_seg_ptr);
        DPV_CHECK_LAUNCH();
        int32_t ks = 0;
        DPV_CUDA(cudaMemcpyAsync(&ks, P->key_seg_ptr + W, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        P->KS = ks;
        DPV_TRY(P->alloc(&P->key_seg, P->KS));
        DPV_CUDA(cudaMemcpyAsync(P->key_seg, hc_s, sizeof(int32_t) * P->KS,
                                 cudaMemcpyDeviceToDevice, st));

        const int64_t n2 = 2 * P->S;
        uint64_t* vk_s;
        int32_t* vc_s;
        DPV_TRY(sc.get(&vk_s, n2));
        DPV_TRY(sc.get(&vc_s, n2));
        DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, vk, vk_s, vc, vc_s, (int)n2, 0, 64, st);
        }));
        DPV_TRY(P->alloc(&P->var_seg_ptr, P->n + 1));
        k_lower_bounds<uint64_t><<<grid_for(P->n + 1, B), B, 0, st>>>(P->n, vk_s, n2,
                                                                        P->var_seg_ptr);
        DPV_CHECK_LAUNCH();
        int32_t vs = 0;
        DPV_CUDA(cudaMemcpyAsync(&vs, P->var_seg_ptr + P->n, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        P->VS = vs;
        DPV_TRY(P->alloc(&P->var_seg, P->VS));
        DPV_CUDA(cudaMemcpyAsync(P->var_seg, vc_s, sizeof(int32_t) * P->VS,
                                 cudaMemcpyDeviceToDevice, st));
    }

    ptimer.lap("before 12. system arrays");
    // 12. system arrays
    DPV_TRY(P->alloc(&P->frame_R, (int64_t)P->F * 9));
    DPV_TRY(P->alloc(&P->e_terms, E * 8));
    DPV_TRY(P->alloc(&P->seg_h, P->S * 21));
    DPV_TRY(P->alloc(&P->seg_g, P->S * 6));
    DPV_TRY(P->alloc(&P->seg_obj, P->S));
    DPV_TRY(P->alloc(&P->depth_diag, NPD));
    DPV_TRY(P->alloc(&P->rhs_depth, NPD));
    DPV_TRY(P->alloc(&P->active, NPD));
    DPV_TRY(P->alloc(&P->cinv0, NPD));
    DPV_TRY(P->alloc(&P->inc_block, I * 6));
    DPV_TRY(P->alloc(&P->uinc, I * 6));
    // [pose_blocks | schur_blocks | rhs_pose | rhs_schur | reduction tail]
    // in ONE allocation: the sharded BA sums the whole pose system over the
    // ranks with a single all-reduce; the tail carries one
    // depth-gradient slot per rank (max folded into the sum)
    DPV_TRY(P->alloc(&P->sysbuf, 2 * W * 36 + 2 * P->n * 6 + dpv::kRedTail));
    P->pose_blocks = P->sysbuf;
    P->schur_blocks = P->pose_blocks + W * 36;
    P->rhs_pose = P->schur_blocks + W * 36;
    P->rhs_schur = P->rhs_pose + P->n * 6;
    P->red_tail = P->rhs_schur + P->n * 6;
    DPV_TRY(P->alloc(&P->scal, 16));
    DPV_TRY(P->alloc(&P->obj_part, kObjBlocks));
    DPV_TRY(P->alloc(&P->red_rhs, P->n * 6 + 8));
    DPV_TRY(P->alloc(&P->cinv, NPD));
    DPV_TRY(P->alloc(&P->status, 8));
    DPV_TRY(P->alloc(&P->lm_q, (int64_t)P->F * 4));
    DPV_TRY(P->alloc(&P->lm_t, (int64_t)P->F * 3));
    DPV_TRY(P->alloc(&P->lm_d, NPD));
    DPV_TRY(P->alloc(&P->lm_dp, P->n * 6));
    DPV_TRY(P->alloc(&P->lm_dd, NPD));
    DPV_TRY(P->alloc(&P->lm_wq, (int64_t)P->F * 4));
    DPV_TRY(P->alloc(&P->lm_wt, (int64_t)P->F * 3));
    DPV_TRY(P->alloc(&P->lm_wd, NPD));
    DPV_TRY(P->alloc(&P->row_flag, NPD));
    DPV_CUDA(cudaMemsetAsync(P->status, 0, sizeof(int32_t) * 8, st));
    P->lm_host = pinned_slot_get();
    DPV_ARG(P->lm_host != nullptr, "pinned host allocation failed");
    DPV_CUDA(cudaStreamSynchronize(st));
    ptimer.lap("12. system arrays");
    return DPV_OK;
}

namespace {
std::mutex g_pin_mu;
std::vector<double*> g_pin_free;
}  // namespace

double* pinned_slot_get() {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.empty()) {
        constexpr int kSlots = 64;
        double* chunk = nullptr;
        if (cudaHostAlloc(reinterpret_cast<void**>(&chunk), sizeof(double) * 16 * kSlots,
                          cudaHostAllocDefault) != cudaSuccess)
            return nullptr;
        for (int k = kSlots - 1; k >= 0; --k) g_pin_free.push_back(chunk + 16 * k);
    }
    double* p = g_pin_free.back();
    g_pin_free.pop_back();
    return p;
}

void pinned_slot_put(double* p) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(p);
}

// Lazily materialised Schur pair list (reference order: key-major, rows
// ascending within a key) for the parity export (ba.py:190-199 maps).
int32_t ensure_pairs(dpv_problem* P) {
    if (P->pair_l || P->NP == 0) return DPV_OK;
    cudaStream_t st = P->alloc_stream;
    const int B = 256;
    int64_t *len64, *off;
    Scratch sc(st);
    DPV_TRY(sc.get(&len64, P->NR + 1));
    DPV_TRY(sc.get(&off, P->NR + 1));
    if (P->NR > 0) {
        k_i32_to_i64<<<grid_for(P->NR, B), B, 0, st>>>(P->NR, P->run_len, len64);
        DPV_CHECK_LAUNCH();
    }
    DPV_CUDA(cudaMemsetAsync(len64 + P->NR, 0, sizeof(int64_t), st));
    DPV_TRY(cub_run(sc, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, len64, off, (int)P->NR + 1, st);
    }));
    DPV_TRY(P->alloc(&P->pair_l, P->NP));
    DPV_TRY(P->alloc(&P->pair_r, P->NP));
    DPV_TRY(P->alloc(&P->key_pair_ptr, P->W + 1));
    if (P->NR > 0) {
        k_expand_runs<<<grid_for(P->NR * 32, B), B, 0, st>>>(P->NR, off, P->run_l, P->run_r,
                                                             P->run_len, P->pair_l, P->pair_r);
        DPV_CHECK_LAUNCH();
    }
    k_key_pair_ptr<<<grid_for(P->W + 1, B), B, 0, st>>>(P->W, P->key_run_ptr, off,
                                                        P->key_pair_ptr);
    DPV_CHECK_LAUNCH();
    DPV_CUDA(cudaStreamSynchronize(st));
    return DPV_OK;
}

}  // namespace dpv
