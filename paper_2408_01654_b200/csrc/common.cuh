// Shared helpers for the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <exception>
#include <new>
#include <string>

#include "../../include/dpvslam_b200.h"

namespace dpv {

// ---------------------------------------------------------------------------
// error plumbing: never throw across the C ABI

void set_error(const std::string& msg);
void clear_error();
extern std::atomic<int64_t> g_launches;

struct Status {
    int32_t code = DPV_OK;
    bool ok() const { return code == DPV_OK; }
};

#define DPV_CUDA(expr)                                                              \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            (void)cudaGetLastError(); /* a non-sticky error must not resurface */   \
            ::dpv::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) +   \
                             " @ " + __FILE__ + ":" + std::to_string(__LINE__));    \
            return DPV_CUDA_ERROR;                                                  \
        }                                                                           \
    } while (0)

#define DPV_TSTART(name, stream)                                                    \
    do {                                                                            \
        if (::dpv::g_timing) ::dpv::timer_push(name, stream, true);                \
    } while (0)

#define DPV_CHECK_LAUNCH()                                                          \
    do {                                                                            \
        if (::dpv::g_timing) ::dpv::timer_push(nullptr, nullptr, false);           \
        ::dpv::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
        cudaError_t _e = cudaGetLastError();                                        \
        if (_e != cudaSuccess) {                                                    \
            ::dpv::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e) + \
                             " @ " + __FILE__ + ":" + std::to_string(__LINE__));    \
            return DPV_CUDA_ERROR;                                                  \
        }                                                                           \
    } while (0)

#define DPV_TRY(expr)                                                               \
    do {                                                                            \
        int32_t _s = (expr);                                                        \
        if (_s != DPV_OK) return _s;                                                \
    } while (0)

#define DPV_ARG(cond, msg)                                                          \
    do {                                                                            \
        if (!(cond)) {                                                              \
            ::dpv::set_error(msg);                                                  \
            return DPV_BAD_ARGS;                                                    \
        }                                                                           \
    } while (0)

// Every extern "C" entry point runs its body inside DPV_ABI_TRY { ... }
// DPV_ABI_CATCH: a C++ exception (std::bad_alloc from a host vector, a
// std::system_error from a worker thread) becomes a status code and a
// dpv_last_error() message instead of crossing the C ABI.
#define DPV_ABI_TRY try {
#define DPV_ABI_CATCH                                                               \
    }                                                                               \
    catch (const std::bad_alloc&) {                                                 \
        ::dpv::set_error(std::string(__func__) + ": host allocation failed");       \
        return DPV_CUDA_ERROR;                                                      \
    }                                                                               \
    catch (const std::exception& _x) {                                              \
        ::dpv::set_error(std::string(__func__) + ": " + _x.what());                 \
        return DPV_CUDA_ERROR;                                                      \
    }                                                                               \
    catch (...) {                                                                   \
        ::dpv::set_error(std::string(__func__) + ": unknown C++ exception");        \
        return DPV_CUDA_ERROR;                                                      \
    }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Optional per-kernel CUDA-event timing (dpv_timing_*): DPV_TSTART before a
// launch records a start event on the launch stream, the DPV_CHECK_LAUNCH
// that follows records the matching stop event.
extern bool g_timing;
void timer_push(const char* name, cudaStream_t st, bool start);

inline int grid_for(int64_t n, int block, int cap = 148 * 32) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<int>(g);
}

int sm_count();

inline std::mutex& smem_attr_mutex() {
    static std::mutex mu;
    return mu;
}

// raise a kernel's dynamic shared-memory limit to `bytes` (once per growth;
// serialised: batched solves call in from several host threads)
template <typename K>
int32_t ensure_smem(K kernel, size_t bytes, size_t& current) {
    std::lock_guard<std::mutex> lk(smem_attr_mutex());
    if (bytes > current) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)bytes);
        if (e != cudaSuccess) {
            set_error(std::string("cudaFuncSetAttribute(smem ") + std::to_string(bytes) +
                      "): " + cudaGetErrorString(e));
            return DPV_CUDA_ERROR;
        }
        current = bytes;
    }
    return DPV_OK;
}

// ---------------------------------------------------------------------------
// device math

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// quaternion (x,y,z,w) -> row-major rotation; restates geometry.py:70-86
__device__ __forceinline__ void quat_to_rot(const double* q, double* r) {
    const double x = q[0], y = q[1], z = q[2], w = q[3];
    const double xx = x * x, yy = y * y, zz = z * z;
    const double xy = x * y, xz = x * z, yz = y * z;
    const double wx = w * x, wy = w * y, wz = w * z;
    r[0] = 1.0 - 2.0 * (yy + zz);
    r[1] = 2.0 * (xy - wz);
    r[2] = 2.0 * (xz + wy);
    r[3] = 2.0 * (xy + wz);
    r[4] = 1.0 - 2.0 * (xx + zz);
    r[5] = 2.0 * (yz - wx);
    r[6] = 2.0 * (xz - wy);
    r[7] = 2.0 * (yz + wx);
    r[8] = 1.0 - 2.0 * (xx + yy);
}

constexpr double kDepthEps = 1e-8;          // geometry.py:24
constexpr double kInverseDepthFloor = 1e-6; // geometry.py:28
constexpr double kSmallAngle = 1e-8;        // geometry.py:26
constexpr double kActiveEps = 1e-12;        // ba.py:47

}  // namespace dpv
