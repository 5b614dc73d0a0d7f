// Shared device helpers for the CULSH-MF sm_100a kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/culsh.h"

namespace culsh {

constexpr int kWarp = 32;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMix2 = 0x94D049BB133111EBULL;

// Reference: lsh.py:53-58 (_splitmix64), wrapping u64 arithmetic.
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + kGolden;
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
}

// Reference: lsh.py:61-65 (_map_key).
__host__ __device__ __forceinline__ uint64_t map_key(uint64_t seed, int64_t g, int64_t m) {
    uint64_t h = splitmix64(seed);
    h = splitmix64(h ^ ((uint64_t)(g + 1) * kGolden));
    return splitmix64(h ^ ((uint64_t)(m + 1) * kMix1));
}

// Reference: lsh.py:117-123 (_psi); exact same expression tree.
__device__ __forceinline__ double psi_of(double v, int e) {
    if (e == 1) return v;
    if (e == 2) return __dmul_rn(v, v);
    return __dmul_rn(__dmul_rn(v, v), __dmul_rn(v, v));
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_volatile(const int *p) {
    return *(const volatile int *)p;
}

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// True the first time it is called for the current device (per-device bit, thread-safe):
// for per-device state such as cudaFuncSetAttribute or the mempool threshold, which must be
// set again after a set_device to another GPU of the same process.
inline bool first_on_device(std::atomic<uint64_t> &done) {
    const uint64_t bit = 1ull << (current_device() & 63);
    return (done.fetch_or(bit) & bit) == 0;
}

inline int num_sms() {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
    return n > 0 ? n : 148;
}

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default pool; keep
// freed blocks cached in the pool instead of returning them to the driver at every
// synchronisation (release threshold 0 by default), which would re-map memory on each
// call of a frequently called entry point.
inline void keep_pool_memory() {
    static std::atomic<uint64_t> done{0};
    if (first_on_device(done)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
}

inline int status_of(cudaError_t e) { return e == cudaSuccess ? CULSH_OK : CULSH_ECUDA; }

// mbarrier + 1-D bulk copy (TMA engine, non-tensor form) helpers shared by the kernels
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// order this thread's earlier generic-proxy shared accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace culsh

#define CULSH_CHECK(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) {                            \
            culsh_set_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
            return CULSH_ECUDA;                             \
        }                                                   \
    } while (0)

#define CULSH_LAUNCH_CHECK() CULSH_CHECK(cudaGetLastError())

#define CULSH_REQUIRE(cond, msg)                            \
    do {                                                    \
        if (!(cond)) {                                      \
            culsh_set_error(msg, __FILE__, __LINE__);       \
            return CULSH_EINVAL;                            \
        }                                                   \
    } while (0)

void culsh_set_error(const char *msg, const char *file, int line);
