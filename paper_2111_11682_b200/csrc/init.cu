// Parameter initialisation on the device (factorization.py:196-211
// init_params, online.py:187-227 extend_params).
//
// The reference draws U then V from numpy's default_rng(seed).uniform(0, scale, ...):
// PCG64 (XSL-RR 128/64: a 128-bit LCG, state' = state * A + inc, output
// rotr64(hi ^ lo, state' >> 122)), one 64-bit output per element, each turned into
// (out >> 11) * 2^-53 and scaled as 0.0 + scale * u.  Element k of the stream is a pure
// function of the seeded (state, inc) and k, so every thread jumps its 128-bit LCG
// ahead to its own first element (O(log k) multiplies, Brown's algorithm) and then steps
// sequentially: the values are the reference's bit for bit, generated in HBM in well
// under a millisecond instead of ~0.27 s of host numpy at Netflix shape.
#include "common.cuh"

namespace culsh {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

template <typename T>
__global__ void pcg64_uniform_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                                     uint64_t skip, int64_t n, double scale, int per_thread, T *out) {
    const int64_t first = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * per_thread;
    if (first >= n) return;
    const u128 inc = ((u128)i_hi << 64) | i_lo;
    u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, inc, skip + (uint64_t)first);
    const u128 A = pcg_mult();
    const int64_t last = first + per_thread < n ? first + per_thread : n;
    for (int64_t k = first; k < last; ++k) {
        s = s * A + inc;                                   // step, then output (numpy pcg64_next64)
        const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
        out[k] = (T)__dadd_rn(0.0, __dmul_rn(scale, u));   // random_uniform: low + range * u
    }
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                   uint64_t skip, int64_t n, double scale, int fp32, void *out,
                                   void *stream) {
    CULSH_REQUIRE(n >= 0, "n must be nonnegative");
    if (n == 0) return CULSH_OK;
    const int per = 64;
    const int64_t threads = (n + per - 1) / per;
    const int blocks = (int)((threads + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    if (fp32)
        pcg64_uniform_kernel<float><<<blocks, 256, 0, st>>>(state_hi, state_lo, inc_hi, inc_lo, skip, n, scale,
                                                            per, (float *)out);
    else
        pcg64_uniform_kernel<double><<<blocks, 256, 0, st>>>(state_hi, state_lo, inc_hi, inc_lo, skip, n, scale,
                                                             per, (double *)out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// ---- synthetic workload generator (bench / tests; not a reference path) ------------
// Column j of a random_sparse-shaped matrix (datasets.py:147-164: per-column counts,
// distinct uniform rows, stars 1..5) without a host build and without duplicates: its
// c_j rows are the first c_j values of a keyed pseudo-random permutation of [0, M)
// (a 4-round Feistel network on 2^b >= M, cycle-walked into range), so any range of
// columns -- one rank's column shard, or all columns filtered to a row shard -- is
// generated independently and identically on every rank.
namespace culsh {

__device__ __forceinline__ uint64_t feistel(uint64_t x, int half, uint64_t k0, uint64_t k1, uint64_t k2,
                                            uint64_t k3) {
    const uint64_t mh = (1ull << half) - 1;
    uint64_t L = x >> half, R = x & mh;
    const uint64_t ks[4] = {k0, k1, k2, k3};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint64_t nl = R;
        R = L ^ (splitmix64(R ^ ks[r]) & mh);
        L = nl;
    }
    return (L << half) | R;
}

__global__ void synth_columns_kernel(int64_t M, int half, int64_t col_lo, int64_t col_hi, const int64_t *col_ptr,
                                     uint64_t seed, int32_t *rows, double *vals) {
    const int64_t base = col_ptr[col_lo];
    const int64_t total = col_ptr[col_hi] - base;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = base + x;
        int64_t lo = col_lo, hi = col_hi;   // column of entry e
        while (hi - lo > 1) {
            const int64_t m = (lo + hi) >> 1;
            if (col_ptr[m] <= e) lo = m; else hi = m;
        }
        const int64_t j = lo, k = e - col_ptr[j];
        const uint64_t kj = splitmix64(seed ^ ((uint64_t)(j + 1) * kGolden));
        const uint64_t k0 = splitmix64(kj ^ 1), k1 = splitmix64(kj ^ 2), k2 = splitmix64(kj ^ 3),
                       k3 = splitmix64(kj ^ 4);
        uint64_t y = feistel((uint64_t)k, half, k0, k1, k2, k3);
        while (y >= (uint64_t)M) y = feistel(y, half, k0, k1, k2, k3);
        rows[x] = (int32_t)y;
        vals[x] = (double)(1 + splitmix64(kj ^ (y * kMix1) ^ 0x5EED) % 5);
    }
}

}  // namespace culsh

extern "C" int culsh_synth_columns(int64_t M, int64_t col_lo, int64_t col_hi, const int64_t *col_ptr,
                                   uint64_t seed, int32_t *rows, double *vals, void *stream) {
    CULSH_REQUIRE(M >= 1 && M < (1LL << 31), "M out of range");
    if (col_hi <= col_lo) return CULSH_OK;
    int b = 2;
    while ((1LL << b) < M) b += 2;
    const int blocks = num_sms() * 8;
    synth_columns_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(M, b / 2, col_lo, col_hi, col_ptr, seed, rows,
                                                                   vals);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
