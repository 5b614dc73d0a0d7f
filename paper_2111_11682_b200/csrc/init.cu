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
