// Hogwild fp32 SGD epoch -- the performance mode of the nonlinear-neighbourhood
// update (paper Alg. 3 CULSH-MF).
//
// One warp owns one column j for a whole epoch: v_j (F floats, FV per lane),
// w_j / c_j (lane k owns k), b_hat_j stay in registers; the column's ratings are
// streamed in CSC order (row, value, explicit-neighbour mask, compact residuals)
// and every update reads and writes the row parameters u_i / b_i in HBM without
// locks (rows are Hogwild, as in Alg. 3).  Per update the warp does one float4
// gather of u_i per lane, one fused warp reduction of
//   u_i.v_j + |R|^-1/2 sum_expl resid*w + |N|^-1/2 sum_impl c
// and one float4 atomic add of the u_i delta (b_i travels with the entry window:
// read when the entry is staged, its update applied when the slot is refilled).
// Columns are handed out through a
// ticket counter in descending-nnz order (longest first) for load balance.
//
// The explicit-neighbour test and residuals depend only on (data, J^K)
// (factorization.py:287-298 with the fixed baselines, :12-16), so they are
// precomputed once per fit (explicit_mask_kernel / explicit_resid_kernel): a K-bit mask per rating
// plus the residuals of the set bits, compacted in (entry, k) order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace culsh {

__device__ __forceinline__ void cp_async_bytes16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_bytes8(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_bytes4(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Paired fp32 arithmetic (sm_100 FFMA2 / FMUL2: two IEEE fp32 ops, each rounded
// exactly like FFMA / FMUL, in one instruction).
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(uint64_t x) { return __uint_as_float((uint32_t)x); }
__device__ __forceinline__ float hi2(uint64_t x) { return __uint_as_float((uint32_t)(x >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// u-row ring slot layout: FV % 4 == 0 stores a lane's floats 4..7, 8..11, ... in further
// 512-byte planes (plane q/4 at +32*q floats), so every 16-byte access of the warp covers
// 512 contiguous bytes (bank-conflict-free); otherwise lane-contiguous FV floats.
template <int FV>
constexpr int ring_lane_stride() { return FV % 4 == 0 ? 4 : FV; }

template <int FV>
__device__ __forceinline__ void cp_async_row(float *dst, const float *src) {
    if constexpr (FV % 4 == 0) {
#pragma unroll
        for (int x = 0; x < FV; x += 4) cp_async_bytes16(dst + 32 * x, src + x);
    } else if constexpr (FV == 4) {
        cp_async_bytes16(dst, src);
    } else if constexpr (FV == 2) {
        cp_async_bytes8(dst, src);
    } else {
        cp_async_bytes4(dst, src);
    }
}

template <int FV>
__device__ __forceinline__ void store_row(float *__restrict__ p, const float (&x)[FV]) {
    if constexpr (FV % 4 == 0 && FV > 8) {
#pragma unroll
        for (int q = 0; q < FV; q += 4)
            *reinterpret_cast<float4 *>(p + q) = make_float4(x[q], x[q + 1], x[q + 2], x[q + 3]);
    } else if constexpr (FV == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
    } else if constexpr (FV == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(x[0], x[1]);
    } else if constexpr (FV == 8) {
        *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
        *reinterpret_cast<float4 *>(p + 4) = make_float4(x[4], x[5], x[6], x[7]);
    } else {
        *p = x[0];
    }
}

template <int FV>
__device__ __forceinline__ void add_row(float *__restrict__ p, const float (&x)[FV], const float (&x0)[FV]) {
    if constexpr (FV == 4) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(x[0] - x0[0], x[1] - x0[1], x[2] - x0[2], x[3] - x0[3]));
    } else if constexpr (FV == 2) {
        atomicAdd(reinterpret_cast<float2 *>(p), make_float2(x[0] - x0[0], x[1] - x0[1]));
    } else if constexpr (FV == 8) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(x[0] - x0[0], x[1] - x0[1], x[2] - x0[2], x[3] - x0[3]));
        atomicAdd(reinterpret_cast<float4 *>(p + 4), make_float4(x[4] - x0[4], x[5] - x0[5], x[6] - x0[6], x[7] - x0[7]));
    } else {
        atomicAdd(p, x[0] - x0[0]);
    }
}

template <int FV>
__device__ __forceinline__ void load_row(const float *__restrict__ p, float (&x)[FV]) {
    if constexpr (FV % 4 == 0 && FV > 8) {
#pragma unroll
        for (int q = 0; q < FV; q += 4) {
            const float4 t = *reinterpret_cast<const float4 *>(p + q);
            x[q] = t.x; x[q + 1] = t.y; x[q + 2] = t.z; x[q + 3] = t.w;
        }
    } else if constexpr (FV == 4) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
    } else if constexpr (FV == 2) {
        const float2 t = *reinterpret_cast<const float2 *>(p);
        x[0] = t.x; x[1] = t.y;
    } else if constexpr (FV == 8) {
        const float4 t0 = *reinterpret_cast<const float4 *>(p);
        const float4 t1 = *reinterpret_cast<const float4 *>(p + 4);
        x[0] = t0.x; x[1] = t0.y; x[2] = t0.z; x[3] = t0.w;
        x[4] = t1.x; x[5] = t1.y; x[6] = t1.z; x[7] = t1.w;
    } else {
        x[0] = *p;
    }
}

// Ring read (layout: ring_lane_stride): one 16-byte ld.shared per 4 floats.  (Left to itself the compiler splits the
// float4 into two 8-byte loads, which at a 16-byte lane stride are 2-way bank-conflicted:
// 8 shared wavefronts per row instead of 4.)
template <int FV>
__device__ __forceinline__ void load_ring(const float *p, float (&x)[FV]) {
    if constexpr (FV % 4 == 0) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(p);
#pragma unroll
        for (int q = 0; q < FV; q += 4)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[q]), "=f"(x[q + 1]), "=f"(x[q + 2]), "=f"(x[q + 3])
                         : "r"(a + 4 * 32 * q));
    } else {
        load_row<FV>(p, x);
    }
}

// Decay factors a = 1 - gamma*lambda of the six rules, so every update is
// x' = a*x + gamma*(gradient term): one FMUL + one FFMA per element.
struct HwCoef {
    float gb, gbh, gu, gv, gw, gc;
    float ab, abh, au, av, aw, ac;
    float abm1;   // ab - 1: the b_i delta is (ab - 1) * b_i + gb * e
};

constexpr int kHwWarps = 8;      // warps per CTA
// u_i prefetch depth (ring slots per warp): 4 for K <= 32, 2 for K > 32 (A/B: C3 11.8 ms at 4
// vs 12.4 at 2 and 12.0 at 8; C5 (K = 64) 35.1 ms at 2 vs 37.2 at 4 and 40.5 at 8 -- the
// smaller ring leaves more of the SM's shared/L1 split to L1)
template <int KPL>
constexpr int hw_depth() { return KPL == 2 ? 2 : 4; }

template <int FV, int KPL>
constexpr int hw_smem_per_warp() {
    // metadata window, mask word 1, u-row ring, b_i and deferred b updates of the window,
    // start values of a work segment
    return 64 * 16 + (KPL == 2 ? 64 * 4 : 0) + hw_depth<KPL>() * 32 * FV * 4 + 2 * 64 * 4 + 32 * (FV + 2 * KPL + 1) * 4;
}

// FV floats per lane; F == 32*FV (vector path) or F < 32 with FV == 1 (masked).
//
// Per warp, shared memory holds (a) the column's next 64 entries' metadata
// {row, value, mask, residual offset} refilled 32 at a time, read with one
// broadcast LDS.128 per update (+ b_i of each entry), and (b) a ring of hw_depth u-rows that
// cp.async fills hw_depth-1 updates ahead, so the HBM/L2 latency of the row
// gather is off the update's critical path.  Each lane copies and later reads
// only its own FV floats of every row, so the ring needs no warp barrier.
//
// PACK: the rating stream is the packed form built by culsh_pack_stream -- one
// u32 per rating {row: bits 0-26, value code: bits 27-30 (into lut), has-mask:
// bit 31} and mask words only for ratings with a set bit (column base mptr[j]),
// 4 + MW*4*(fraction with explicit neighbours) bytes per rating instead of
// 8 + 4*MW.  Whole columns only (no seg); rotation keeps two mask cursors.
//
// P16 (with PACK, no rotation): 2-byte records {row delta from the previous entry of the
// column: 12 bits, value code: 3 bits, has-mask: 1 bit}, rows rebuilt by a warp prefix sum
// from first_row[j]; the per-epoch stream is then 2 + MW*4*(fraction flagged) bytes per
// rating + 4 per column.
template <int FV, int KPL, bool ATOMIC, bool PACK, bool P16>
__global__ void __launch_bounds__(kHwWarps * 32, 4)
hogwild_kernel(int64_t N, const int64_t *__restrict__ col_ptr, const int64_t *__restrict__ seg,
               const int32_t *__restrict__ rows, const float *__restrict__ vals,
               const uint32_t *__restrict__ mask, const int64_t *__restrict__ resid_ptr,
               const float *__restrict__ resid, const int32_t *__restrict__ col_order, float mu,
               float *__restrict__ Bv, float *__restrict__ BHv, float *__restrict__ U,
               float *__restrict__ V, float *__restrict__ W, float *__restrict__ C, int F, int K,
               HwCoef R, int flags, int *__restrict__ ticket, double *__restrict__ loss,
               int *__restrict__ status, const float *__restrict__ lut, const int64_t *__restrict__ mptr,
               const int32_t *__restrict__ first_row) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    constexpr int P = hw_depth<KPL>();
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    unsigned char *wbase = s_raw + (size_t)warp * hw_smem_per_warp<FV, KPL>();
    int4 *s_meta = reinterpret_cast<int4 *>(wbase);                           // 64 x 16 B
    uint32_t *s_m1 = reinterpret_cast<uint32_t *>(wbase + 64 * 16);           // KPL == 2
    float *s_ring = reinterpret_cast<float *>(wbase + 64 * 16 + (KPL == 2 ? 64 * 4 : 0));
    float *s_b = s_ring + P * 32 * FV;   // b_i of the staged entries (cp.async at chunk load)
    float *s_db = s_b + 64;               // their b updates, applied when the slot is refilled
    float *my_ring = s_ring + lane * ring_lane_stride<FV>();
    float *my_start = s_db + 64 + lane * (FV + 2 * KPL + 1);   // this lane's segment start values

    const bool fl = FV > 1 || (int)lane < F;   // lane owns factor slots (F == 32*FV when FV > 1)
    const unsigned lt_mask = (1u << lane) - 1u;
    const float invK = K > 0 ? rsqrtf((float)K) : 0.f;
    float kgc[KPL];   // gc * |N|^-1/2 with |N| = K (no explicit neighbour), 0 for slots >= K
#pragma unroll
    for (int q = 0; q < KPL; ++q) kgc[q] = (int)lane + 32 * q < K ? R.gc * invK : 0.f;
    s_meta[lane] = make_int4(0, 0, 0, 0);   // every row index the prefetch can see is valid
    s_meta[lane + 32] = make_int4(0, 0, 0, 0);
    __syncwarp();
    double col_loss = 0.0;
    int bad = 0;
    const float *Ulane = U + lane * FV;
    // (a constant-stride IMAD.WIDE row address -- 40 fewer SASS instructions, 56 registers --
    // measured 11.5 ms for 5 epochs then a steady 12.2 ms against 11.7 ms, A/B on one box:
    // not kept)
    auto urow_of = [&](int ip) -> float * { return U + (size_t)(unsigned)ip * (unsigned)F + lane * FV; };

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= N) break;
        const int64_t j = col_order ? (int64_t)col_order[t] : (int64_t)t;

        float v[FV];
        if (fl) load_row<FV>(V + j * F + lane * FV, v);
        else {
#pragma unroll
            for (int x = 0; x < FV; ++x) v[x] = 0.f;
        }
        float w[KPL], c[KPL];
        bool kin[KPL];
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            kin[q] = k < K;
            w[q] = kin[q] ? W[j * K + k] : 0.f;
            c[q] = kin[q] ? C[j * K + k] : 0.f;
        }
        float bh = BHv[j];
        const int64_t c_lo = col_ptr[j], c_hi = col_ptr[j + 1];
        // entry range: per-ticket work segment (flags bit 3), per-column DSGD block, or the column;
        // flags bit 4: work segments carry precomputed stream cursors at lo (stride 4:
        // lo, hi | S << 40, compact-mask slot, residual offset | P16 row carry << 32)
        const int sstride = (flags & 16) ? 4 : 2;
        const int64_t lo = seg ? seg[(flags & 8) ? sstride * (int64_t)t : 2 * j] : c_lo;
        int64_t hi = seg ? seg[(flags & 8) ? sstride * (int64_t)t + 1 : 2 * j + 1] : c_hi;
        // a work segment that is only part of its column runs concurrently with the column's
        // other S segments (S in bits 40-63 of its end): its column parameters are merged
        // back as atomic adds of (change / S) -- the average of the segments' changes
        const int nparts = (flags & 8) ? (int)((uint64_t)hi >> 40) : 1;
        hi &= (int64_t)0xFFFFFFFFFFLL;
        const int n = (int)(hi - lo);
        const bool part_col = nparts > 1;
        const float inv_parts = 1.f / (float)max(nparts, 1);
        if (part_col) {   // start values, for the deltas merged at the end (lane-private slots)
#pragma unroll
            for (int x = 0; x < FV; ++x) my_start[x] = v[x];
#pragma unroll
            for (int q = 0; q < KPL; ++q) { my_start[FV + q] = w[q]; my_start[FV + KPL + q] = c[q]; }
            my_start[FV + 2 * KPL] = bh;
        }
        const float *rcol = resid + resid_ptr[j];
        const uint16_t *p16 = reinterpret_cast<const uint16_t *>(rows);
        int carry = 0;   // P16: row of the entry before the next chunk
        if constexpr (P16) carry = first_row[j];
        // packed: next compact mask slot of the rotated range's segment 1 ([rot, n)) / 2 ([0, rot))
        int64_t mrun1 = PACK ? mptr[j] : 0, mrun2 = mrun1;
        // Visiting order: the column's entries rotated to start at position `rot`
        // (a per-column hash when `rotate` is set).  Warps then sweep the rows out of
        // phase with each other instead of in lock-step, which keeps concurrent
        // Hogwild writes to the same u_i rare.
        const int rot = ((flags & 1) && n > 1) ? (int)(splitmix64((uint64_t)j ^ 0x5bd1e995ULL) % (uint64_t)n) : 0;
        int rrel2 = 0;   // residual offset (relative to the column base) at position lo
        if ((flags & 16) && lo > c_lo) {   // cursors from the plan (segment_cursors_kernel)
            const int64_t c3 = seg[sstride * (int64_t)t + 3];
            if constexpr (PACK) {
                mrun2 = seg[sstride * (int64_t)t + 2];
                mrun1 = mrun2;
            }
            rrel2 = (int)(uint32_t)(uint64_t)c3;
            if constexpr (P16) carry = (int)((uint64_t)c3 >> 32);
        } else if (PACK && lo > c_lo) {   // work segment: mask cursor and residual offset at lo
            int h = 0, dsum = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = c_lo + lane; x < lo; x += 32) {
                if constexpr (P16) {
                    const uint32_t w16 = __ldg(p16 + x);
                    h += (int)(w16 >> 15);
                    dsum += (int)(w16 & 0xFFFu);
                } else {
                    h += (int)(__ldg(reinterpret_cast<const uint32_t *>(rows) + x) >> 31);
                }
            }
            h = warp_sum(h);
            if constexpr (P16) carry += warp_sum(dsum);
            int skip = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = mrun2 + lane; x < mrun2 + h; x += 32)
#pragma unroll
                for (int q = 0; q < KPL; ++q) skip += __popc(mask[x * KPL + q]);
            mrun2 += h;
            mrun1 = mrun2;
            rrel2 = warp_sum(skip);
        } else if (lo > c_lo) {   // DSGD block: skip the residuals of the column's earlier row blocks
            int skip = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = c_lo + lane; x < lo; x += 32)
#pragma unroll
                for (int q = 0; q < KPL; ++q) skip += __popc(mask[x * KPL + q]);
            rrel2 = warp_sum(skip);
        }
        int rrel1 = rrel2;   // ... at position lo + rot
        if (PACK && rot > 0) {
            int h = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = lo + lane; x < lo + rot; x += 32)
                h += (int)(__ldg(reinterpret_cast<const uint32_t *>(rows) + x) >> 31);
            h = warp_sum(h);
            int skip = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = mrun2 + lane; x < mrun2 + h; x += 32)
#pragma unroll
                for (int q = 0; q < KPL; ++q) skip += __popc(mask[x * KPL + q]);
            mrun1 += h;
            rrel1 += warp_sum(skip);
        } else if (rot > 0) {
            int skip = 0;
#pragma unroll 8   // independent loads: keep several in flight
            for (int64_t x = lo + lane; x < lo + rot; x += 32)
#pragma unroll
                for (int q = 0; q < KPL; ++q) skip += __popc(mask[x * KPL + q]);
            rrel1 += warp_sum(skip);
        }

        // stage 32 entries' metadata (+ exclusive prefix of explicit counts); processing
        // index k maps to position (k + rot) mod n, i.e. segment 1 = [rot, n), segment 2 = [0, rot).
        // Packed streams stage a chunk in three steps one chunk (32 updates) apart, so no
        // step waits on a global load: fetch_word issues the record load, decode turns the
        // record into row / value / mask cursor and issues the mask-word and value loads,
        // stage_chunk writes the window slot (the chunk-level waits were 8 % of the stall
        // samples when the three ran back to back).
        struct Dec {
            int ri;
            float rv;
            uint32_t m0, m1;
        };
        auto chunk_pos = [&](int ch, bool &have, bool &seg2) -> int64_t {
            const int k = 32 * ch + (int)lane;
            have = k < n;
            int pos = k + rot;
            seg2 = pos >= n;
            if (seg2) pos -= n;
            return lo + pos;
        };
        auto fetch_word = [&](int ch) -> uint32_t {
            if constexpr (PACK) {
                bool have, seg2;
                const int64_t e = chunk_pos(ch, have, seg2);
                if constexpr (P16) return have ? (uint32_t)__ldg(p16 + e) : 0u;
                else return have ? __ldg(reinterpret_cast<const uint32_t *>(rows) + e) : 0u;
            } else {
                return 0u;
            }
        };
        auto decode = [&](int ch, uint32_t wd_in) -> Dec {
            bool have, seg2;
            const int64_t e = chunk_pos(ch, have, seg2);
            int ri;
            float rv;
            uint32_t m0 = 0u, m1 = 0u;
            if constexpr (PACK) {
                uint32_t code;
                bool hm;
                if constexpr (P16) {
                    const uint32_t w16 = wd_in;
                    int incl = (int)(w16 & 0xFFFu);
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if ((int)lane >= o) incl += y;
                    }
                    ri = carry + incl;   // lanes past the end repeat the last row (a valid row)
                    carry = __shfl_sync(0xffffffffu, ri, 31);
                    code = (w16 >> 12) & 7u;
                    hm = (w16 >> 15) != 0u;
                } else {
                    const uint32_t wd = wd_in;
                    ri = (int)(wd & 0x07FFFFFFu);
                    code = (wd >> 27) & 15u;
                    hm = (wd >> 31) != 0u;
                }
                rv = __ldg(lut + code);
                const unsigned b1 = __ballot_sync(0xffffffffu, hm && !seg2);
                const unsigned b2 = __ballot_sync(0xffffffffu, hm && seg2);
                if (hm) {
                    const int64_t mi = seg2 ? mrun2 + __popc(b2 & lt_mask) : mrun1 + __popc(b1 & lt_mask);
                    m0 = mask[mi * KPL];
                    if constexpr (KPL == 2) m1 = mask[mi * KPL + 1];
                }
                mrun1 += __popc(b1);
                mrun2 += __popc(b2);
            } else {
                ri = have ? rows[e] : 0;
                rv = have ? vals[e] : 0.f;
                m0 = have ? mask[e * KPL] : 0u;
                m1 = (KPL == 2 && have) ? mask[e * KPL + 1] : 0u;
            }
            return Dec{ri, rv, m0, m1};
        };
        auto stage_chunk = [&](int ch, const Dec &d) {
            bool have, seg2;
            chunk_pos(ch, have, seg2);
            const int ri = d.ri;
            const uint32_t m0 = d.m0, m1 = d.m1;
            const int pc = __popc(m0) + __popc(m1);
            int roff = 0;
            if (__any_sync(0xffffffffu, pc != 0)) {
                int incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += y;
                }
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                const int tot1 = warp_sum((have && !seg2) ? pc : 0);
                roff = seg2 ? rrel2 + (incl - pc - tot1) : rrel1 + (incl - pc);
                rrel1 += tot1;
                rrel2 += tot - tot1;
            }
            const int slot = (32 * ch + lane) & 63;
            s_meta[slot] = make_int4(ri, __float_as_int(d.rv), (int)m0, roff);
            if constexpr (KPL == 2) s_m1[slot] = m1;
            cp_async_bytes4(s_b + slot, Bv + ri);   // lands with the next committed group
        };
        // b_i is read when its entry is staged (32-64 updates ahead) and its update is
        // applied when the slot is refilled: one gather and one atomic per lane per 32
        // updates instead of a lane-0 copy and atomic per update (Hogwild staleness)
        auto flush_b = [&](int first, int count) {
            if ((int)lane < count) {
                const int slot = (first + (int)lane) & 63;
                const int ib = s_meta[slot].x;
                if constexpr (ATOMIC) atomicAdd(Bv + ib, s_db[slot]);
                else Bv[ib] = s_db[slot];
            }
        };
        auto issue = [&](int tp) {
            const int ip = s_meta[tp & 63].x;
            float *dst = my_ring + (tp % P) * 32 * FV;
            if (fl) cp_async_row<FV>(dst, Ulane + (size_t)(unsigned)ip * (unsigned)F);
        };

        // pipeline registers: pd = the decoded chunk staged next, pwd = the record word of the
        // chunk decoded next
        Dec pd{0, 0.f, 0u, 0u};
        uint32_t pwd = 0u;
        {
            const uint32_t w0 = fetch_word(0);
            const uint32_t w1 = n > 32 ? fetch_word(1) : 0u;
            const uint32_t w2 = n > 64 ? fetch_word(2) : 0u;
            stage_chunk(0, decode(0, w0));
            if (n > 32) stage_chunk(1, decode(1, w1));
            if (n > 64) {
                pd = decode(2, w2);
                if (n > 96) pwd = fetch_word(3);
            }
        }
        __syncwarp();
#pragma unroll
        for (int p = 0; p < P - 1; ++p) {
            if (p < n) issue(p);
            cp_async_commit();
        }
        float lossf = 0.f;
        const float ngu = -R.gu * (1.f - R.au) / R.gu;   // = -(gu*lu): delta_u = ngu*u + gu*e*v
        // one update: entry in metadata slot ms / ring slot rsl; prefetch of the entry P-1
        // ahead (slots pms / prs)
        auto step = [&](const int ms, const int pms, const int rsl, const int prs) {
            // prefetch P-1 ahead.  Past the column's end the slot holds a padding (0) or an
            // older row of this launch (s_meta is zeroed at entry): always a valid row, the
            // copy lands in a ring slot nobody reads before the column's final wait.
            {
                const int ip = s_meta[pms].x;
                float *dst = my_ring + prs * 32 * FV;
                if (fl) cp_async_row<FV>(dst, Ulane + (size_t)(unsigned)ip * (unsigned)F);
            }
            cp_async_commit();
            cp_async_wait<P - 1>();
            const int4 me = s_meta[ms];
            const int i = me.x;
            const float r = __int_as_float(me.y);
            const uint32_t m0 = (uint32_t)me.z;
            const uint32_t m1 = KPL == 2 ? s_m1[ms] : 0u;
            float u[FV];
            load_ring<FV>(my_ring + rsl * 32 * FV, u);
            if constexpr (FV == 1) {
                if (!fl) u[0] = 0.f;   // lanes >= F never fill their ring slot (garbage, maybe NaN)
            }
            const float bi = s_b[ms];
            float part;
            if constexpr (FV % 2 == 0) {
                // paired fp32 (FFMA2): even / odd factor partial sums, folded once
                uint64_t acc = pack2(0.f, 0.f);
#pragma unroll
                for (int x = 0; x < FV; x += 2) acc = ffma2(pack2(u[x], u[x + 1]), pack2(v[x], v[x + 1]), acc);
                part = lo2(acc) + hi2(acc);
            } else {
                part = 0.f;
#pragma unroll
                for (int x = 0; x < FV; ++x) part = fmaf(u[x], fl ? v[x] : 0.f, part);
            }
            const bool anyex = (m0 | m1) != 0u;   // warp-uniform
            float inv_r = 0.f, inv_n = invK;
            float rs[KPL];
            bool ex[KPL];
            if (!anyex) {
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    ex[q] = false;
                    rs[q] = 0.f;
                    part = fmaf(c[q], invK, part);
                }
            } else {
                const int nr = __popc(m0) + __popc(m1);
                const int nn = K - nr;
                inv_r = rsqrtf((float)nr);
                inv_n = nn > 0 ? rsqrtf((float)nn) : 0.f;
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    const uint32_t mq = q == 0 ? m0 : m1;
                    ex[q] = (mq >> lane) & 1u;
                    const int rank = (q == 0 ? 0 : __popc(m0)) + __popc(mq & lt_mask);
                    rs[q] = ex[q] ? rcol[me.w + rank] : 0.f;
                    part += ex[q] ? rs[q] * w[q] * inv_r : c[q] * inv_n;
                }
            }
            // warp sum: 2^-20 fixed point through one redux.sync while every lane's partial is
            // inside +-32 (always, for a model that has not diverged: the partials are O(1));
            // the quantisation (<= 32 * 2^-21 on the sum) is far below the fp32 SGD noise.
            // Otherwise the fp32 shuffle tree, so overflow and non-finite values still surface.
            if (!__any_sync(0xffffffffu, !(fabsf(part) < 32.f)))
                part = (float)__reduce_add_sync(0xffffffffu, __float2int_rn(part * 1048576.f)) * (1.f / 1048576.f);
            else
                part = warp_sum(part);
            const float e = r - (mu + bh + bi + part);
            lossf = fmaf(e, e, lossf);
            // fused update of every touched parameter (factorization.py:307-328 rules)
            const float geu = R.gu * e, gev = R.gv * e;
            float *urow = urow_of(i);
            if constexpr (ATOMIC) {
                // add the update instead of storing the new value: a concurrent update of the
                // same row by another warp is then never lost (only computed from a stale u_i)
                float dlt[FV];
                if constexpr (FV % 2 == 0) {
                    const uint64_t ngu2 = pack2(ngu, ngu), geu2 = pack2(geu, geu);
                    const uint64_t av2 = pack2(R.av, R.av), gev2 = pack2(gev, gev);
#pragma unroll
                    for (int x = 0; x < FV; x += 2) {
                        const uint64_t uo = pack2(u[x], u[x + 1]), vo = pack2(v[x], v[x + 1]);
                        const uint64_t d = ffma2(ngu2, uo, fmul2(geu2, vo));
                        const uint64_t vn = ffma2(av2, vo, fmul2(gev2, uo));
                        dlt[x] = lo2(d); dlt[x + 1] = hi2(d);
                        v[x] = lo2(vn); v[x + 1] = hi2(vn);
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < FV; ++x) {
                        const float uo = u[x];
                        dlt[x] = fmaf(ngu, uo, geu * v[x]);
                        v[x] = fmaf(R.av, v[x], gev * uo);
                    }
                }
                if (fl) {
                    if constexpr (FV % 4 == 0) {
#pragma unroll
                        for (int x = 0; x < FV; x += 4)
                            atomicAdd(reinterpret_cast<float4 *>(urow + x),
                                      make_float4(dlt[x], dlt[x + 1], dlt[x + 2], dlt[x + 3]));
                    } else if constexpr (FV == 2) {
                        atomicAdd(reinterpret_cast<float2 *>(urow), make_float2(dlt[0], dlt[1]));
                    } else {
                        atomicAdd(urow, dlt[0]);
                    }
                }
                s_db[ms] = fmaf(R.abm1, bi, R.gb * e);   // same value from every lane
            } else {
#pragma unroll
                for (int x = 0; x < FV; ++x) {
                    const float uo = u[x];
                    u[x] = fmaf(R.au, uo, geu * v[x]);
                    v[x] = fmaf(R.av, v[x], gev * uo);
                }
                if (fl) store_row<FV>(urow, u);
                s_db[ms] = fmaf(R.ab, bi, R.gb * e);
            }
            bh = fmaf(R.abh, bh, R.gbh * e);
            if (!anyex) {
                // no explicit neighbour: only the implicit weights move (kgc = 0 off K)
#pragma unroll
                for (int q = 0; q < KPL; ++q) c[q] = fmaf(R.ac, c[q], kgc[q] * e);
            } else {
                const float gce = R.gc * inv_n * e, gwe = R.gw * inv_r * e;
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    const float wn = fmaf(R.aw, w[q], gwe * rs[q]);
                    const float cn = fmaf(R.ac, c[q], gce);
                    w[q] = (kin[q] && ex[q]) ? wn : w[q];
                    c[q] = (kin[q] && !ex[q]) ? cn : c[q];
                }
            }
        };
        for (int base = 0; base < n; base += 32) {
            if (base > 0) {
                __syncwarp();   // every lane is done with the half being refilled
                flush_b(base - 32, 32);
                if (base + 32 < n) {
                    const int c = (base >> 5) + 1;
                    stage_chunk(c, pd);
                    if (32 * (c + 1) < n) {
                        pd = decode(c + 1, pwd);
                        if (32 * (c + 2) < n) pwd = fetch_word(c + 2);
                    }
                }
                __syncwarp();
            }
            const int cnt = min(32, n - base);
            if (FV <= 4 && cnt == 32) {
                // whole chunk: P-update groups with compile-time ring slots (base % 32 == 0);
                // FV == 8 keeps the rolled loop (register budget of 4 CTAs per SM)
                // updates per unrolled group (a multiple of P): P for K <= 32; 8 for K > 32
                // (2-deep ring), where it measured 34.6 -> 33.6 ms at C5 (and 4 -> 8 at C3: slower)
                constexpr int GS = KPL == 2 ? 8 : P;
                static_assert(32 % GS == 0 && GS % P == 0, "group must divide the chunk, ring the group");
                for (int k = 0; k < 32; k += GS) {
                    const int g0 = (base + k) & 63, g1 = (base + k + GS) & 63;
#pragma unroll
                    for (int s = 0; s < GS; ++s) {
                        const int t = s + P - 1;   // prefetch offset inside / past the group
                        step(g0 + s, t < GS ? g0 + t : g1 + (t - GS), s % P, t % P);
                    }
                }
            } else {
                for (int k = 0; k < cnt; ++k) {
                    const int tt = base + k;
                    step(tt & 63, (tt + P - 1) & 63, tt % P, (tt + P - 1) % P);
                }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
        if (n > 0) flush_b(((n - 1) >> 5) << 5, n - (((n - 1) >> 5) << 5));
        if (!isfinite(lossf)) bad = 1;
        col_loss += (double)lossf;
        if (!part_col) {
            if (fl) store_row<FV>(V + j * F + lane * FV, v);
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                if (kin[q]) {
                    W[j * K + k] = w[q];
                    C[j * K + k] = c[q];
                }
            }
            if (lane == 0) BHv[j] = bh;
        } else {
            float vd[FV], zero[FV];
#pragma unroll
            for (int x = 0; x < FV; ++x) {
                vd[x] = (v[x] - my_start[x]) * inv_parts;
                zero[x] = 0.f;
            }
            if (fl) add_row<FV>(V + j * F + lane * FV, vd, zero);
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                if (kin[q]) {
                    atomicAdd(W + j * K + k, (w[q] - my_start[FV + q]) * inv_parts);
                    atomicAdd(C + j * K + k, (c[q] - my_start[FV + KPL + q]) * inv_parts);
                }
            }
            if (lane == 0) atomicAdd(BHv + j, (bh - my_start[FV + 2 * KPL]) * inv_parts);
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (loss) atomicAdd(loss, col_loss);
        if (bad) atomicOr(status, 1);
    }
}

// ---- explicit-neighbour stream (one pass per fit) ---------------------------

__device__ __forceinline__ int64_t find_row(const int32_t *__restrict__ rows, int64_t lo, int64_t hi,
                                            int32_t i) {
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        const int32_t x = __ldg(rows + m);
        if (x == i) return m;
        if (x < i) lo = m + 1; else hi = m;
    }
    return -1;
}

template <int FV, int KPL, bool PACK = false, bool P16 = false>
int launch_hogwild(int64_t N, const int64_t *col_ptr, const int64_t *seg, const int32_t *rows, const float *vals,
                   const uint32_t *mask, const int64_t *resid_ptr, const float *resid,
                   const int32_t *col_order, CulshModel32 *m, const HwCoef &R, int flags, int max_warps,
                   int *ticket,
                   double *loss, int *status, cudaStream_t st, const float *lut = nullptr,
                   const int64_t *mptr = nullptr, const int32_t *first_row = nullptr) {
    const int threads = kHwWarps * 32;
    const size_t smem = (size_t)kHwWarps * hw_smem_per_warp<FV, KPL>();
    {   // per device and cheap: set on every launch (a once-per-process flag breaks on a 2nd GPU)
        cudaFuncSetAttribute(hogwild_kernel<FV, KPL, true, PACK, P16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(hogwild_kernel<FV, KPL, false, PACK, P16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    int occ = 0;
    auto kern = (flags & 2) ? hogwild_kernel<FV, KPL, true, PACK, P16> : hogwild_kernel<FV, KPL, false, PACK, P16>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (occ < 1) occ = 1;
    int64_t blocks = (int64_t)num_sms() * occ;
    const int64_t need = (N + kHwWarps - 1) / kHwWarps;
    if (blocks > need) blocks = need;
    if (max_warps > 0 && blocks > (max_warps + kHwWarps - 1) / kHwWarps)
        blocks = (max_warps + kHwWarps - 1) / kHwWarps;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, threads, smem, st>>>(
        N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m->mu, m->b, m->bhat, m->U, m->V, m->W,
        m->C, m->F, m->K, R, flags, ticket, loss, status, lut, mptr, first_row);
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

// ---- packed rating stream (see hogwild_kernel PACK) ---------------------------
//
// Warp per column, entries in CSC order.  Pass 1 (packed == nullptr): per-column
// count of ratings whose mask is non-zero.  Pass 2: packed words + compact mask
// words at mptr[j] in entry order.  A value missing from lut or a row >= 2^27
// sets *status |= 4 (the caller then keeps the wide stream).
__global__ void pack_stream_kernel(int64_t N, const int64_t *__restrict__ col_ptr,
                                   const int32_t *__restrict__ rows, const float *__restrict__ vals,
                                   const uint32_t *__restrict__ mask, int MW, const float *__restrict__ lut,
                                   int n_lut, uint32_t *__restrict__ packed, int64_t *__restrict__ mcount,
                                   const int64_t *__restrict__ mptr, uint32_t *__restrict__ cmask,
                                   int *__restrict__ status) {
    const unsigned lane = lane_id();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < N; j += warps) {
        const int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        int64_t run = packed ? mptr[j] : 0;
        int bad = 0;
        for (int64_t b = lo; b < hi; b += 32) {
            const int64_t e = b + lane;
            const bool have = e < hi;
            uint32_t m0 = 0u, m1 = 0u;
            if (have) {
                m0 = mask[e * MW];
                if (MW == 2) m1 = mask[e * MW + 1];
            }
            const bool hm = (m0 | m1) != 0u;
            const unsigned bal = __ballot_sync(0xffffffffu, hm);
            if (packed && have) {
                const float v = vals[e];
                int code = -1;
                for (int c = 0; c < n_lut; ++c)
                    if (lut[c] == v) { code = c; break; }
                const int32_t r = rows[e];
                if (code < 0 || r < 0 || r >= (1 << 27)) bad = 1;
                packed[e] = ((uint32_t)r & 0x07FFFFFFu) | ((uint32_t)(code & 15) << 27) | (hm ? 0x80000000u : 0u);
                if (hm) {
                    const int64_t mi = run + __popc(bal & lt_mask);
                    cmask[mi * MW] = m0;
                    if (MW == 2) cmask[mi * MW + 1] = m1;
                }
            }
            run += __popc(bal);
        }
        if (!packed && lane == 0) mcount[j] = run;
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 4);
    }
}

// 2-byte packed records (see hogwild_kernel P16): warp per column, delta from the
// previous entry's row (0 for the first, whose row goes to first_row[j]); *status |= 4
// when a delta needs more than 12 bits or a value more than 3 code bits.  The mask
// words of the flagged entries are those of culsh_pack_stream (cmask, mptr).
__global__ void pack16_kernel(int64_t N, const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ rows,
                              const float *__restrict__ vals, const uint32_t *__restrict__ mask, int MW,
                              const float *__restrict__ lut, int n_lut, uint16_t *__restrict__ words,
                              int32_t *__restrict__ first_row, int *__restrict__ status) {
    const unsigned lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < N; j += warps) {
        const int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        if (lane == 0) first_row[j] = hi > lo ? rows[lo] : 0;
        int bad = 0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int32_t r = rows[e];
            const int32_t prev = e > lo ? rows[e - 1] : r;
            const int delta = r - prev;
            const float v = vals[e];
            int code = -1;
            for (int c = 0; c < n_lut; ++c)
                if (lut[c] == v) { code = c; break; }
            uint32_t m = mask[e * MW];
            if (MW == 2) m |= mask[e * MW + 1];
            if (code < 0 || code > 7 || delta < 0 || delta > 0xFFF) bad = 1;
            words[e] = (uint16_t)((delta & 0xFFF) | ((code & 7) << 12) | (m ? 0x8000u : 0u));
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 4);
    }
}

}  // namespace culsh

using namespace culsh;

// Explicit-neighbour stream, intersection form.  Pass 1: one warp per (column j,
// neighbour slot k) intersects j's sorted row list with J[j,k]'s by a sliced merge
// (lane l owns the l-th 32nd of j's entries, finds its start in J's list by one binary
// search, then advances linearly): O(n_j + n_J) per pair instead of n_j binary searches;
// hits set bit k of the entry's mask word (atomicOr) and count into col_nexpl[j].
// Pass 2: one warp per column, residual slots from a warp scan of the entries'
// popcounts, one binary search per explicit pair for r(i, J).  (Replaces a CTA-per-
// column kernel with nnz*K global binary searches: 2 x 26 ms at C3.)
__global__ void explicit_mask_kernel(CulshData d, const int32_t *__restrict__ nbr, int K, int MW,
                                     uint32_t *__restrict__ mask, unsigned long long *__restrict__ col_nexpl) {
    const unsigned lane = lane_id();
    const int64_t pairs = d.N * (int64_t)K;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < pairs; w += warps) {
        const int64_t j = w / K;
        const int k = (int)(w % K);
        const int64_t a0 = d.col_ptr[j], nA = d.col_ptr[j + 1] - a0;
        const int32_t J = nbr[j * K + k];
        const int64_t b0 = d.col_ptr[J], nB = d.col_ptr[J + 1] - b0;
        const int32_t *A = d.col_rows + a0;
        const int32_t *B = d.col_rows + b0;
        const int64_t s0 = nA * lane / 32, s1 = nA * (lane + 1) / 32;
        int matches = 0;
        if (s0 < s1 && nB > 0) {
            const int32_t x0 = __ldg(A + s0);
            int64_t lo = 0, hi = nB;   // lower_bound(B, x0)
            while (lo < hi) {
                const int64_t m = (lo + hi) >> 1;
                if (__ldg(B + m) < x0) lo = m + 1; else hi = m;
            }
            int64_t bp = lo;
            int32_t bv = bp < nB ? __ldg(B + bp) : INT32_MAX;
            for (int64_t a = s0; a < s1 && bp < nB; ++a) {
                const int32_t xa = __ldg(A + a);
                while (bv < xa) {
                    ++bp;
                    bv = bp < nB ? __ldg(B + bp) : INT32_MAX;
                }
                if (bv == xa) {
                    atomicOr(mask + (a0 + a) * MW + (k >> 5), 1u << (k & 31));
                    ++matches;
                }
            }
        }
        matches = warp_sum(matches);
        if (lane == 0 && matches) atomicAdd(col_nexpl + j, (unsigned long long)matches);
    }
}

// Stream cursors at the start of every work segment (once per plan; the epoch kernel with
// flags bit 4 reads them instead of scanning from its column's start every epoch -- that scan
// made late DSGD stages, whose segments start deep in their columns, the slowest).  The same
// arithmetic as the kernel's scan: number of flagged entries before lo (compact-mask slot),
// popcount of their masks (residual offset), and for 2-byte records the row before lo.
__global__ void segment_cursors_kernel(int64_t n_list, const int64_t *__restrict__ col_ptr,
                                       const int32_t *__restrict__ col_order, const int64_t *__restrict__ seg2,
                                       const uint32_t *__restrict__ words, const uint16_t *__restrict__ w16,
                                       const int32_t *__restrict__ first_row, const int64_t *__restrict__ mptr,
                                       const uint32_t *__restrict__ mask, int MW, int64_t *__restrict__ seg4) {
    const unsigned lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < n_list; t += warps) {
        const int64_t j = col_order[t];
        const int64_t lo = seg2[2 * t], hi = seg2[2 * t + 1];
        const int64_t c_lo = col_ptr[j];
        int h = 0, dsum = 0, skip = 0;
        int64_t m0 = mptr ? mptr[j] : 0;
        if (mptr) {   // packed: flagged entries before lo, then their compact mask words
            for (int64_t x = c_lo + lane; x < lo; x += 32) {
                if (w16) {
                    const uint32_t v = w16[x];
                    h += (int)(v >> 15);
                    dsum += (int)(v & 0xFFFu);
                } else {
                    h += (int)(words[x] >> 31);
                }
            }
            h = warp_sum(h);
            for (int64_t x = m0 + lane; x < m0 + h; x += 32)
                for (int q = 0; q < MW; ++q) skip += __popc(mask[x * MW + q]);
        } else {      // wide stream: a mask word (pair) per entry
            for (int64_t x = c_lo + lane; x < lo; x += 32)
                for (int q = 0; q < MW; ++q) skip += __popc(mask[x * MW + q]);
        }
        skip = warp_sum(skip);
        dsum = warp_sum(dsum);
        if (lane == 0) {
            seg4[4 * t] = lo;
            seg4[4 * t + 1] = hi;
            seg4[4 * t + 2] = m0 + h;
            const uint32_t carry = w16 ? (uint32_t)(first_row[j] + dsum) : 0u;
            seg4[4 * t + 3] = (int64_t)(((uint64_t)carry << 32) | (uint32_t)skip);
        }
    }
}

// Row-major explicit-neighbour test (once per fit; replaces the column-pair merge above
// when N <= 65,536 columns).  Warp per row i: the row's column set becomes an N-bit bitmap in
// shared memory, and every entry (i, j) of the row tests its K neighbours J[j, k] with one
// bit probe each -- nnz*K shared-memory probes instead of N*K merges of two CSC columns
// (C3: 19.3 ms for the merge kernel, most of it 15 GB of DRAM reads).  Words come out in
// CSR order; explicit_gather_kernel moves them to CSC order through csc2csr.
constexpr int kRowBitmapMaxWords = 2048;     // N <= 65,536
constexpr int kRowWarps = 8;

__global__ void __launch_bounds__(kRowWarps * 32)
explicit_row_kernel(CulshData d, const int32_t *__restrict__ nbr, int K, int MW, int words,
                    uint32_t *__restrict__ mask_csr) {
    extern __shared__ uint32_t s_bitmap[];
    uint32_t *bm = s_bitmap + (threadIdx.x >> 5) * words;
    const unsigned lane = lane_id();
    for (int w = lane; w < words; w += 32) bm[w] = 0u;
    __syncwarp();
    const int64_t nw = (int64_t)gridDim.x * kRowWarps;
    for (int64_t i = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5); i < d.M; i += nw) {
        const int64_t lo = d.row_ptr[i], hi = d.row_ptr[i + 1];
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int32_t c = d.row_cols[e];
            atomicOr(bm + (c >> 5), 1u << (c & 31));
        }
        __syncwarp();
        // lane k probes neighbour k of one entry at a time (coalesced 128-byte J^K row,
        // one bit probe, one ballot = the entry's mask word); lane x keeps entry x's words
        for (int64_t e0 = lo; e0 < hi; e0 += 32) {
            const int ne = (int)min64(32, hi - e0);
            const int32_t my_j = (int)lane < ne ? d.row_cols[e0 + lane] : 0;
            uint32_t mine0 = 0u, mine1 = 0u;
#pragma unroll 4   // independent entries: several J^K rows in flight
            for (int x = 0; x < ne; ++x) {
                const int32_t *J = nbr + (int64_t)__shfl_sync(0xffffffffu, my_j, x) * K;
                uint32_t bit = 0u;
                if ((int)lane < K) {
                    const int32_t c = __ldg(J + lane);
                    bit = (bm[c >> 5] >> (c & 31)) & 1u;
                }
                const uint32_t m0 = __ballot_sync(0xffffffffu, bit);
                uint32_t m1 = 0u;
                if (MW == 2) {
                    uint32_t bit1 = 0u;
                    if ((int)lane + 32 < K) {
                        const int32_t c = __ldg(J + 32 + lane);
                        bit1 = (bm[c >> 5] >> (c & 31)) & 1u;
                    }
                    m1 = __ballot_sync(0xffffffffu, bit1);
                }
                if ((int)lane == x) {
                    mine0 = m0;
                    mine1 = m1;
                }
            }
            if ((int)lane < ne) {
                mask_csr[(e0 + lane) * MW] = mine0;
                if (MW == 2) mask_csr[(e0 + lane) * MW + 1] = mine1;
            }
        }
        __syncwarp();
        for (int64_t e = lo + lane; e < hi; e += 32) bm[d.row_cols[e] >> 5] = 0u;
        __syncwarp();
    }
}

// CSR-order mask words -> CSC order (csc2csr[q] = CSR position of CSC entry q), with the
// per-column count of explicit pairs.
__global__ void explicit_gather_kernel(CulshData d, int MW, const uint32_t *__restrict__ mask_csr,
                                       uint32_t *__restrict__ mask, unsigned long long *__restrict__ col_nexpl) {
    const unsigned lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < d.N; j += warps) {
        int cnt = 0;
        for (int64_t q = d.col_ptr[j] + lane; q < d.col_ptr[j + 1]; q += 32) {
            const int64_t p = d.csc2csr[q];
            const uint32_t m0 = mask_csr[p * MW];
            mask[q * MW] = m0;
            cnt += __popc(m0);
            if (MW == 2) {
                const uint32_t m1 = mask_csr[p * MW + 1];
                mask[q * MW + 1] = m1;
                cnt += __popc(m1);
            }
        }
        cnt = warp_sum(cnt);
        if (lane == 0) col_nexpl[j] = (unsigned long long)cnt;
    }
}

__global__ void explicit_resid_kernel(CulshData d, double mu, const int32_t *__restrict__ nbr, int K, int MW,
                                      const uint32_t *__restrict__ mask, const int64_t *__restrict__ resid_ptr,
                                      float *__restrict__ resid) {
    const unsigned lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < d.N; j += warps) {
        const int64_t lo = d.col_ptr[j], hi = d.col_ptr[j + 1];
        int64_t run = resid_ptr[j];
        for (int64_t b = lo; b < hi; b += 32) {
            const int64_t e = b + lane;
            uint32_t m0 = 0u, m1 = 0u;
            if (e < hi) {
                m0 = mask[e * MW];
                if (MW == 2) m1 = mask[e * MW + 1];
            }
            const int pc = __popc(m0) + __popc(m1);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            int64_t pos = run + incl - pc;
            run += __shfl_sync(0xffffffffu, incl, 31);
            if (pc) {
                const int32_t i = d.col_rows[e];
                const double bb = d.base_b[i];
                for (int q = 0; q < MW; ++q) {
                    uint32_t m = q == 0 ? m0 : m1;
                    while (m) {
                        const int k = 32 * q + __ffs(m) - 1;
                        m &= m - 1u;
                        const int32_t j1 = nbr[j * K + k];
                        // r(i, j1) from row i's CSR slice (mean 209 entries at C3) when the CSR
                        // view exists, else from column j1's CSC slice (~5,600)
                        double rv;
                        if (d.row_ptr) {
                            rv = d.row_vals[find_row(d.row_cols, d.row_ptr[i], d.row_ptr[i + 1], j1)];
                        } else {
                            rv = d.col_vals[find_row(d.col_rows, d.col_ptr[j1], d.col_ptr[j1 + 1], i)];
                        }
                        resid[pos++] = (float)(rv - (mu + bb + d.base_bhat[j1]));
                    }
                }
            }
        }
    }
}

extern "C" int culsh_explicit_stream(const CulshData *d, double mu, const int32_t *nbr, int K,
                                     uint32_t *mask, int64_t *col_nexpl, const int64_t *resid_ptr,
                                     float *resid, void *stream) {
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    if (d->N <= 0) return CULSH_OK;
    const int MW = K <= 32 ? 1 : 2;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = (int64_t)num_sms() * 16;
    if (!resid) {
        CULSH_CHECK(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * (size_t)(d->nnz * MW), st));
        CULSH_CHECK(cudaMemsetAsync(col_nexpl, 0, sizeof(int64_t) * (size_t)d->N, st));
        if (K == 0 || d->nnz == 0) return CULSH_OK;
        const int words = (int)((d->N + 31) / 32);
        if (words <= kRowBitmapMaxWords && d->row_ptr && d->row_cols && d->csc2csr) {
            uint32_t *mask_csr = nullptr;
            CULSH_CHECK(cudaMallocAsync((void **)&mask_csr, sizeof(uint32_t) * (size_t)(d->nnz * MW), st));
            const size_t smem = sizeof(uint32_t) * (size_t)words * kRowWarps;
            CULSH_CHECK(cudaFuncSetAttribute(explicit_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
            const int64_t rblocks = min64((d->M + kRowWarps - 1) / kRowWarps, (int64_t)num_sms() * 8);
            explicit_row_kernel<<<(unsigned)rblocks, kRowWarps * 32, smem, st>>>(*d, nbr, K, MW, words, mask_csr);
            CULSH_LAUNCH_CHECK();
            explicit_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(*d, MW, mask_csr, mask,
                                                                     reinterpret_cast<unsigned long long *>(col_nexpl));
            CULSH_LAUNCH_CHECK();
            CULSH_CHECK(cudaFreeAsync(mask_csr, st));
            return CULSH_OK;
        }
        explicit_mask_kernel<<<(unsigned)blocks, 256, 0, st>>>(*d, nbr, K, MW, mask,
                                                                reinterpret_cast<unsigned long long *>(col_nexpl));
    } else {
        if (K == 0 || d->nnz == 0) return CULSH_OK;
        explicit_resid_kernel<<<(unsigned)blocks, 256, 0, st>>>(*d, mu, nbr, K, MW, mask, resid_ptr, resid);
    }
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_sgd_hogwild_epoch(int64_t N, const int64_t *col_ptr, const int64_t *seg,
                                       const int32_t *rows,
                                       const float *vals, const uint32_t *mask, const int64_t *resid_ptr,
                                       const float *resid, const int32_t *col_order, CulshModel32 *m,
                                       const CulshRates *r, int flags, int max_warps, int *ticket,
                                       double *loss_out,
                                       int *status, void *stream) {
    const int F = m->F, K = m->K;
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    CULSH_REQUIRE((F >= 1 && F <= 32) || F == 64 || F == 128 || F == 256,
                  "Hogwild mode needs F <= 32 or F in {64, 128, 256}");
    if (N <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CULSH_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    HwCoef R{(float)r->gb, (float)r->gbh, (float)r->gu, (float)r->gv, (float)r->gw, (float)r->gc,
             (float)(1.0 - r->gb * r->lb), (float)(1.0 - r->gbh * r->lbh), (float)(1.0 - r->gu * r->lu),
             (float)(1.0 - r->gv * r->lv), (float)(1.0 - r->gw * r->lw), (float)(1.0 - r->gc * r->lc),
             (float)(1.0 - r->gb * r->lb) - 1.f};
    const bool k2 = K > 32;
    CULSH_REQUIRE((flags & 4) == 0, "flags bit 2 (sub-warp kernel) is no longer supported");
#define HW(FVv) (k2 ? launch_hogwild<FVv, 2>(N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st) \
                    : launch_hogwild<FVv, 1>(N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st))
    if (F <= 32) return HW(1);
    if (F == 64) return HW(2);
    if (F == 128) return HW(4);
    return HW(8);
#undef HW
}

extern "C" int culsh_pack_stream(int64_t N, const int64_t *col_ptr, const int32_t *rows, const float *vals,
                                 const uint32_t *mask, int MW, const float *lut, int n_lut, uint32_t *packed,
                                 int64_t *mcount, const int64_t *mptr, uint32_t *cmask, int *status,
                                 void *stream) {
    CULSH_REQUIRE(MW == 1 || MW == 2, "MW must be 1 or 2");
    CULSH_REQUIRE(n_lut >= 1 && n_lut <= 16, "the value table holds 1..16 values");
    CULSH_REQUIRE(packed ? (mptr != nullptr && cmask != nullptr) : mcount != nullptr,
                  "pass 1 needs mcount; pass 2 needs mptr and cmask");
    if (N <= 0) return CULSH_OK;
    const int64_t blocks = min64((N + 7) / 8, (int64_t)num_sms() * 16);
    pack_stream_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(N, col_ptr, rows, vals, mask, MW, lut,
                                                                           n_lut, packed, mcount, mptr, cmask,
                                                                           status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_sgd_hogwild_epoch_packed(int64_t N_list, const int64_t *col_ptr, const int64_t *seg,
                                              const uint32_t *packed,
                                              const float *lut, const int64_t *mptr, const uint32_t *cmask,
                                              const int64_t *resid_ptr, const float *resid,
                                              const int32_t *col_order, CulshModel32 *m, const CulshRates *r,
                                              int flags, int max_warps, int *ticket, double *loss_out,
                                              int *status, void *stream) {
    const int F = m->F, K = m->K;
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    CULSH_REQUIRE((F >= 1 && F <= 32) || F == 64 || F == 128 || F == 256,
                  "Hogwild mode needs F <= 32 or F in {64, 128, 256}");
    CULSH_REQUIRE((flags & 4) == 0, "flags bit 2 (sub-warp kernel) is no longer supported");
    CULSH_REQUIRE(seg == nullptr || (flags & 8), "the packed stream takes whole columns or work segments");
    if (N_list <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CULSH_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    HwCoef R{(float)r->gb, (float)r->gbh, (float)r->gu, (float)r->gv, (float)r->gw, (float)r->gc,
             (float)(1.0 - r->gb * r->lb), (float)(1.0 - r->gbh * r->lbh), (float)(1.0 - r->gu * r->lu),
             (float)(1.0 - r->gv * r->lv), (float)(1.0 - r->gw * r->lw), (float)(1.0 - r->gc * r->lc),
             (float)(1.0 - r->gb * r->lb) - 1.f};
    const bool k2 = K > 32;
    const int32_t *rows = reinterpret_cast<const int32_t *>(packed);
#define HWP(FVv) (k2 ? launch_hogwild<FVv, 2, true>(N_list, col_ptr, seg, rows, nullptr, cmask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st, lut, mptr) \
                     : launch_hogwild<FVv, 1, true>(N_list, col_ptr, seg, rows, nullptr, cmask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st, lut, mptr))
    if (F <= 32) return HWP(1);
    if (F == 64) return HWP(2);
    if (F == 128) return HWP(4);
    return HWP(8);
#undef HWP
}

extern "C" int culsh_sgd_hogwild_epoch_packed16(int64_t N_list, const int64_t *col_ptr, const int64_t *seg,
                                                const uint16_t *packed, const int32_t *first_row,
                                              const float *lut, const int64_t *mptr, const uint32_t *cmask,
                                              const int64_t *resid_ptr, const float *resid,
                                              const int32_t *col_order, CulshModel32 *m, const CulshRates *r,
                                              int flags, int max_warps, int *ticket, double *loss_out,
                                              int *status, void *stream) {
    const int F = m->F, K = m->K;
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    CULSH_REQUIRE((F >= 1 && F <= 32) || F == 64 || F == 128 || F == 256,
                  "Hogwild mode needs F <= 32 or F in {64, 128, 256}");
    CULSH_REQUIRE((flags & 4) == 0, "flags bit 2 (sub-warp kernel) is no longer supported");
    CULSH_REQUIRE(seg == nullptr || (flags & 8), "the packed stream takes whole columns or work segments");
    CULSH_REQUIRE((flags & 1) == 0, "the 2-byte stream does not run the rotated order");
    if (N_list <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CULSH_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    HwCoef R{(float)r->gb, (float)r->gbh, (float)r->gu, (float)r->gv, (float)r->gw, (float)r->gc,
             (float)(1.0 - r->gb * r->lb), (float)(1.0 - r->gbh * r->lbh), (float)(1.0 - r->gu * r->lu),
             (float)(1.0 - r->gv * r->lv), (float)(1.0 - r->gw * r->lw), (float)(1.0 - r->gc * r->lc),
             (float)(1.0 - r->gb * r->lb) - 1.f};
    const bool k2 = K > 32;
    const int32_t *rows = reinterpret_cast<const int32_t *>(packed);
#define HWP(FVv) (k2 ? launch_hogwild<FVv, 2, true, true>(N_list, col_ptr, seg, rows, nullptr, cmask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st, lut, mptr, first_row) \
                     : launch_hogwild<FVv, 1, true, true>(N_list, col_ptr, seg, rows, nullptr, cmask, resid_ptr, resid, col_order, m, R, flags, max_warps, ticket, loss_out, status, st, lut, mptr, first_row))
    if (F <= 32) return HWP(1);
    if (F == 64) return HWP(2);
    if (F == 128) return HWP(4);
    return HWP(8);
#undef HWP
}

extern "C" int culsh_segment_cursors(int64_t n_list, const int64_t *col_ptr, const int32_t *col_order,
                                     const int64_t *seg2, const uint32_t *words, const uint16_t *w16,
                                     const int32_t *first_row, const int64_t *mptr, const uint32_t *mask, int MW,
                                     int64_t *seg4, void *stream) {
    CULSH_REQUIRE(MW == 1 || MW == 2, "MW must be 1 or 2");
    CULSH_REQUIRE(!w16 || (mptr && first_row), "2-byte records need mptr and first_row");
    CULSH_REQUIRE(!mptr || words || w16, "the packed stream needs its words");
    if (n_list <= 0) return CULSH_OK;
    const int64_t blocks = min64((n_list + 7) / 8, (int64_t)num_sms() * 16);
    segment_cursors_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n_list, col_ptr, col_order, seg2,
                                                                               words, w16, first_row, mptr, mask,
                                                                               MW, seg4);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_pack16(int64_t N, const int64_t *col_ptr, const int32_t *rows, const float *vals,
                            const uint32_t *mask, int MW, const float *lut, int n_lut, uint16_t *words,
                            int32_t *first_row, int *status, void *stream) {
    CULSH_REQUIRE(MW == 1 || MW == 2, "MW must be 1 or 2");
    CULSH_REQUIRE(n_lut >= 1 && n_lut <= 8, "the 2-byte stream holds 1..8 values");
    if (N <= 0) return CULSH_OK;
    const int64_t blocks = min64((N + 7) / 8, (int64_t)num_sms() * 16);
    pack16_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(N, col_ptr, rows, vals, mask, MW, lut, n_lut,
                                                                      words, first_row, status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

