// Hogwild fp32 SGD epoch -- the performance mode of the nonlinear-neighbourhood
// update (paper Alg. 3 CULSH-MF).
//
// One warp owns one column j for a whole epoch: v_j (F floats, FV per lane),
// w_j / c_j (lane k owns k), b_hat_j stay in registers; the column's ratings are
// streamed in CSC order (row, value, explicit-neighbour mask, compact residuals)
// and every update reads and writes the row parameters u_i / b_i in HBM without
// locks (rows are Hogwild, as in Alg. 3).  Per update the warp does one float4
// gather of u_i per lane, one fused shuffle reduction of
//   u_i.v_j + |R|^-1/2 sum_expl resid*w + |N|^-1/2 sum_impl c
// and one float4 store of the updated u_i.  Columns are handed out through a
// ticket counter in descending-nnz order (longest first) for load balance.
//
// The explicit-neighbour test and residuals depend only on (data, J^K)
// (factorization.py:287-298 with the fixed baselines, :12-16), so they are
// precomputed once per fit by explicit_stream_kernel: a K-bit mask per rating
// plus the residuals of the set bits, compacted in (entry, k) order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace culsh {

struct HwRates {
    float gb, gbh, gu, gv, gw, gc, lb, lbh, lu, lv, lw, lc;
};

template <int FV>
__device__ __forceinline__ void load_row(const float *__restrict__ p, float (&x)[FV]) {
    if constexpr (FV == 4) {
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

template <int FV>
__device__ __forceinline__ void store_row(float *__restrict__ p, const float (&x)[FV]) {
    if constexpr (FV == 4) {
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

// FV floats per lane; F == 32*FV (vector path) or F < 32 with FV == 1 (masked).
template <int FV, int KPL>
__global__ void __launch_bounds__(256)
hogwild_kernel(int64_t N, const int64_t *__restrict__ col_ptr, const int64_t *__restrict__ seg,
               const int32_t *__restrict__ rows,
               const float *__restrict__ vals, const uint32_t *__restrict__ mask,
               const int64_t *__restrict__ resid_ptr, const float *__restrict__ resid,
               const int32_t *__restrict__ col_order, float mu, float *__restrict__ Bv,
               float *__restrict__ BHv, float *__restrict__ U, float *__restrict__ V,
               float *__restrict__ W, float *__restrict__ C, int F, int K, HwRates R,
               int *__restrict__ ticket, double *__restrict__ loss, int *__restrict__ status) {
    const unsigned lane = lane_id();
    const bool fl = (int)(lane * FV) < F;   // lane owns factor slots
    const unsigned lt_mask = (1u << lane) - 1u;
    double col_loss = 0.0;
    int bad = 0;

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
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            w[q] = k < K ? W[j * K + k] : 0.f;
            c[q] = k < K ? C[j * K + k] : 0.f;
        }
        float bh = BHv[j];
        const int64_t c_lo = col_ptr[j];
        const int64_t lo = seg ? seg[2 * j] : c_lo;
        const int64_t hi = seg ? seg[2 * j + 1] : col_ptr[j + 1];
        int64_t rbase = resid_ptr[j];
        if (lo > c_lo) {   // DSGD block: skip the residuals of the column's earlier row blocks
            int skip = 0;
            for (int64_t x = c_lo + lane; x < lo; x += 32)
#pragma unroll
                for (int q = 0; q < KPL; ++q) skip += __popc(mask[x * KPL + q]);
            rbase += warp_sum(skip);
        }

        for (int64_t c0 = lo; c0 < hi; c0 += 32) {
            const int n = (int)min64(32, hi - c0);
            const bool have = (int)lane < n;
            const int my_i = have ? rows[c0 + lane] : 0;
            const float my_r = have ? vals[c0 + lane] : 0.f;
            uint32_t my_m[KPL];
            int my_pc = 0;
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                my_m[q] = have ? mask[(c0 + lane) * KPL + q] : 0u;
                my_pc += __popc(my_m[q]);
            }
            // exclusive prefix of explicit counts -> residual offset per entry
            int incl = my_pc;
            if (__any_sync(0xffffffffu, my_pc != 0)) {
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += y;
                }
            }
            const int64_t my_roff = rbase + (incl - my_pc);
            rbase += __shfl_sync(0xffffffffu, incl, 31);

            // software pipeline: u_i of the next update is in flight while this one runs
            float un[FV];
            float bn = 0.f;
            {
                const int i0 = __shfl_sync(0xffffffffu, my_i, 0);
                if (fl) load_row<FV>(U + (int64_t)i0 * F + lane * FV, un);
                bn = Bv[i0];
            }
            for (int tt = 0; tt < n; ++tt) {
                const int i = __shfl_sync(0xffffffffu, my_i, tt);
                const float r = __shfl_sync(0xffffffffu, my_r, tt);
                uint32_t mk[KPL];
#pragma unroll
                for (int q = 0; q < KPL; ++q) mk[q] = __shfl_sync(0xffffffffu, my_m[q], tt);
                const int64_t roff = __shfl_sync(0xffffffffu, my_roff, tt);
                float u[FV];
#pragma unroll
                for (int x = 0; x < FV; ++x) u[x] = un[x];
                const float bi = bn;
                if (tt + 1 < n) {
                    const int i1 = __shfl_sync(0xffffffffu, my_i, tt + 1);
                    if (fl) load_row<FV>(U + (int64_t)i1 * F + lane * FV, un);
                    bn = Bv[i1];
                }
                int nr = 0;
#pragma unroll
                for (int q = 0; q < KPL; ++q) nr += __popc(mk[q]);
                const int nn = K - nr;
                const float inv_r = nr > 0 ? rsqrtf((float)nr) : 0.f;
                const float inv_n = nn > 0 ? rsqrtf((float)nn) : 0.f;
                bool ex[KPL];
                float rs[KPL];
                float part = 0.f;
#pragma unroll
                for (int x = 0; x < FV; ++x) part = fmaf(u[x], v[x], part);
                int before = 0;
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    const int k = lane + 32 * q;
                    ex[q] = (mk[q] >> lane) & 1u;
                    rs[q] = ex[q] ? resid[roff + before + __popc(mk[q] & lt_mask)] : 0.f;
                    before += __popc(mk[q]);
                    if (k < K) part += ex[q] ? rs[q] * w[q] * inv_r : c[q] * inv_n;
                }
                part = warp_sum(part);
                const float e = r - (mu + bi + bh + part);
                col_loss += (double)e * (double)e;
                if (!isfinite(e)) bad = 1;
                // fused update of every touched parameter (factorization.py:307-328 rules)
#pragma unroll
                for (int x = 0; x < FV; ++x) {
                    const float uo = u[x];
                    u[x] = uo + R.gu * (e * v[x] - R.lu * uo);
                    v[x] = v[x] + R.gv * (e * uo - R.lv * v[x]);
                }
                if (fl) store_row<FV>(U + (int64_t)i * F + lane * FV, u);
                if (lane == 0) Bv[i] = bi + R.gb * (e - R.lb * bi);
                bh = bh + R.gbh * (e - R.lbh * bh);
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    if (ex[q]) w[q] = w[q] + R.gw * (inv_r * e * rs[q] - R.lw * w[q]);
                    else c[q] = c[q] + R.gc * (inv_n * e - R.lc * c[q]);
                }
            }
        }
        if (fl) store_row<FV>(V + j * F + lane * FV, v);
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            if (k < K) {
                W[j * K + k] = w[q];
                C[j * K + k] = c[q];
            }
        }
        if (lane == 0) BHv[j] = bh;
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

constexpr int kStreamThreads = 256;

// CTA per column.  Pass 1 (resid == nullptr): mask words + per-column explicit count.
// Pass 2: residuals at resid_ptr[j] + exclusive prefix over the column's entries.
__global__ void __launch_bounds__(kStreamThreads)
explicit_stream_kernel(CulshData d, double mu, const int32_t *__restrict__ nbr, int K, int MW,
                       uint32_t *__restrict__ mask, int64_t *__restrict__ col_nexpl,
                       const int64_t *__restrict__ resid_ptr, float *__restrict__ resid) {
    using BlockScan = cub::BlockScan<int, kStreamThreads>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ int64_t s_run;
    __shared__ int64_t s_nlo[64], s_nhi[64];
    const int64_t j = blockIdx.x;
    const int64_t lo = d.col_ptr[j], hi = d.col_ptr[j + 1];
    if (threadIdx.x < K && threadIdx.x < 64) {
        const int32_t j1 = nbr[j * K + threadIdx.x];
        s_nlo[threadIdx.x] = d.col_ptr[j1];
        s_nhi[threadIdx.x] = d.col_ptr[j1 + 1];
    }
    if (threadIdx.x == 0) s_run = resid ? resid_ptr[j] : 0;
    __syncthreads();
    int64_t count = 0;
    for (int64_t base = lo; base < hi; base += kStreamThreads) {
        const int64_t idx = base + threadIdx.x;
        const bool have = idx < hi;
        const int32_t i = have ? d.col_rows[idx] : 0;
        uint32_t m[2] = {0u, 0u};
        if (have) {
            if (resid) {
                for (int q = 0; q < MW; ++q) m[q] = mask[idx * MW + q];
            } else {
                for (int k = 0; k < K; ++k)
                    if (find_row(d.col_rows, s_nlo[k], s_nhi[k], i) >= 0) m[k >> 5] |= 1u << (k & 31);
                for (int q = 0; q < MW; ++q) mask[idx * MW + q] = m[q];
            }
        }
        const int pc = __popc(m[0]) + __popc(m[1]);
        if (resid) {
            int excl = 0, tot = 0;
            BlockScan(scan_tmp).ExclusiveSum(pc, excl, tot);
            int64_t o = s_run + excl;
            if (have && pc) {
                const double bb = d.base_b[i];
                for (int k = 0; k < K; ++k) {
                    if ((m[k >> 5] >> (k & 31)) & 1u) {
                        const int32_t j1 = nbr[j * K + k];
                        const int64_t pos = find_row(d.col_rows, s_nlo[k], s_nhi[k], i);
                        const double rv = d.col_vals[pos];
                        resid[o++] = (float)(rv - (mu + bb + d.base_bhat[j1]));
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_run += tot;
            __syncthreads();
        } else {
            count += pc;
        }
    }
    if (!resid) {
        typedef cub::BlockReduce<int64_t, kStreamThreads> BR;
        __shared__ typename BR::TempStorage red_tmp;
        const int64_t tot = BR(red_tmp).Sum(count);
        if (threadIdx.x == 0) col_nexpl[j] = tot;
    }
}

template <int FV, int KPL>
int launch_hogwild(int64_t N, const int64_t *col_ptr, const int64_t *seg, const int32_t *rows, const float *vals,
                   const uint32_t *mask, const int64_t *resid_ptr, const float *resid,
                   const int32_t *col_order, CulshModel32 *m, const HwRates &R, int *ticket, double *loss,
                   int *status, cudaStream_t st) {
    const int threads = 256;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hogwild_kernel<FV, KPL>, threads, 0);
    if (occ < 1) occ = 1;
    int64_t blocks = (int64_t)num_sms() * occ;
    const int64_t need = (N + 7) / 8;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    hogwild_kernel<FV, KPL><<<(unsigned)blocks, threads, 0, st>>>(
        N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m->mu, m->b, m->bhat, m->U, m->V, m->W,
        m->C, m->F, m->K, R, ticket, loss, status);
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_explicit_stream(const CulshData *d, double mu, const int32_t *nbr, int K,
                                     uint32_t *mask, int64_t *col_nexpl, const int64_t *resid_ptr,
                                     float *resid, void *stream) {
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    if (d->N <= 0) return CULSH_OK;
    const int MW = K <= 32 ? 1 : 2;
    explicit_stream_kernel<<<(unsigned)d->N, kStreamThreads, 0, (cudaStream_t)stream>>>(
        *d, mu, nbr, K, MW, mask, col_nexpl, resid_ptr, resid);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_sgd_hogwild_epoch(int64_t N, const int64_t *col_ptr, const int64_t *seg,
                                       const int32_t *rows,
                                       const float *vals, const uint32_t *mask, const int64_t *resid_ptr,
                                       const float *resid, const int32_t *col_order, CulshModel32 *m,
                                       const CulshRates *r, int *ticket, double *loss_out, int *status,
                                       void *stream) {
    const int F = m->F, K = m->K;
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    CULSH_REQUIRE((F >= 1 && F <= 32) || F == 64 || F == 128 || F == 256,
                  "Hogwild mode needs F <= 32 or F in {64, 128, 256}");
    if (N <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CULSH_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    HwRates R{(float)r->gb, (float)r->gbh, (float)r->gu, (float)r->gv, (float)r->gw, (float)r->gc,
              (float)r->lb, (float)r->lbh, (float)r->lu, (float)r->lv, (float)r->lw, (float)r->lc};
    const bool k2 = K > 32;
#define HW(FVv) (k2 ? launch_hogwild<FVv, 2>(N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m, R, ticket, loss_out, status, st) \
                    : launch_hogwild<FVv, 1>(N, col_ptr, seg, rows, vals, mask, resid_ptr, resid, col_order, m, R, ticket, loss_out, status, st))
    if (F <= 32) return HW(1);
    if (F == 64) return HW(2);
    if (F == 128) return HW(4);
    return HW(8);
#undef HW
}
