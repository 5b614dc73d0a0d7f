// Exact column similarity (similarity.py): shrunk Pearson over co-rated rows and
// the all-pairs GSM top-K (the quality oracle for simLSH).
//
// Two exact routes to the six co-rating statistics {n, s1, s2, s12, q1, q2} of a
// column pair (similarity.py:57-90):
//  * merge route: one thread per pair walks both sorted row lists in ascending
//    row order and sums in fp64 exactly as _pair_stats does (bit-identical for
//    any values);
//  * count route (integer ratings, |r| <= 11): with X = indicator, R = values,
//    Q = R*R as dense int8 column panels, n = X'X, s1 = R'X, s2 = X'R, s12 = R'R,
//    q1 = Q'X, q2 = X'Q are integer matrix products (tensor-core int8 GEMMs with
//    exact int32 accumulation).  Every partial sum of the reference is then an
//    exact integer (< 2^53), so the fp64 statistics -- and everything computed
//    from them -- are bit-identical to the reference's.
// The selection kernel turns the statistics into the shrunk similarity with the
// reference's exact fp64 expression tree (compiled -fmad=false) and keeps, per
// target column, the K best by (similarity desc, index asc) -- the order
// _topk_insert's strict comparisons produce (similarity.py:137-161).
#include <cfloat>

#include "common.cuh"

namespace culsh {

struct PairStats {
    double n, s1, s2, s12, q1, q2;
};

// similarity.py:93-107 _pearson_from_stats, same operation order.
__device__ __forceinline__ double pearson_from_stats(const PairStats &st) {
    if (st.n < 2.0) return 0.0;
    const double cov = st.s12 - st.s1 * st.s2 / st.n;
    const double var1 = st.q1 - st.s1 * st.s1 / st.n;
    const double var2 = st.q2 - st.s2 * st.s2 / st.n;
    if (var1 <= 0.0 || var2 <= 0.0) return 0.0;
    double rho = cov / sqrt(var1 * var2);
    if (rho > 1.0) rho = 1.0;
    else if (rho < -1.0) rho = -1.0;
    return rho;
}

// similarity.py:175-178 (and shrunk_similarity :128-135): n/(n+lambda) * rho.
__device__ __forceinline__ double shrunk_of(const PairStats &st, double lambda_rho) {
    if (st.n == 0.0) return 0.0;
    return st.n / (st.n + lambda_rho) * pearson_from_stats(st);
}

// similarity.py:57-90 _pair_stats by sorted merge (ascending rows, fp64 sums).
__device__ __forceinline__ PairStats merge_stats(const int32_t *__restrict__ r1, const double *__restrict__ v1,
                                                 int64_t n1, const int32_t *__restrict__ r2,
                                                 const double *__restrict__ v2, int64_t n2) {
    PairStats st{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int64_t a = 0, b = 0, n = 0;
    while (a < n1 && b < n2) {
        const int32_t x = r1[a], y = r2[b];
        if (x == y) {
            const double p = v1[a], q = v2[b];
            ++n;
            st.s1 += p;
            st.s2 += q;
            st.s12 += p * q;
            st.q1 += p * p;
            st.q2 += q * q;
            ++a;
            ++b;
        } else if (x < y) {
            ++a;
        } else {
            ++b;
        }
    }
    st.n = (double)n;
    return st;
}

// (sim, idx) total order of the reference's top-K: larger sim first, then lower index.
__device__ __forceinline__ bool better(double s, int32_t j, double t, int32_t k) {
    return s > t || (s == t && j < k);
}

constexpr int kSelThreads = 256;

// Per-thread descending top-K list (insertion exactly as _topk_insert: the thread
// scans its j2 in ascending order, so strict comparisons keep lower indices first).
template <int KMAX>
struct LocalTopK {
    double s[KMAX];
    int32_t j[KMAX];
    int count = 0;
    __device__ __forceinline__ void insert(double v, int32_t idx, int K) {
        int pos;
        if (count < K) {
            pos = count++;
        } else if (v > s[K - 1]) {
            pos = K - 1;
        } else {
            return;
        }
        while (pos > 0 && s[pos - 1] < v) {
            s[pos] = s[pos - 1];
            j[pos] = j[pos - 1];
            --pos;
        }
        s[pos] = v;
        j[pos] = idx;
    }
};

// Block-wide K-way merge of the per-thread lists: K rounds of a block argmax over
// the list heads under `better`.
template <int KMAX>
__device__ void block_merge_topk(LocalTopK<KMAX> &L, int K, int32_t *__restrict__ out) {
    __shared__ double s_s[kSelThreads / 32];
    __shared__ int32_t s_j[kSelThreads / 32];
    __shared__ int s_t[kSelThreads / 32];
    __shared__ int s_win;
    int head = 0;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    for (int r = 0; r < K; ++r) {
        double v = head < L.count ? L.s[head] : -DBL_MAX;
        int32_t jj = head < L.count ? L.j[head] : INT32_MAX;
        int who = threadIdx.x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
            const int32_t j2 = __shfl_xor_sync(0xffffffffu, jj, o);
            const int w2 = __shfl_xor_sync(0xffffffffu, who, o);
            if (better(v2, j2, v, jj)) { v = v2; jj = j2; who = w2; }
        }
        if (lane == 0) { s_s[warp] = v; s_j[warp] = jj; s_t[warp] = who; }
        __syncthreads();
        if (warp == 0) {
            const bool have = (int)lane < kSelThreads / 32;
            v = have ? s_s[lane] : -DBL_MAX;
            jj = have ? s_j[lane] : INT32_MAX;
            who = have ? s_t[lane] : -1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int32_t j2 = __shfl_xor_sync(0xffffffffu, jj, o);
                const int w2 = __shfl_xor_sync(0xffffffffu, who, o);
                if (better(v2, j2, v, jj)) { v = v2; jj = j2; who = w2; }
            }
            if (lane == 0) {
                s_win = who;
                out[r] = jj;
            }
        }
        __syncthreads();
        if ((int)threadIdx.x == s_win) ++head;
        __syncthreads();
    }
}

// Merge route: block per target column j1 (rows [j_lo, j_lo + n_rows)), thread per
// candidate j2 stride; j1's row list is staged in shared memory when it fits.
template <int KMAX>
__global__ void __launch_bounds__(kSelThreads)
gsm_merge_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                 const double *__restrict__ col_vals, int64_t N, int64_t j_lo, int K, double lambda_rho,
                 int smem_cap, int32_t *__restrict__ entries) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int64_t j1 = j_lo + blockIdx.x;
    const int64_t a0 = col_ptr[j1], n1 = col_ptr[j1 + 1] - a0;
    const int32_t *r1 = col_rows + a0;
    const double *v1 = col_vals + a0;
    if (n1 <= smem_cap) {
        double *sv = reinterpret_cast<double *>(s_raw);
        int32_t *sr = reinterpret_cast<int32_t *>(sv + smem_cap);
        for (int64_t x = threadIdx.x; x < n1; x += blockDim.x) {
            sv[x] = v1[x];
            sr[x] = r1[x];
        }
        __syncthreads();
        r1 = sr;
        v1 = sv;
    }
    LocalTopK<KMAX> L;
    for (int64_t j2 = threadIdx.x; j2 < N; j2 += blockDim.x) {
        if (j2 == j1) continue;
        const int64_t b0 = col_ptr[j2];
        const PairStats st = merge_stats(r1, v1, n1, col_rows + b0, col_vals + b0, col_ptr[j2 + 1] - b0);
        L.insert(shrunk_of(st, lambda_rho), (int32_t)j2, K);
    }
    block_merge_topk<KMAX>(L, K, entries + blockIdx.x * (int64_t)K);
}

// Warp top-K list in registers: entry k = q * 32 + lane lives in lane `lane`, slot q (KE
// slots per lane, K <= 32 * KE), kept sorted best-first under `better` (similarity desc,
// index asc -- the order _topk_insert's strict comparisons produce).  Only static indexing,
// so the list never touches local memory (the per-thread insertion lists it replaces
// spilled: 32 GB of local-memory DRAM writes per C3 select).
template <int KE>
struct WarpTopK {
    double s[KE];
    int32_t j[KE];
    int count = 0;
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int q = 0; q < KE; ++q) { s[q] = -DBL_MAX; j[q] = INT32_MAX; }
    }
    // the K-th (worst kept) entry, warp-uniform
    __device__ __forceinline__ void kth(int K, double &ts, int32_t &tj) const {
        const int q = (K - 1) >> 5, l = (K - 1) & 31;
        double v = s[0];
        int32_t x = j[0];
#pragma unroll
        for (int p = 1; p < KE; ++p) if (p == q) { v = s[p]; x = j[p]; }
        ts = __shfl_sync(0xffffffffu, v, l);
        tj = __shfl_sync(0xffffffffu, x, l);
    }
    // insert a warp-uniform candidate (caller guarantees it belongs in the top K)
    __device__ __forceinline__ void insert(double cs, int32_t cj, int K) {
        const unsigned lane = lane_id();
        int pos = 0;
#pragma unroll
        for (int q = 0; q < KE; ++q) {
            const int k = q * 32 + (int)lane;
            pos += __popc(__ballot_sync(0xffffffffu, k < count && better(s[q], j[q], cs, cj)));
        }
        double ps[KE];
        int32_t pj[KE];
#pragma unroll
        for (int q = 0; q < KE; ++q) {   // entry k - 1 of every k: lane - 1 of slot q, or lane 31 of slot q - 1
            double up = __shfl_up_sync(0xffffffffu, s[q], 1);
            int32_t upj = __shfl_up_sync(0xffffffffu, j[q], 1);
            const double wrap = __shfl_sync(0xffffffffu, q > 0 ? s[q > 0 ? q - 1 : 0] : 0.0, 31);
            const int32_t wrapj = __shfl_sync(0xffffffffu, q > 0 ? j[q > 0 ? q - 1 : 0] : 0, 31);
            ps[q] = lane == 0 ? wrap : up;
            pj[q] = lane == 0 ? wrapj : upj;
        }
#pragma unroll
        for (int q = 0; q < KE; ++q) {
            const int k = q * 32 + (int)lane;
            if (k == pos) { s[q] = cs; j[q] = cj; }
            else if (k > pos && k < K) { s[q] = ps[q]; j[q] = pj[q]; }
        }
        if (count < K) ++count;
    }
    // offer one candidate per lane (valid lanes only): accepted ones are inserted in lane order
    __device__ __forceinline__ void offer(bool valid, double cs, int32_t cj, int K) {
        double ts = -DBL_MAX;
        int32_t tj = INT32_MAX;
        if (count >= K) kth(K, ts, tj);
        unsigned acc = __ballot_sync(0xffffffffu, valid && (count < K || better(cs, cj, ts, tj)));
        while (acc) {
            const int l = __ffs(acc) - 1;
            acc &= acc - 1u;
            const double vs = __shfl_sync(0xffffffffu, cs, l);
            const int32_t vj = __shfl_sync(0xffffffffu, cj, l);
            if (count >= K) {                       // the threshold moved: re-check
                kth(K, ts, tj);
                if (!better(vs, vj, ts, tj)) continue;
            }
            insert(vs, vj, K);
        }
    }
};

// Count route selection, warp-parallel: block per target column j1, each warp offers 32
// candidates j2 at a time to its register top-K list, then warp 0 merges the others' lists.
// All six statistics are read row-wise (s2 / q2 from the transposed copies g_xr / g_xq
// written by the tensor-core kernel's epilogue; the strided reads of the transposes cost
// ~20 GB of sector traffic at C3).
template <int KE>
__global__ void __launch_bounds__(kSelThreads)
gsm_count_select_warp_kernel(const int32_t *__restrict__ g_xx, const int32_t *__restrict__ g_rx,
                             const int32_t *__restrict__ g_rr, const int32_t *__restrict__ g_qx,
                             const int32_t *__restrict__ g_xr, const int32_t *__restrict__ g_xq, int64_t ld,
                             int64_t N, int64_t j_lo, int K, double lambda_rho, int32_t *__restrict__ entries) {
    constexpr int NW = kSelThreads / 32;
    __shared__ double m_s[NW][32 * KE];
    __shared__ int32_t m_j[NW][32 * KE];
    __shared__ int m_n[NW];
    const int64_t j1 = j_lo + blockIdx.x;
    const int64_t row = j1 * ld;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    WarpTopK<KE> L;
    L.init();
    for (int64_t base = (int64_t)warp * 32; base < N; base += kSelThreads) {
        const int64_t j2 = base + lane;
        const bool valid = j2 < N && j2 != j1;
        double sim = 0.0;
        if (valid) {
            PairStats st;
            st.n = (double)g_xx[row + j2];
            st.s1 = (double)g_rx[row + j2];
            st.s2 = (double)g_xr[row + j2];
            st.s12 = (double)g_rr[row + j2];
            st.q1 = (double)g_qx[row + j2];
            st.q2 = (double)g_xq[row + j2];
            sim = shrunk_of(st, lambda_rho);
        }
        L.offer(valid, sim, (int32_t)j2, K);
    }
#pragma unroll
    for (int q = 0; q < KE; ++q) {
        m_s[warp][q * 32 + lane] = L.s[q];
        m_j[warp][q * 32 + lane] = L.j[q];
    }
    if (lane == 0) m_n[warp] = L.count;
    __syncthreads();
    if (warp == 0) {
        for (int w = 1; w < NW; ++w)
            for (int k0 = 0; k0 < m_n[w]; k0 += 32) {
                const int k = k0 + (int)lane;
                const bool v = k < m_n[w];
                L.offer(v, v ? m_s[w][k] : -DBL_MAX, v ? m_j[w][k] : INT32_MAX, K);
            }
#pragma unroll
        for (int q = 0; q < KE; ++q) {
            const int k = q * 32 + (int)lane;
            if (k < K) entries[blockIdx.x * (int64_t)K + k] = L.j[q];
        }
    }
}

// Count route, selection over the int32 products (rows [j_lo, j_lo + n_rows) of
// the N x N statistics; g_* row r holds target column j_lo + r, ld = row stride).
// s2 / q2 are read from the transposed entry of the full products g_rx / g_qx.
template <int KMAX>
__global__ void __launch_bounds__(kSelThreads)
gsm_count_select_kernel(const int32_t *__restrict__ g_xx, const int32_t *__restrict__ g_rx,
                        const int32_t *__restrict__ g_rr, const int32_t *__restrict__ g_qx, int64_t ld,
                        int64_t N, int64_t j_lo, int K, double lambda_rho, int32_t *__restrict__ entries) {
    const int64_t j1 = j_lo + blockIdx.x;
    const int64_t row = j1 * ld;
    LocalTopK<KMAX> L;
    for (int64_t j2 = threadIdx.x; j2 < N; j2 += blockDim.x) {
        if (j2 == j1) continue;
        PairStats st;
        st.n = (double)g_xx[row + j2];
        st.s1 = (double)g_rx[row + j2];
        st.s2 = (double)g_rx[j2 * ld + j1];
        st.s12 = (double)g_rr[row + j2];
        st.q1 = (double)g_qx[row + j2];
        st.q2 = (double)g_qx[j2 * ld + j1];
        L.insert(shrunk_of(st, lambda_rho), (int32_t)j2, K);
    }
    block_merge_topk<KMAX>(L, K, entries + blockIdx.x * (int64_t)K);
}

// Dense int8 column panels for the count route: row j of xt/rt/qt (stride ld) gets
// 1 / r / r*r at column i - row_lo for every rating (i, j) with row_lo <= i < row_hi.  *status |= 1 when a value is
// not an integer in [-11, 11] (then r*r does not fit int8 / the route is invalid).
__global__ void gsm_densify_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                                   const double *__restrict__ col_vals, int64_t N, int64_t row_lo, int64_t row_hi,
                                   int64_t ld, int8_t *__restrict__ xt, int8_t *__restrict__ rt,
                                   int8_t *__restrict__ qt, int *__restrict__ status) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const unsigned lane = lane_id();
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < N; j += warps) {
        int bad = 0;
        for (int64_t e = col_ptr[j] + lane; e < col_ptr[j + 1]; e += 32) {
            const int32_t i = col_rows[e];
            if (i < row_lo || i >= row_hi) continue;
            const double v = col_vals[e];
            const int iv = (int)v;
            if ((double)iv != v || iv < -11 || iv > 11) bad = 1;
            const int64_t o = j * ld + (i - row_lo);
            xt[o] = 1;
            rt[o] = (int8_t)iv;
            qt[o] = (int8_t)(iv * iv);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1);
    }
}

// pearson / shrunk_similarity of one pair (similarity.py:110-135) by the merge route.
__global__ void pair_similarity_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                                       const double *__restrict__ col_vals, int64_t j1, int64_t j2,
                                       double lambda_rho, double *__restrict__ out) {
    const int64_t a0 = col_ptr[j1], b0 = col_ptr[j2];
    const PairStats st = merge_stats(col_rows + a0, col_vals + a0, col_ptr[j1 + 1] - a0, col_rows + b0,
                                     col_vals + b0, col_ptr[j2 + 1] - b0);
    out[0] = pearson_from_stats(st);
    out[1] = shrunk_of(st, lambda_rho);
    out[2] = st.n;
}

}  // namespace culsh

using namespace culsh;

#define CULSH_GSM_KDISPATCH(KERNEL, ...)                                       \
    do {                                                                       \
        if (K <= 16) KERNEL<16><<<grid, kSelThreads, smem, st>>>(__VA_ARGS__); \
        else if (K <= 32) KERNEL<32><<<grid, kSelThreads, smem, st>>>(__VA_ARGS__); \
        else if (K <= 64) KERNEL<64><<<grid, kSelThreads, smem, st>>>(__VA_ARGS__); \
        else KERNEL<128><<<grid, kSelThreads, smem, st>>>(__VA_ARGS__);       \
    } while (0)

extern "C" int culsh_gsm_merge_topk(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                                    int64_t N, int64_t j_lo, int64_t n_rows, int K, double lambda_rho,
                                    int32_t *entries, void *stream) {
    CULSH_REQUIRE(K >= 1 && K <= 128 && K <= N - 1, "GSM needs 1 <= K <= min(128, N-1)");
    CULSH_REQUIRE(j_lo >= 0 && n_rows >= 0 && j_lo + n_rows <= N, "row range out of bounds");
    if (n_rows == 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int smem_cap = 8192;   // j1's list in shared memory up to 8192 ratings (96 KB)
    const size_t smem = (size_t)smem_cap * 12;
    {   // per device and cheap: set on every launch (a once-per-process flag breaks on a 2nd GPU)
        cudaFuncSetAttribute(gsm_merge_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(gsm_merge_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(gsm_merge_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(gsm_merge_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const unsigned grid = (unsigned)n_rows;
    CULSH_GSM_KDISPATCH(gsm_merge_kernel, col_ptr, col_rows, col_vals, N, j_lo, K, lambda_rho, smem_cap, entries);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_gsm_densify_rows(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                                      int64_t N, int64_t row_lo, int64_t row_hi, int64_t ld, int8_t *xt,
                                      int8_t *rt, int8_t *qt, int *status, void *stream) {
    CULSH_REQUIRE(row_hi - row_lo <= ld, "panel row stride shorter than the row range");
    if (N <= 0) return CULSH_OK;
    const int64_t blocks = min64((N + 7) / 8, (int64_t)num_sms() * 16);
    gsm_densify_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(col_ptr, col_rows, col_vals, N, row_lo,
                                                                            row_hi, ld, xt, rt, qt, status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_gsm_count_select(const int32_t *g_xx, const int32_t *g_rx, const int32_t *g_rr,
                                      const int32_t *g_qx, const int32_t *g_xr, const int32_t *g_xq, int64_t ld,
                                      int64_t N, int64_t j_lo, int64_t n_rows, int K, double lambda_rho,
                                      int32_t *entries, void *stream) {
    CULSH_REQUIRE(K >= 1 && K <= 128 && K <= N - 1, "GSM needs 1 <= K <= min(128, N-1)");
    CULSH_REQUIRE(j_lo >= 0 && n_rows >= 0 && j_lo + n_rows <= N && ld >= N, "row range out of bounds");
    if (n_rows == 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)n_rows;
    const size_t smem = 0;
    if (g_xr && g_xq) {
        if (K <= 32) gsm_count_select_warp_kernel<1><<<grid, kSelThreads, 0, st>>>(
            g_xx, g_rx, g_rr, g_qx, g_xr, g_xq, ld, N, j_lo, K, lambda_rho, entries);
        else if (K <= 64) gsm_count_select_warp_kernel<2><<<grid, kSelThreads, 0, st>>>(
            g_xx, g_rx, g_rr, g_qx, g_xr, g_xq, ld, N, j_lo, K, lambda_rho, entries);
        else gsm_count_select_warp_kernel<4><<<grid, kSelThreads, 0, st>>>(
            g_xx, g_rx, g_rr, g_qx, g_xr, g_xq, ld, N, j_lo, K, lambda_rho, entries);
        CULSH_LAUNCH_CHECK();
        return CULSH_OK;
    }
    CULSH_GSM_KDISPATCH(gsm_count_select_kernel, g_xx, g_rx, g_rr, g_qx, ld, N, j_lo, K, lambda_rho, entries);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_pair_similarity(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                                     int64_t j1, int64_t j2, double lambda_rho, double *out, void *stream) {
    pair_similarity_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(col_ptr, col_rows, col_vals, j1, j2, lambda_rho, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
