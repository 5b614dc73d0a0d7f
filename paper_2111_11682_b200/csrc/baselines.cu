// Residual baselines in the reference's exact summation order, for ANY rating values
// (data.py:289-309 compute_baselines):
//   mu        = np.mean(entry_values): numpy's pairwise sum (8 accumulators on leaves of
//               <= 128 elements, halving splits rounded down to multiples of 8) / nnz
//   row sums  = np.add.at(zeros(M), entry_rows, entry_values): per row, 0.0 + the row's
//               values one by one in ENTRY order (likewise for columns)
// Integer-valued data make every order exact and keep the cheaper warp sums
// (culsh_segment_sums); these kernels give the same bytes as the host numpy for real values.
#include "common.cuh"

namespace culsh {

// numpy pairwise_sum (loops_utils.h.src) for one contiguous run, n <= 2^16.
__device__ double np_pairwise(const double *__restrict__ a, int64_t n) {
    // explicit stack of pending right halves: depth <= log2(2^16 / 128) + 1
    const double *sa[16];
    int64_t sn[16];
    double sres[16];
    int sp = 0;
    double res = 0.0;
    // iterative post-order over the split tree: walk left, push right
    for (;;) {
        if (n > 128) {
            int64_t n2 = n / 2;
            n2 -= n2 % 8;
            sa[sp] = a + n2;
            sn[sp] = n - n2;
            sres[sp] = 0.0;   // placeholder until the left result exists
            ++sp;
            n = n2;
            continue;
        }
        // leaf
        if (n < 8) {
            res = 0.0;
            for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        } else {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = a[j];
            int64_t i = 8;
            for (; i < n - (n % 8); i += 8)
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        }
        // unwind: a finished subtree is either a left child (start its right sibling) or a
        // right child (combine with the stored left result)
        for (;;) {
            if (sp == 0) return res;
            if (sn[sp - 1] > 0) {          // left child just finished: keep it, do the right
                sres[sp - 1] = res;
                a = sa[sp - 1];
                n = sn[sp - 1];
                sn[sp - 1] = -1;           // mark: right half in progress
                break;
            }
            res = __dadd_rn(sres[sp - 1], res);   // right finished: left + right
            --sp;
        }
    }
}

__global__ void pairwise_chunks_kernel(const double *__restrict__ x, const int64_t *__restrict__ off,
                                       const int64_t *__restrict__ len, int64_t nchunks, double *__restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nchunks) out[c] = np_pairwise(x + off[c], len[c]);
}

// out[s] = (init ? init[s] : 0.0) + val[order[ptr[s]]] + val[order[ptr[s] + 1]] + ... in that
// order (thread per segment; order == nullptr: identity).
__global__ void ordered_segment_sums_kernel(int64_t n, const int64_t *__restrict__ ptr,
                                            const int64_t *__restrict__ order, const double *__restrict__ val,
                                            const double *__restrict__ init, double *__restrict__ out) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        double acc = init ? init[s] : 0.0;
        const int64_t hi = ptr[s + 1];
        for (int64_t x = ptr[s]; x < hi; ++x) acc = __dadd_rn(acc, val[order ? order[x] : x]);
        out[s] = acc;
    }
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_pairwise_chunks(const double *x, const int64_t *off, const int64_t *len, int64_t nchunks,
                                     double *out, void *stream) {
    CULSH_REQUIRE(nchunks >= 0, "bad chunk count");
    if (nchunks == 0) return CULSH_OK;
    const int threads = 128;
    pairwise_chunks_kernel<<<(unsigned)((nchunks + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        x, off, len, nchunks, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_ordered_segment_sums(int64_t n, const int64_t *ptr, const int64_t *order, const double *val,
                                          const double *init, double *out, void *stream) {
    CULSH_REQUIRE(n >= 0, "bad segment count");
    if (n == 0) return CULSH_OK;
    const int threads = 128;
    const int64_t blocks = min64((n + threads - 1) / threads, (int64_t)num_sms() * 32);
    ordered_segment_sums_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(n, ptr, order, val, init,
                                                                                        out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
