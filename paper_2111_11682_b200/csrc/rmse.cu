// Evaluation: exact fp64 prediction and RMSE.
// predict_one restates factorization.py:235-263 in its exact operation order
// (compiled with -fmad=false); the RMSE sum is sequential (bit-identical to
// factorization.py:394-409) when `sequential` is set, otherwise a fixed
// pairwise tree (deterministic, within a few ulp of the sequential sum).
#include "common.cuh"

namespace culsh {

__device__ __forceinline__ bool lookup_rv(const int64_t *row_ptr, const int32_t *row_cols,
                                          const double *row_vals, int64_t i, int32_t j, double *rv) {
    int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        const int32_t c = row_cols[mid];
        if (c == j) { *rv = row_vals[mid]; return true; }
        if (c < j) lo = mid + 1; else hi = mid;
    }
    return false;
}

template <typename P>
__device__ double predict_one(const CulshData &d, double mu, const P *b, const P *bhat, const P *U,
                              const P *V, const P *W, const P *C, const int32_t *nbr, int F, int K,
                              int64_t i, int64_t j) {
    double pred = mu + (double)b[i] + (double)bhat[j];
    double dot = 0.0;
    for (int f = 0; f < F; ++f) dot = dot + (double)U[i * F + f] * (double)V[j * F + f];
    pred = pred + dot;
    if (K > 0) {
        int nr = 0, nn = 0;
        double sw = 0.0, sc = 0.0;
        for (int k = 0; k < K; ++k) {
            const int32_t j1 = nbr[j * K + k];
            double rv;
            if (lookup_rv(d.row_ptr, d.row_cols, d.row_vals, i, j1, &rv)) {
                ++nr;
                sw = sw + (rv - (mu + d.base_b[i] + d.base_bhat[j1])) * (double)W[j * K + k];
            } else {
                ++nn;
                sc = sc + (double)C[j * K + k];
            }
        }
        if (nr > 0) pred = pred + sw / sqrt((double)nr);
        if (nn > 0) pred = pred + sc / sqrt((double)nn);
    }
    return pred;
}

template <typename P>
__global__ void sqerr_kernel(CulshData d, double mu, const P *b, const P *bhat, const P *U, const P *V,
                             const P *W, const P *C, const int32_t *nbr, int F, int K,
                             const int32_t *t_rows, const int32_t *t_cols, const double *t_vals,
                             int64_t n, int do_clamp, double lo, double hi, double unscale,
                             double *out, int mode) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        double pred = predict_one<P>(d, mu, b, bhat, U, V, W, C, nbr, F, K, t_rows[x], t_cols[x]);
        if (mode == 1) { out[x] = pred; continue; }
        if (do_clamp) {
            if (pred < lo) pred = lo;
            else if (pred > hi) pred = hi;
        }
        const double dd = (pred - t_vals[x]) * unscale;
        out[x] = dd * dd;
    }
}

__global__ void seq_sum_kernel(const double *x, int64_t n, double *out) {
    double total = 0.0;
    for (int64_t k = 0; k < n; ++k) total = total + x[k];
    *out = sqrt(total / (double)n);
}

// fixed-shape pairwise tree: 1024-wide blocks, then one block over the partials
__global__ void tree_sum_kernel(const double *x, int64_t n, double *partial) {
    __shared__ double s[1024];
    double acc = 0.0;
    for (int64_t k = blockIdx.x * 1024LL + threadIdx.x; k < n; k += (int64_t)gridDim.x * 1024) acc = acc + x[k];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] = s[threadIdx.x] + s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void finish_kernel(const double *partial, int np, int64_t n, double *out) {
    double t = 0.0;
    for (int k = 0; k < np; ++k) t = t + partial[k];
    *out = sqrt(t / (double)n);
}

int reduce_rmse(const double *sq, int64_t n, double *out, double *scratch_partials, bool sequential,
                cudaStream_t st) {
    if (sequential) {
        seq_sum_kernel<<<1, 1, 0, st>>>(sq, n, out);
    } else {
        const int np = 256;
        tree_sum_kernel<<<np, 1024, 0, st>>>(sq, n, scratch_partials);
        finish_kernel<<<1, 1, 0, st>>>(scratch_partials, np, n, out);
    }
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

}  // namespace culsh

using namespace culsh;

// sqerr_scratch must hold n + 256 doubles.  Sequential (bit-exact) sum for n <= 2^22.
extern "C" int culsh_rmse(const CulshData *d, const CulshModel64 *m, const int32_t *t_rows,
                          const int32_t *t_cols, const double *t_vals, int64_t n, int do_clamp,
                          double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                          double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 127) / 128, (int64_t)num_sms() * 16);
    sqerr_kernel<double><<<blocks, 128, 0, st>>>(*d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C, m->nbr,
                                                 m->F, m->K, t_rows, t_cols, t_vals, n, do_clamp, clamp_lo,
                                                 clamp_hi, unscale, sqerr_scratch, 0);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, n <= (1LL << 22), st);
}

extern "C" int culsh_rmse32(const CulshData *d, const CulshModel32 *m, const int32_t *nbr,
                            const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                            double *sqerr_scratch, double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 127) / 128, (int64_t)num_sms() * 16);
    sqerr_kernel<float><<<blocks, 128, 0, st>>>(*d, (double)m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                nbr, m->F, m->K, t_rows, t_cols, t_vals, n, 0, 0.0, 0.0, 1.0,
                                                sqerr_scratch, 0);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, false, st);
}

extern "C" int culsh_predict(const CulshData *d, const CulshModel64 *m, const int32_t *rows,
                             const int32_t *cols, int64_t n, double *out, void *stream) {
    if (n <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 127) / 128, (int64_t)num_sms() * 16);
    sqerr_kernel<double><<<blocks, 128, 0, st>>>(*d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C, m->nbr,
                                                 m->F, m->K, rows, cols, nullptr, n, 0, 0.0, 0.0, 1.0, out, 1);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
