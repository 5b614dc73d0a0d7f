// Device-side index helpers for SparseRatings (data.py:166-207).
#include "common.cuh"

namespace culsh {

// csc2csr[idx]: position of CSC entry (i, j) inside row i's CSR segment (rows are
// sorted by column, data.py:189-194), found by binary search.
__global__ void csc2csr_kernel(CulshData d, int32_t *__restrict__ out) {
    for (int64_t j = blockIdx.x; j < d.N; j += gridDim.x) {
        for (int64_t idx = d.col_ptr[j] + threadIdx.x; idx < d.col_ptr[j + 1]; idx += blockDim.x) {
            const int32_t i = d.col_rows[idx];
            int64_t lo = d.row_ptr[i], hi = d.row_ptr[i + 1];
            while (lo < hi) {
                const int64_t m = (lo + hi) >> 1;
                if (d.row_cols[m] < j) lo = m + 1; else hi = m;
            }
            out[idx] = (int32_t)lo;
        }
    }
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_csc_to_csr_map(const CulshData *d, int32_t *csc2csr, void *stream) {
    CULSH_REQUIRE(d->nnz < (1LL << 31), "nnz must be < 2^31");
    if (d->N <= 0 || d->nnz == 0) return CULSH_OK;
    const int blocks = (int)min64(d->N, (int64_t)num_sms() * 16);
    csc2csr_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(*d, csc2csr);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

namespace culsh {

// out segment s = old segment s (s < n_old) followed by add segment s; out_ptr is
// (n_total+1).  One warp per segment, coalesced copies.  Used to append an online
// increment to both index views (new rows / columns sort after the old ones, so
// every merged segment stays sorted; online.py:84-93 rebuilds instead).
__global__ void append_segments_kernel(int64_t n_old, int64_t n_total, const int64_t *__restrict__ old_ptr,
                                       const int32_t *__restrict__ old_idx, const double *__restrict__ old_val,
                                       const int64_t *__restrict__ add_ptr, const int32_t *__restrict__ add_idx,
                                       const double *__restrict__ add_val, int64_t *__restrict__ out_ptr,
                                       int32_t *__restrict__ out_idx, double *__restrict__ out_val) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const unsigned lane = lane_id();
    for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s <= n_total; s += warps) {
        const int64_t o_lo = old_ptr[min64(s, n_old)];
        const int64_t base = o_lo + add_ptr[s];
        if (lane == 0) out_ptr[s] = base;
        if (s == n_total) continue;
        const int64_t o_hi = s < n_old ? old_ptr[s + 1] : o_lo;
        const int64_t a_lo = add_ptr[s], a_hi = add_ptr[s + 1];
        for (int64_t x = lane; x < o_hi - o_lo; x += 32) {
            out_idx[base + x] = old_idx[o_lo + x];
            out_val[base + x] = old_val[o_lo + x];
        }
        const int64_t b2 = base + (o_hi - o_lo);
        for (int64_t x = lane; x < a_hi - a_lo; x += 32) {
            out_idx[b2 + x] = add_idx[a_lo + x];
            out_val[b2 + x] = add_val[a_lo + x];
        }
    }
}

}  // namespace culsh

extern "C" int culsh_append_segments(int64_t n_old, int64_t n_total, const int64_t *old_ptr,
                                     const int32_t *old_idx, const double *old_val, const int64_t *add_ptr,
                                     const int32_t *add_idx, const double *add_val, int64_t *out_ptr,
                                     int32_t *out_idx, double *out_val, void *stream) {
    CULSH_REQUIRE(n_old >= 0 && n_total >= n_old, "bad segment counts");
    const int blocks = (int)min64((n_total + 1 + 7) / 8, (int64_t)num_sms() * 16);
    append_segments_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_old, n_total, old_ptr, old_idx, old_val,
                                                                      add_ptr, add_idx, add_val, out_ptr,
                                                                      out_idx, out_val);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

namespace culsh {

// After appending an increment to both views: an old CSC entry (i, j) keeps its
// place inside row i (new entries of row i have columns >= n_old_cols > j) and
// shifts by the add entries of the rows before i, i.e. by add_row_ptr[i]; the
// added entries are located by binary search in the merged row view.
__global__ void append_map_kernel(CulshData d, int64_t n_old_cols, const int64_t *__restrict__ old_col_ptr,
                                  const int32_t *__restrict__ old_map, const int64_t *__restrict__ add_row_ptr,
                                  int64_t M_old, int32_t *__restrict__ out) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const unsigned lane = lane_id();
    for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < d.N; j += warps) {
        const int64_t lo = d.col_ptr[j], hi = d.col_ptr[j + 1];
        int64_t n_keep = 0, o_lo = 0;
        if (j < n_old_cols) {
            o_lo = old_col_ptr[j];
            n_keep = old_col_ptr[j + 1] - o_lo;
        }
        for (int64_t x = lane; x < hi - lo; x += 32) {
            const int32_t i = d.col_rows[lo + x];
            int64_t pos;
            if (x < n_keep && i < M_old) {
                pos = (int64_t)old_map[o_lo + x] + add_row_ptr[i];
            } else {
                int64_t a = d.row_ptr[i], b = d.row_ptr[i + 1];
                while (a < b) {
                    const int64_t m = (a + b) >> 1;
                    if (d.row_cols[m] < j) a = m + 1; else b = m;
                }
                pos = a;
            }
            out[lo + x] = (int32_t)pos;
        }
    }
}

// out[s] = sum of val[ptr[s] .. ptr[s+1]) (warp per segment; exact for integer data).
__global__ void segment_sums_kernel(int64_t n, const int64_t *__restrict__ ptr, const double *__restrict__ val,
                                    double *__restrict__ out) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const unsigned lane = lane_id();
    for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < n; s += warps) {
        double acc = 0.0;
        for (int64_t x = ptr[s] + lane; x < ptr[s + 1]; x += 32) acc += val[x];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[s] = acc;
    }
}

}  // namespace culsh

extern "C" int culsh_append_csc2csr(const CulshData *d, int64_t n_old_cols, const int64_t *old_col_ptr,
                                    const int32_t *old_map, const int64_t *add_row_ptr, int64_t M_old,
                                    int32_t *csc2csr, void *stream) {
    CULSH_REQUIRE(d->nnz < (1LL << 31), "nnz must be < 2^31");
    CULSH_REQUIRE(n_old_cols >= 0 && n_old_cols <= d->N && M_old >= 0 && M_old <= d->M, "bad old shape");
    if (d->N <= 0 || d->nnz == 0) return CULSH_OK;
    const int blocks = (int)min64((d->N + 7) / 8, (int64_t)num_sms() * 16);
    append_map_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*d, n_old_cols, old_col_ptr, old_map,
                                                                 add_row_ptr, M_old, csc2csr);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_segment_sums(int64_t n, const int64_t *ptr, const double *val, double *out, void *stream) {
    CULSH_REQUIRE(n >= 0, "bad segment count");
    if (n == 0) return CULSH_OK;
    const int blocks = (int)min64((n + 7) / 8, (int64_t)num_sms() * 16);
    segment_sums_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, ptr, val, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
