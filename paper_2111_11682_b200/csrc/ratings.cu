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
