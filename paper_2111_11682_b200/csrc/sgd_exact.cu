// Deterministic serial-order SGD.
//
// Reproduces the reference's fp64 column-major passes bit for bit:
//   train_full       -> _full_pass_block over all columns       factorization.py:332-363
//   parallel_train   -> D stages of D disjoint blocks             parallel.py:110-128,186-215
//   train_incremental-> _online_row_pass / _online_col_pass      online.py:230-271
// with _update_one's exact operation order (factorization.py:266-329).  This
// translation unit is compiled with -fmad=false so no product is fused into an
// add, matching numba's fastmath-off code.
//
// Parallel schedule (a dependency wavefront, not a reordering): an update (i, j)
// depends only on the previous update of row i (an earlier column) and of
// column j (the previous entry of the same column).  One warp owns a column for
// the whole pass and walks it in order; columns are handed out in ascending
// order through a ticket counter, and before touching row i a warp waits until
// row i's previous updater column (its CSR predecessor inside the pass) has
// published.  The smallest active column never waits on an unfinished one, so
// the schedule is deadlock-free for any grid size, and the result equals the
// serial order exactly.
#include "common.cuh"

namespace culsh {

struct ExactModel {
    const int64_t *col_ptr;
    const int32_t *col_rows;
    const double *col_vals;
    const int64_t *row_ptr;
    const int32_t *row_cols;
    const double *row_vals;
    const int32_t *csc2csr;
    double mu;
    double *b, *bhat, *U, *V, *W, *C;
    const int32_t *nbr;
    const double *base_b, *base_bhat;
    int F, K;
};

// factorization.py:218-232 _lookup (binary search in row i's sorted CSR columns)
__device__ __forceinline__ bool lookup(const int64_t *row_ptr, const int32_t *row_cols,
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

// Sequential (reference-order) scalar part of _update_one, evaluated redundantly by
// every lane from the per-lane products staged in shared memory.
struct Scalars {
    double e, inv_r, inv_n;
};

// variant bit 0: basic-MF summation (factorization.py:375-379: pred starts at the
//   bias sum and the products are added to it one by one, no separate dot);
// variant bit 1: the pass runs on the transposed matrix (rows as columns, for the
//   row-major basic pass) -- the reference's bias sum is (mu + b_i) + b_hat_j with
//   b_i then being the register-resident side.
__device__ __forceinline__ Scalars exact_error(const double *buf, int F, int K, const uint32_t *emask,
                                               double mu, double bi, double bhj, double r, int variant) {
    double pred = (variant & 2) ? mu + bhj + bi : mu + bi + bhj;
    if (variant & 1) {
        for (int f = 0; f < F; ++f) pred = pred + buf[f];
    } else {
        double dot = 0.0;
        for (int f = 0; f < F; ++f) dot = dot + buf[f];
        pred = pred + dot;
    }
    int nr = 0, nn = 0;
    double sw = 0.0, sc = 0.0;
    for (int k = 0; k < K; ++k) {
        if ((emask[k >> 5] >> (k & 31)) & 1u) { ++nr; sw = sw + buf[F + k]; }
        else { ++nn; sc = sc + buf[F + k]; }
    }
    if (nr > 0) pred = pred + sw / sqrt((double)nr);
    if (nn > 0) pred = pred + sc / sqrt((double)nn);
    Scalars s;
    s.e = r - pred;
    s.inv_r = nr > 0 ? 1.0 / sqrt((double)nr) : 0.0;
    s.inv_n = nn > 0 ? 1.0 / sqrt((double)nn) : 0.0;
    return s;
}

// Precomputed neighbour lookups of a column range (culsh_exact_lookup): per CSC entry
// idx, KPL mask words at mask[(idx - base) * KPL] (bit k: row i rated J[j,k]) and the
// looked-up ratings rv[(idx - base) * K + k].  With them the column kernel's per-update
// critical path loses its K dependent binary searches; the values are the same reads.
struct ExactPre {
    const uint32_t *mask;
    const double *rv;
    int64_t base;
};

template <int FPL, int KPL>
__global__ void __launch_bounds__(256)
exact_col_kernel(ExactModel P, CulshRates R, const int64_t *__restrict__ seg,
                 const int32_t *__restrict__ chain_lo, int64_t col_lo, int64_t col_hi, int row_mode,
                 int64_t M_old, int variant, int *__restrict__ row_last, int *__restrict__ ticket,
                 int *__restrict__ status, ExactPre pre) {
    extern __shared__ double s_buf[];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int F = P.F, K = P.K;
    double *buf = s_buf + (size_t)warp * (F + K);
    const double mu = P.mu;

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int64_t j = col_lo + t;
        if (j >= col_hi) break;
        if (ld_volatile(status)) break;

        double v[FPL], w[KPL], c[KPL], bbn[KPL];
        int32_t nb[KPL];
#pragma unroll
        for (int q = 0; q < FPL; ++q) {
            const int f = lane + 32 * q;
            v[q] = f < F ? P.V[j * F + f] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            w[q] = k < K ? P.W[j * K + k] : 0.0;
            c[q] = k < K ? P.C[j * K + k] : 0.0;
            nb[q] = k < K ? P.nbr[j * K + k] : 0;
            bbn[q] = k < K ? P.base_bhat[nb[q]] : 0.0;
        }
        double bhj = P.bhat[j];
        const int32_t cl = chain_lo ? chain_lo[j] : (int32_t)col_lo;
        const int64_t lo = seg[2 * j], hi = seg[2 * j + 1];
        bool stop = false;

        for (int64_t idx = lo; idx < hi && !stop; ++idx) {
            const int32_t i = P.col_rows[idx];
            const double r = P.col_vals[idx];
            const bool upd_row = row_mode == 1 || (row_mode == 2 && i >= M_old);

            // neighbour lookups: independent of the parameters, issued before the wait
            const double bbi = P.base_b[i];
            bool expl[KPL];
            double resid[KPL];
            uint32_t emask[KPL];
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                double rv = 0.0;
                if (pre.mask) {
                    const int64_t li = idx - pre.base;
                    expl[q] = k < K && ((__ldg(pre.mask + li * KPL + q) >> lane) & 1u);
                    if (expl[q]) rv = __ldg(pre.rv + li * K + k);
                } else {
                    expl[q] = k < K && lookup(P.row_ptr, P.row_cols, P.row_vals, i, nb[q], &rv);
                }
                resid[q] = expl[q] ? rv - (mu + bbi + bbn[q]) : 0.0;
                emask[q] = __ballot_sync(0xffffffffu, expl[q]);
            }

            if (upd_row) {
                const int64_t pos = P.csc2csr[idx];
                int32_t pc = pos > P.row_ptr[i] ? P.row_cols[pos - 1] : -1;
                if (pc < cl) pc = -1;
                if (pc >= 0 && lane == 0) {
                    // watchdog: a predecessor that never publishes means the caller's plan
                    // is inconsistent; report (status bit 2) instead of hanging the GPU
                    const uint64_t t0 = global_ns();
                    while (ld_acquire(&row_last[i]) < pc) {
                        if (ld_volatile(status)) break;
                        if (global_ns() - t0 > 20000000000ULL) { atomicOr(status, 2); break; }
                        __nanosleep(32);
                    }
                }
                __syncwarp();
            }
            double u[FPL];
#pragma unroll
            for (int q = 0; q < FPL; ++q) {
                const int f = lane + 32 * q;
                u[q] = f < F ? __ldcg(&P.U[(int64_t)i * F + f]) : 0.0;
                if (f < F) buf[f] = u[q] * v[q];
            }
            const double bi = __ldcg(&P.b[i]);
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                if (k < K) buf[F + k] = expl[q] ? resid[q] * w[q] : c[q];
            }
            __syncwarp();
            const Scalars s = exact_error(buf, F, K, emask, mu, bi, bhj, r, variant);
            const double e = s.e;
            if (!isfinite(e)) {
                if (lane == 0) atomicOr(status, 1);
                stop = true;
            }
            // factorization.py:307-328 update rules, same expressions
            if (upd_row) {
                const double bn = bi + R.gb * (e - R.lb * bi);
#pragma unroll
                for (int q = 0; q < FPL; ++q) {
                    const int f = lane + 32 * q;
                    const double uf = u[q], vf = v[q];
                    if (f < F) {
                        __stcg(&P.U[(int64_t)i * F + f], uf + R.gu * (e * vf - R.lu * uf));
                        v[q] = vf + R.gv * (e * uf - R.lv * vf);
                    }
                }
                if (lane == 0) __stcg(&P.b[i], bn);
            } else {
#pragma unroll
                for (int q = 0; q < FPL; ++q) {
                    const int f = lane + 32 * q;
                    if (f < F) v[q] = v[q] + R.gv * (e * u[q] - R.lv * v[q]);
                }
            }
            bhj = bhj + R.gbh * (e - R.lbh * bhj);
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                if (k < K) {
                    if (expl[q]) w[q] = w[q] + R.gw * (s.inv_r * e * resid[q] - R.lw * w[q]);
                    else c[q] = c[q] + R.gc * (s.inv_n * e - R.lc * c[q]);
                }
            }
            if (upd_row) {
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(&row_last[i], (int)j);
            }
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < FPL; ++q) {
            const int f = lane + 32 * q;
            if (f < F) P.V[j * F + f] = v[q];
        }
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            if (k < K) {
                P.W[j * K + k] = w[q];
                P.C[j * K + k] = c[q];
            }
        }
        if (lane == 0) P.bhat[j] = bhj;
        if (stop) break;
    }
}

// online.py:230-250 _online_row_pass: rows are independent (column parameters are
// read-only in this phase); one warp per row walks its CSR entries in order.
template <int FPL, int KPL>
__global__ void __launch_bounds__(256)
exact_row_kernel(ExactModel P, CulshRates R, int64_t row_lo, int64_t row_hi, int64_t N_old,
                 int *__restrict__ status) {
    extern __shared__ double s_buf[];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int F = P.F, K = P.K;
    double *buf = s_buf + (size_t)warp * (F + K);
    const double mu = P.mu;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = row_lo + blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; i < row_hi; i += nwarps) {
        double u[FPL];
#pragma unroll
        for (int q = 0; q < FPL; ++q) {
            const int f = lane + 32 * q;
            u[q] = f < F ? P.U[i * F + f] : 0.0;
        }
        double bi = P.b[i];
        const double bbi = P.base_b[i];
        bool stop = false;
        for (int64_t idx = P.row_ptr[i]; idx < P.row_ptr[i + 1] && !stop; ++idx) {
            const int32_t j = P.row_cols[idx];
            if (j >= N_old) continue;
            const double r = P.row_vals[idx];
            double v[FPL], w[KPL], c[KPL], resid[KPL];
            bool expl[KPL];
            uint32_t emask[KPL];
#pragma unroll
            for (int q = 0; q < FPL; ++q) {
                const int f = lane + 32 * q;
                v[q] = f < F ? P.V[(int64_t)j * F + f] : 0.0;
                if (f < F) buf[f] = u[q] * v[q];
            }
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int k = lane + 32 * q;
                double rv = 0.0;
                int32_t j1 = k < K ? P.nbr[(int64_t)j * K + k] : 0;
                expl[q] = k < K && lookup(P.row_ptr, P.row_cols, P.row_vals, i, j1, &rv);
                resid[q] = expl[q] ? rv - (mu + bbi + P.base_bhat[j1]) : 0.0;
                w[q] = k < K ? P.W[(int64_t)j * K + k] : 0.0;
                c[q] = k < K ? P.C[(int64_t)j * K + k] : 0.0;
                emask[q] = __ballot_sync(0xffffffffu, expl[q]);
                if (k < K) buf[F + k] = expl[q] ? resid[q] * w[q] : c[q];
            }
            __syncwarp();
            const Scalars s = exact_error(buf, F, K, emask, mu, bi, P.bhat[j], r, 0);
            const double e = s.e;
            if (!isfinite(e)) {
                if (lane == 0) atomicOr(status, 1);
                stop = true;
            }
            bi = bi + R.gb * (e - R.lb * bi);
#pragma unroll
            for (int q = 0; q < FPL; ++q) u[q] = u[q] + R.gu * (e * v[q] - R.lu * u[q]);
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < FPL; ++q) {
            const int f = lane + 32 * q;
            if (f < F) P.U[i * F + f] = u[q];
        }
        if (lane == 0) P.b[i] = bi;
    }
}

// Per-column entry ranges [seg[2j], seg[2j+1]) and row-chain cut-offs for one pass.
// mode 0: rows [row_lo,row_hi) of columns [col_lo,col_hi), chains start at col_lo
//         (factorization.py:346-355; online.py:262-263 with row range = all rows)
// mode 1: DSGD stage s of D: column j in block d takes row block (d+s)%D
//         (parallel.py:36-41,197-207); chains start at the block's first column
__global__ void plan_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                            int64_t N, int mode, int64_t col_lo, int64_t col_hi, int64_t row_lo,
                            int64_t row_hi, const int64_t *__restrict__ block_ptr,
                            const int64_t *__restrict__ col_bounds, int D, int s,
                            int64_t *__restrict__ seg, int32_t *__restrict__ chain_lo) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = 0, c = 0;
        int32_t cl = 0;
        if (mode == 0) {
            if (j >= col_lo && j < col_hi) {
                const int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
                a = lo;
                c = hi;
                if (row_lo > 0) {
                    int64_t l = lo, h = hi;
                    while (l < h) { int64_t m = (l + h) / 2; if (col_rows[m] < row_lo) l = m + 1; else h = m; }
                    a = l;
                }
                int64_t l = a, h = hi;
                while (l < h) { int64_t m = (l + h) / 2; if (col_rows[m] < row_hi) l = m + 1; else h = m; }
                c = l;
            }
            cl = (int32_t)col_lo;
        } else {
            int d = 0;
            while (d + 1 < D && j >= col_bounds[d + 1]) ++d;
            const int rb = (d + s) % D;
            a = block_ptr[j * (D + 1) + rb];
            c = block_ptr[j * (D + 1) + rb + 1];
            cl = (int32_t)col_bounds[d];
        }
        seg[2 * j] = a;
        seg[2 * j + 1] = c;
        chain_lo[j] = cl;
    }
}

// parallel.py:55-64 _block_pointers
__global__ void block_pointers_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                                      int64_t N, const int64_t *__restrict__ row_bounds, int nb,
                                      int64_t *__restrict__ out) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N * nb;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = x / nb;
        const int r = (int)(x % nb);
        int64_t l = col_ptr[j], h = col_ptr[j + 1];
        const int64_t v = row_bounds[r];
        while (l < h) { int64_t m = (l + h) / 2; if (col_rows[m] < v) l = m + 1; else h = m; }
        out[x] = l;
    }
}

// Neighbour lookups of every entry of columns [col_lo, col_hi): warp per entry (grid
// stride), lane k searches J[j,k] in row i (the _lookup of factorization.py:218-232).
__global__ void exact_lookup_kernel(ExactModel P, int64_t col_lo, int64_t col_hi, int KPL,
                                    uint32_t *__restrict__ mask, double *__restrict__ rv) {
    const unsigned lane = lane_id();
    const int K = P.K;
    const int64_t e_lo = P.col_ptr[col_lo], e_hi = P.col_ptr[col_hi];
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = e_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < e_hi; e += warps) {
        int64_t lo = col_lo, hi = col_hi;   // column of entry e: last j with col_ptr[j] <= e
        while (hi - lo > 1) {
            const int64_t m = (lo + hi) >> 1;
            if (P.col_ptr[m] <= e) lo = m; else hi = m;
        }
        const int64_t j = lo;
        const int32_t i = P.col_rows[e];
        for (int q = 0; q < KPL; ++q) {
            const int k = (int)lane + 32 * q;
            double v = 0.0;
            const bool hit = k < K && lookup(P.row_ptr, P.row_cols, P.row_vals, i, P.nbr[j * K + k], &v);
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (lane == 0) mask[(e - e_lo) * KPL + q] = bal;
            if (k < K) rv[(e - e_lo) * K + k] = v;
        }
    }
}

template <int FPL, int KPL>
int launch_col(const ExactModel &P, const CulshRates &R, const int64_t *seg, const int32_t *chain_lo,
               int64_t col_lo, int64_t col_hi, int row_mode, int64_t M_old, int variant, int *row_last,
               int *ticket, int *status, cudaStream_t st, ExactPre pre) {
    const int threads = 128;
    const size_t smem = (size_t)(threads / 32) * (P.F + P.K) * sizeof(double);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, exact_col_kernel<FPL, KPL>, threads, smem);
    if (occ < 1) occ = 1;
    const int64_t ncols = col_hi - col_lo;
    int64_t blocks = (int64_t)num_sms() * occ;
    const int64_t need = (ncols + (threads / 32) - 1) / (threads / 32);
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    exact_col_kernel<FPL, KPL><<<(unsigned)blocks, threads, smem, st>>>(
        P, R, seg, chain_lo, col_lo, col_hi, row_mode, M_old, variant, row_last, ticket, status, pre);
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

template <int FPL, int KPL>
int launch_row(const ExactModel &P, const CulshRates &R, int64_t row_lo, int64_t row_hi, int64_t N_old,
               int *status, cudaStream_t st) {
    const int threads = 128;
    const size_t smem = (size_t)(threads / 32) * (P.F + P.K) * sizeof(double);
    int64_t blocks = (row_hi - row_lo + 3) / 4;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) return CULSH_OK;
    exact_row_kernel<FPL, KPL><<<(unsigned)blocks, threads, smem, st>>>(P, R, row_lo, row_hi, N_old, status);
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

// explicit-neighbour mask words per rating: 1 (K <= 32), 2 (K <= 64), 4 (K <= 128, the
// top-K kernels' bound; the reference's K is unbounded)
__host__ __device__ constexpr int exact_kpl(int K) { return K <= 32 ? 1 : K <= 64 ? 2 : 4; }

#define CULSH_DISPATCH_FK(F, K, CALL)                                  \
    do {                                                               \
        const int _fpl = (F) <= 32 ? 1 : (F) <= 64 ? 2 : (F) <= 128 ? 4 : (F) <= 256 ? 8 : 16; \
        const int _kpl = exact_kpl(K);                                 \
        if (_fpl == 1 && _kpl == 1) return CALL(1, 1);                 \
        if (_fpl == 1 && _kpl == 2) return CALL(1, 2);                 \
        if (_fpl == 1 && _kpl == 4) return CALL(1, 4);                 \
        if (_fpl == 2 && _kpl == 1) return CALL(2, 1);                 \
        if (_fpl == 2 && _kpl == 2) return CALL(2, 2);                 \
        if (_fpl == 2 && _kpl == 4) return CALL(2, 4);                 \
        if (_fpl == 4 && _kpl == 1) return CALL(4, 1);                 \
        if (_fpl == 4 && _kpl == 2) return CALL(4, 2);                 \
        if (_fpl == 4 && _kpl == 4) return CALL(4, 4);                 \
        if (_fpl == 8 && _kpl == 1) return CALL(8, 1);                 \
        if (_fpl == 8 && _kpl == 2) return CALL(8, 2);                 \
        if (_fpl == 8 && _kpl == 4) return CALL(8, 4);                 \
        if (_fpl == 16 && _kpl == 1) return CALL(16, 1);               \
        if (_fpl == 16 && _kpl == 2) return CALL(16, 2);               \
        return CALL(16, 4);                                            \
    } while (0)

}  // namespace culsh

using namespace culsh;

static ExactModel make_model(const CulshData *d, const CulshModel64 *m) {
    ExactModel P;
    P.col_ptr = d->col_ptr;
    P.col_rows = d->col_rows;
    P.col_vals = d->col_vals;
    P.row_ptr = d->row_ptr;
    P.row_cols = d->row_cols;
    P.row_vals = d->row_vals;
    P.csc2csr = d->csc2csr;
    P.mu = m->mu;
    P.b = m->b;
    P.bhat = m->bhat;
    P.U = m->U;
    P.V = m->V;
    P.W = m->W;
    P.C = m->C;
    P.nbr = m->nbr;
    P.base_b = d->base_b;
    P.base_bhat = d->base_bhat;
    P.F = m->F;
    P.K = m->K;
    return P;
}

extern "C" int culsh_block_pointers(const int64_t *col_ptr, const int32_t *col_rows, int64_t N,
                                    const int64_t *row_bounds, int nb, int64_t *out, void *stream) {
    if (N <= 0) return CULSH_OK;
    const int64_t total = N * nb;
    const int blocks = (int)min64((total + 255) / 256, (int64_t)num_sms() * 8);
    block_pointers_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(col_ptr, col_rows, N, row_bounds, nb, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_pass_plan(const int64_t *col_ptr, const int32_t *col_rows, int64_t N, int mode,
                               int64_t col_lo, int64_t col_hi, int64_t row_lo, int64_t row_hi,
                               const int64_t *block_ptr, const int64_t *col_bounds, int D, int s,
                               int64_t *seg, int32_t *chain_lo, void *stream) {
    if (N <= 0) return CULSH_OK;
    CULSH_REQUIRE(mode == 0 || (block_ptr && col_bounds && D >= 1), "bad pass plan");
    const int blocks = (int)min64((N + 255) / 256, (int64_t)num_sms() * 8);
    plan_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(col_ptr, col_rows, N, mode, col_lo, col_hi,
                                                          row_lo, row_hi, block_ptr, col_bounds, D, s,
                                                          seg, chain_lo);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

static int exact_colpass_impl(const CulshData *d, CulshModel64 *m, const CulshRates *r, const int64_t *seg,
                              const int32_t *chain_lo, int64_t col_lo, int64_t col_hi, int row_mode,
                              int64_t M_old, int variant, int *row_last, int *ticket, int *status, void *stream,
                              ExactPre pre) {
    CULSH_REQUIRE(m->F >= 1 && m->F <= 512, "F must be in [1, 512]");
    CULSH_REQUIRE(m->K >= 0 && m->K <= 128, "K must be in [0, 128]");
    if (col_hi <= col_lo) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CULSH_CHECK(cudaMemsetAsync(row_last, 0xFF, sizeof(int) * d->M, st));
    CULSH_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const ExactModel P = make_model(d, m);
    const CulshRates R = *r;
#define CALL_COL(a, b) launch_col<a, b>(P, R, seg, chain_lo, col_lo, col_hi, row_mode, M_old, variant, row_last, ticket, status, st, pre)
    CULSH_DISPATCH_FK(m->F, m->K, CALL_COL);
#undef CALL_COL
}

extern "C" int culsh_sgd_exact_colpass(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                                       const int64_t *seg, const int32_t *chain_lo, int64_t col_lo,
                                       int64_t col_hi, int row_mode, int64_t M_old, int variant,
                                       int *row_last, int *ticket, int *status, void *stream) {
    return exact_colpass_impl(d, m, r, seg, chain_lo, col_lo, col_hi, row_mode, M_old, variant, row_last, ticket,
                              status, stream, ExactPre{nullptr, nullptr, 0});
}

extern "C" int culsh_exact_lookup(const CulshData *d, const CulshModel64 *m, int64_t col_lo, int64_t col_hi,
                                  uint32_t *mask, double *rv, void *stream) {
    CULSH_REQUIRE(m->K >= 1 && m->K <= 128, "K must be in [1, 128]");
    if (col_hi <= col_lo) return CULSH_OK;
    const ExactModel P = make_model(d, m);
    const int KPL = exact_kpl(m->K);
    exact_lookup_kernel<<<(unsigned)(num_sms() * 16), 256, 0, (cudaStream_t)stream>>>(P, col_lo, col_hi, KPL,
                                                                                     mask, rv);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_sgd_exact_colpass_pre(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                                           const int64_t *seg, const int32_t *chain_lo, int64_t col_lo,
                                           int64_t col_hi, int row_mode, int64_t M_old, int variant,
                                           int *row_last, int *ticket, int *status, const uint32_t *pre_mask,
                                           const double *pre_rv, int64_t pre_base, void *stream) {
    CULSH_REQUIRE(pre_mask != nullptr && pre_rv != nullptr, "precomputed lookups missing");
    return exact_colpass_impl(d, m, r, seg, chain_lo, col_lo, col_hi, row_mode, M_old, variant, row_last, ticket,
                              status, stream, ExactPre{pre_mask, pre_rv, pre_base});
}

extern "C" int culsh_sgd_exact_rowpass(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                                       int64_t row_lo, int64_t row_hi, int64_t N_old, int *status,
                                       void *stream) {
    CULSH_REQUIRE(m->F >= 1 && m->F <= 512, "F must be in [1, 512]");
    CULSH_REQUIRE(m->K >= 0 && m->K <= 128, "K must be in [0, 128]");
    if (row_hi <= row_lo) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const ExactModel P = make_model(d, m);
    const CulshRates R = *r;
#define CALL_ROW(a, b) launch_row<a, b>(P, R, row_lo, row_hi, N_old, status, st)
    CULSH_DISPATCH_FK(m->F, m->K, CALL_ROW);
#undef CALL_ROW
}
