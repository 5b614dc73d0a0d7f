// Evaluation: exact fp64 prediction and RMSE.
// pred_tile_kernel restates factorization.py:235-263 _predict_one in its exact operation
// order (explicit _rn intrinsics; the TU is also compiled with -fmad=false); the RMSE sum
// is the reference's sequential one (bit-identical to factorization.py:394-409, at any n:
// seq_sum_exact) when `sequential` is set, otherwise a fixed pairwise tree.
#include <type_traits>

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

// Sequential sum in index order (the reference's serial loop, bit-exact).  The chain of
// dependent adds cannot be parallelised, but its operands can be staged: warps 1..31
// copy the next 2048-element chunk into shared memory while lane 0 of warp 0 adds the
// current one, so the loop runs at add latency instead of global-load latency (1M adds:
// 5.9 ms with the shared loads issued next to their adds, see the group loop below).
__global__ void __launch_bounds__(1024) seq_sum_kernel(const double *__restrict__ x, int64_t n,
                                                       double *out) {
    constexpr int CH = 2048;
    __shared__ __align__(16) double buf[2][CH];
    const int tid = threadIdx.x;
    double total = 0.0;
    const int64_t nch = (n + CH - 1) / CH;
    for (int k = tid; k < CH; k += blockDim.x) buf[0][k] = k < n ? x[k] : 0.0;
    __syncthreads();
    for (int64_t c = 0; c < nch; ++c) {
        const int cur = (int)(c & 1);
        if (tid >= 32) {
            const int64_t base = (c + 1) * CH;
            if (base < n)
                for (int k = tid - 32; k < CH; k += blockDim.x - 32)
                    buf[cur ^ 1][k] = base + k < n ? x[base + k] : 0.0;
        } else if (tid == 0) {
            // the chunk's tail is zero-filled and every addend is a square (>= +0, never -0),
            // so whole groups of 16 add the same bits; the next group's shared loads are in
            // flight while the current group's 16 dependent adds run
            const int m = ((int)min64(CH, n - c * CH) + 15) & ~15;
            const double2 *b = reinterpret_cast<const double2 *>(buf[cur]);
            double2 a[8], nx[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = b[q];
            for (int k = 0; k < m; k += 16) {
                const int kn = k + 16 < m ? k + 16 : k;
#pragma unroll
                for (int q = 0; q < 8; ++q) nx[q] = b[(kn >> 1) + q];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    total = __dadd_rn(total, a[q].x);
                    total = __dadd_rn(total, a[q].y);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) a[q] = nx[q];
            }
        }
        __syncthreads();
    }
    if (tid == 0) *out = sqrt(total / (double)n);
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

// ---- warp-tiled prediction ---------------------------------------------------------
// A warp evaluates 32 ratings at once, lane l owning rating l.  The dot product's
// operands are read cooperatively (for each rating r of the group, lane f loads U[i_r, f]
// and V[j_r, f]: one coalesced row segment instead of 32 scattered per-lane walks), the
// products go through a per-warp 32x33 shared tile, and lane l then adds its rating's
// products in f order -- the reference's sequential fp64 sum, so predictions are
// bit-identical to predict_one.  The neighbour part is lane-local: rating values either
// by binary search in the CSR row (any triplets) or from the per-fit lookup cache of the
// training set (PRE: explicit-neighbour mask + CSC positions of the rated neighbours).
struct PreLookup {
    const uint32_t *mask;        // (nnz * MW) explicit-neighbour bits per CSC entry
    const int64_t *group_base;   // first pos index of each 32-entry group
    const int32_t *pos;          // CSC position of r(i, J[j, k]) per explicit pair, CSC order
    const int64_t *perm;         // entry index of each CSC position (nullptr: identity)
    int MW;
};

__device__ __forceinline__ int64_t column_of(const int64_t *col_ptr, int64_t N, int64_t e) {
    int64_t lo = 0, hi = N;   // last j with col_ptr[j] <= e
    while (hi - lo > 1) {
        const int64_t m = (lo + hi) >> 1;
        if (__ldg(col_ptr + m) <= e) lo = m; else hi = m;
    }
    return lo;
}

constexpr int kTileLd = 33;

template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// WARPS per block; PRE: training set (CSC entries, V rows mostly shared by the group ->
// read directly), else any triplets (V rows staged like U's).
template <typename P, bool PRE>
__global__ void __launch_bounds__(PRE ? 128 : 64) pred_tile_kernel(CulshData d, double mu, const P *__restrict__ b,
                                                        const P *__restrict__ bhat, const P *__restrict__ U,
                                                        const P *__restrict__ V, const P *__restrict__ W,
                                                        const P *__restrict__ C, const int32_t *__restrict__ nbr,
                                                        int F, int ldF, int K, const int32_t *__restrict__ t_rows,
                                                        const int32_t *__restrict__ t_cols,
                                                        const double *__restrict__ t_vals, int64_t n, PreLookup pre,
                                                        int mode, int do_clamp, double lo, double hi,
                                                        double unscale, double *__restrict__ out) {
    constexpr int WPB = PRE ? 4 : 2;
    constexpr int NT = PRE ? 1 : 2;
    __shared__ P tiles[WPB][NT][32 * kTileLd];
    P *ut = tiles[threadIdx.x >> 5][0];
    P *vt = tiles[threadIdx.x >> 5][NT - 1];
    const int lane = (int)lane_id();
    const int64_t warps = (int64_t)gridDim.x * WPB;
    for (int64_t g = (int64_t)blockIdx.x * WPB + (threadIdx.x >> 5); g * 32 < n; g += warps) {
        const int64_t e = g * 32 + lane;
        const bool valid = e < n;
        int64_t i = 0, j = 0;
        if (valid) {
            if (PRE) {
                i = d.col_rows[e];
                j = column_of(d.col_ptr, d.N, e);
            } else {
                i = t_rows[e];
                j = t_cols[e];
            }
        }
        double pred = valid ? __dadd_rn(__dadd_rn(mu, (double)b[i]), (double)bhat[j]) : 0.0;
        double dot = 0.0;
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        for (int f0 = 0; f0 < F; f0 += 32) {
            const int f = f0 + lane;
            // stage this f-chunk of the group's U (and V) rows: all 32 row segments in flight
            // at once (cp.async, no register staging); lane f fills column f of the tile
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
                if (!((vmask >> r) & 1u)) continue;          // warp-uniform
                const int64_t ir = __shfl_sync(0xffffffffu, i, r);
                const int64_t jr = PRE ? 0 : __shfl_sync(0xffffffffu, j, r);
                if (f < F) {
                    cp_async<sizeof(P)>(ut + lane * kTileLd + r, U + ir * ldF + f);
                    if (!PRE) cp_async<sizeof(P)>(vt + lane * kTileLd + r, V + jr * ldF + f);
                }
            }
            cp_async_wait_all();
            __syncwarp();
            const int fe = F - f0 < 32 ? F - f0 : 32;
            if (valid) {
                for (int q = 0; q < fe; ++q) {
                    const double v = PRE ? (double)__ldg(V + j * ldF + f0 + q) : (double)vt[q * kTileLd + lane];
                    dot = __dadd_rn(dot, __dmul_rn((double)ut[q * kTileLd + lane], v));
                }
            }
            __syncwarp();
        }
        pred = __dadd_rn(pred, dot);
        int nr = 0, nn = 0;
        double sw = 0.0, sc = 0.0;
        int64_t cur = 0;
        uint32_t mw0 = 0u, mw1 = 0u;
        if (PRE) {
            int pc = 0;
            if (valid && K > 0) {
                mw0 = pre.mask[e * pre.MW];
                if (pre.MW == 2) mw1 = pre.mask[e * pre.MW + 1];
                pc = __popc(mw0) + __popc(mw1);
            }
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            cur = (K > 0 ? pre.group_base[g] : 0) + incl - pc;
        }
        if (valid && K > 0) {
            const double bb = d.base_b[i];
            for (int k = 0; k < K; ++k) {
                const int32_t j1 = nbr[j * K + k];
                double rv;
                bool found;
                if (PRE) {
                    found = (((k < 32 ? mw0 : mw1) >> (k & 31)) & 1u) != 0;
                    if (found) rv = d.col_vals[pre.pos[cur++]];
                } else {
                    found = lookup_rv(d.row_ptr, d.row_cols, d.row_vals, i, j1, &rv);
                }
                if (found) {
                    ++nr;
                    sw = __dadd_rn(sw, __dmul_rn(__dsub_rn(rv, __dadd_rn(__dadd_rn(mu, bb), d.base_bhat[j1])),
                                                 (double)W[j * K + k]));
                } else {
                    ++nn;
                    sc = __dadd_rn(sc, (double)C[j * K + k]);
                }
            }
            if (nr > 0) pred = __dadd_rn(pred, __ddiv_rn(sw, __dsqrt_rn((double)nr)));
            if (nn > 0) pred = __dadd_rn(pred, __ddiv_rn(sc, __dsqrt_rn((double)nn)));
        }
        if (!valid) continue;
        if (mode == 1) {
            out[e] = pred;
            continue;
        }
        if (do_clamp) {
            if (pred < lo) pred = lo;
            else if (pred > hi) pred = hi;
        }
        const double val = PRE ? d.col_vals[e] : t_vals[e];
        const double dd = __dmul_rn(__dsub_rn(pred, val), unscale);
        out[PRE && pre.perm ? pre.perm[e] : e] = __dmul_rn(dd, dd);
    }
}

// Training-set RMSE in CSR order (N <= 65,536): one warp per row i at a time, U[i] kept
// in shared memory and the 32 ratings' V rows, J^K rows and C rows staged per 32-rating
// chunk (V, J^K, W and C are the small, L2-resident side; the CSC-order kernel above
// gathers a 1 KB U row per rating from HBM instead).  Staging is 16-byte cp.async into
// 32 x 32-element tiles whose 16-byte granules are XOR-swizzled by row, so lane r reads
// its own row with conflict-free 16-byte shared loads.  The row's columns go into a
// per-warp shared bitmap with per-word prefix counts: "did row i rate J[j, k]" is one bit
// probe and the value's CSR position is rlo + prefix + popc (no search); the rare rated
// neighbour reads its W entry directly.  Lane x owns rating x and runs its f and k loops in
// the reference's order, so the squared errors are the bytes of the CSC kernel's (stored
// at entry index csr_entry[p], NULL: identity).  (Measured alternatives, C3 fp64: one bulk
// copy per lane instead of the cp.async granules 28.8 ms vs 26.2 ms; double-buffered bulk
// stages 79 ms -- 32 KB per warp leaves one 4-warp CTA per SM.)
constexpr int kRowWarpsRmse = 4;
constexpr int kRowTile = 32 * 32;   // elements of one staged tile

template <typename T>
__device__ __forceinline__ int swz(int r, int f) {
    constexpr int GE = 16 / (int)sizeof(T);
    return r * 32 + (((f / GE) ^ (r & 7)) * GE) + f % GE;
}

template <typename P>
struct RowSmem {   // per-warp carve-up (bytes, 16-aligned): V/C tile, J^K tile, bitmap + prefix, U[i]
    static __host__ __device__ int bytes(int words, int F) {
        return kRowTile * (int)sizeof(P) + kRowTile * 4 + 8 * ((words + 1) & ~1) + ((F + 31) & ~31) * (int)sizeof(P);
    }
};

// Rows [0, cnt) of the chunk's ne ratings (lane r's row starts at myrow) -> swizzled tile.
// vec: 16-byte granules (the caller guarantees 16-byte aligned rows and that the last
// granule stays inside the array), else element copies.
template <typename T>
__device__ __forceinline__ void stage_rows(T *tile, const T *myrow, int ne, int cnt, bool vec, int lane) {
    constexpr int GE = 16 / (int)sizeof(T);
    constexpr int G = 32 / GE;     // granules per 32-element row
    constexpr int RPI = 32 / G;    // rows per instruction
    const uintptr_t mine = reinterpret_cast<uintptr_t>(myrow);
    if (vec) {
        const int g = lane % G, rs = lane / G;
        const int ng = (cnt + GE - 1) / GE;
        for (int r0 = 0; r0 < ne; r0 += RPI) {
            const int r = r0 + rs;
            const T *src = reinterpret_cast<const T *>(__shfl_sync(0xffffffffu, mine, r & 31));
            if (r < ne && g < ng) cp_async<16>(tile + r * 32 + ((g ^ (r & 7)) * GE), src + g * GE);
        }
    } else {
#pragma unroll 4
        for (int r = 0; r < ne; ++r) {
            const T *src = reinterpret_cast<const T *>(__shfl_sync(0xffffffffu, mine, r));
            if (lane < cnt) cp_async<sizeof(T)>(tile + swz<T>(r, lane), src + lane);
        }
    }
}

// The ratings to predict, grouped by row: row i's targets are [ptr[i], ptr[i+1]) with
// their columns, values and entry index (the position of their squared error; NULL:
// identity).  The training set is the ratings' own CSR.
struct RowTargets {
    const int64_t *ptr;
    const int32_t *cols;
    const double *vals;
    const int32_t *index;
};

template <typename P>
__global__ void __launch_bounds__(kRowWarpsRmse * 32, 3)
    pred_row_kernel(CulshData d, double mu, const P *__restrict__ b, const P *__restrict__ bhat,
                    const P *__restrict__ U, const P *__restrict__ V, const P *__restrict__ W,
                    const P *__restrict__ C, const int32_t *__restrict__ nbr, int F, int ldF, int K,
                    int words, int vec, RowTargets tg, int do_clamp, double lo, double hi, double unscale,
                    double *__restrict__ out) {
    using V2 = typename std::conditional<sizeof(P) == 8, double2, float4>::type;
    constexpr int GE = 16 / (int)sizeof(P);
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int wid = threadIdx.x >> 5;
    unsigned char *base = s_raw + (size_t)wid * RowSmem<P>::bytes(words, F);
    P *vt = reinterpret_cast<P *>(base);                                              // V tile, then C tile
    int32_t *jt = reinterpret_cast<int32_t *>(base + kRowTile * sizeof(P));           // J^K tile
    uint32_t *bm = reinterpret_cast<uint32_t *>(base + kRowTile * (sizeof(P) + 4));
    uint32_t *pre = bm + words;                                                       // set bits before w
    P *us = reinterpret_cast<P *>(base + kRowTile * (sizeof(P) + 4) + 8 * ((words + 1) & ~1));   // U[i]
    const int Fs = (F + 31) & ~31;
    const int lane = (int)lane_id();
    const bool vecV = vec & 1, vecJ = vec & 2, vecC = vec & 4;
    const int per = (words + 31) >> 5;
    const int w0 = min(words, lane * per), w1 = min(words, w0 + per);
    for (int w = lane; w < words; w += 32) bm[w] = 0u;
    __syncwarp();
    const int64_t nw = (int64_t)gridDim.x * kRowWarpsRmse;
    for (int64_t i = (int64_t)blockIdx.x * kRowWarpsRmse + wid; i < d.M; i += nw) {
        const int64_t tlo = tg.ptr[i], thi = tg.ptr[i + 1];
        if (tlo == thi) continue;
        const int64_t rlo = d.row_ptr[i], rhi = d.row_ptr[i + 1];
        if (K > 0) {
            for (int64_t p = rlo + lane; p < rhi; p += 32) {
                const int32_t c = d.row_cols[p];
                atomicOr(bm + (c >> 5), 1u << (c & 31));
            }
            __syncwarp();
            int cnt = 0;
            for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int run = incl - cnt;
            for (int w = w0; w < w1; ++w) {
                pre[w] = (uint32_t)run;
                run += __popc(bm[w]);
            }
        }
        const double mb = __dadd_rn(mu, (double)b[i]);
        const double mbb = __dadd_rn(mu, d.base_b[i]);
        for (int f = lane; f < Fs; f += 32) us[f] = f < F ? U[i * ldF + f] : P(0);
        __syncwarp();
        for (int64_t c0 = tlo; c0 < thi; c0 += 32) {
            const int ne = (int)min64(32, thi - c0);
            const bool valid = lane < ne;
            const int64_t p = c0 + lane;
            const int32_t j = valid ? tg.cols[p] : 0;
            double pred = valid ? __dadd_rn(mb, (double)bhat[j]) : 0.0;
            double dot = 0.0;
            for (int f0 = 0; f0 < F; f0 += 32) {
                const int fe = F - f0 < 32 ? F - f0 : 32;
                stage_rows<P>(vt, V + (int64_t)j * ldF + f0, ne, fe, vecV, lane);
                cp_async_wait_all();
                __syncwarp();
                if (valid) {
                    const P *uf = us + f0;
                    if (fe == 32) {   // full chunk: no bounds, loads hoisted
#pragma unroll 4
                        for (int g = 0; g < 32 / GE; ++g) {
                            const V2 v = *reinterpret_cast<const V2 *>(vt + lane * 32 + ((g ^ (lane & 7)) * GE));
                            const V2 u = *reinterpret_cast<const V2 *>(uf + g * GE);
                            const P *vv = reinterpret_cast<const P *>(&v);
                            const P *uu = reinterpret_cast<const P *>(&u);
#pragma unroll
                            for (int e = 0; e < GE; ++e) dot = __dadd_rn(dot, __dmul_rn((double)uu[e], (double)vv[e]));
                        }
                    } else {
                        for (int q = 0; q < fe; ++q)
                            dot = __dadd_rn(dot, __dmul_rn((double)uf[q], (double)vt[swz<P>(lane, q)]));
                    }
                }
                __syncwarp();
            }
            pred = __dadd_rn(pred, dot);
            int nr = 0, nn = 0;
            double sw = 0.0, sc = 0.0;
            for (int k0 = 0; k0 < K; k0 += 32) {
                const int kn = K - k0 < 32 ? K - k0 : 32;
                const int64_t jrow = (int64_t)j * K + k0;
                stage_rows<int32_t>(jt, nbr + jrow, ne, kn, vecJ, lane);
                stage_rows<P>(vt, C + jrow, ne, kn, vecC, lane);
                cp_async_wait_all();
                __syncwarp();
                if (valid) {
                    for (int g = 0; g * 4 < kn; ++g) {
                        const int4 j4 = *reinterpret_cast<const int4 *>(jt + lane * 32 + ((g ^ (lane & 7)) * 4));
                        const int32_t *jj = reinterpret_cast<const int32_t *>(&j4);
                        P cv[4];
                        *reinterpret_cast<V2 *>(cv) =
                            *reinterpret_cast<const V2 *>(vt + lane * 32 + (((4 * g / GE) ^ (lane & 7)) * GE));
                        if (GE == 2)
                            *reinterpret_cast<V2 *>(cv + 2) =
                                *reinterpret_cast<const V2 *>(vt + lane * 32 + (((4 * g / GE + 1) ^ (lane & 7)) * GE));
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int k = g * 4 + e;
                            if (k >= kn) break;
                            const int32_t j1 = jj[e];
                            const uint32_t word = bm[j1 >> 5];
                            if ((word >> (j1 & 31)) & 1u) {
                                const int64_t pos = rlo + pre[j1 >> 5] + __popc(word & ((1u << (j1 & 31)) - 1u));
                                ++nr;
                                sw = __dadd_rn(sw, __dmul_rn(__dsub_rn(d.row_vals[pos],
                                                                       __dadd_rn(mbb, d.base_bhat[j1])),
                                                             (double)__ldg(W + jrow + k)));
                            } else {
                                ++nn;
                                sc = __dadd_rn(sc, (double)cv[e]);
                            }
                        }
                    }
                }
                __syncwarp();
            }
            if (nr > 0) pred = __dadd_rn(pred, __ddiv_rn(sw, __dsqrt_rn((double)nr)));
            if (nn > 0) pred = __dadd_rn(pred, __ddiv_rn(sc, __dsqrt_rn((double)nn)));
            if (valid) {
                if (do_clamp) {
                    if (pred < lo) pred = lo;
                    else if (pred > hi) pred = hi;
                }
                const double dd = __dmul_rn(__dsub_rn(pred, tg.vals[p]), unscale);
                out[tg.index ? (int64_t)tg.index[p] : p] = __dmul_rn(dd, dd);
            }
        }
        if (K > 0) {
            __syncwarp();
            for (int64_t p = rlo + lane; p < rhi; p += 32) bm[d.row_cols[p] >> 5] = 0u;
            __syncwarp();
        }
    }
}

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename P>
int launch_pred_rows(const CulshData *d, double mu, const P *b, const P *bhat, const P *U, const P *V, const P *W,
                     const P *C, const int32_t *nbr, int F, int ldF, int K, RowTargets tg, int do_clamp,
                     double lo, double hi, double unscale, double *sq, cudaStream_t st) {
    CULSH_REQUIRE(d->N <= 65536, "the CSR-order rmse needs N <= 65536 (per-warp row bitmap)");
    CULSH_REQUIRE(K >= 0 && K <= 64, "K must be in [0, 64]");
    const int words = (int)((d->N + 31) / 32);
    // 16-byte granule copies: row starts and pitches must be 16-aligned
    // (then the last granule of a row stays inside the array)
    const int vec = ((aligned16(V) && (ldF * sizeof(P)) % 16 == 0) ? 1 : 0) |
                    ((aligned16(nbr) && (K * 4) % 16 == 0) ? 2 : 0) |
                    ((aligned16(C) && (K * sizeof(P)) % 16 == 0) ? 4 : 0);
    const size_t smem = (size_t)kRowWarpsRmse * RowSmem<P>::bytes(words, F);
    CULSH_CHECK(cudaFuncSetAttribute(pred_row_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CULSH_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pred_row_kernel<P>, kRowWarpsRmse * 32, smem));
    const int64_t blocks = min64((d->M + kRowWarpsRmse - 1) / kRowWarpsRmse, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    pred_row_kernel<P><<<(unsigned)blocks, kRowWarpsRmse * 32, smem, st>>>(
        *d, mu, b, bhat, U, V, W, C, nbr, F, ldF, K, words, vec, tg, do_clamp, lo, hi, unscale, sq);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// Lookup cache of the training set: per 32-entry group of CSC entries, the number of
// explicit (i, J[j, k]) pairs, then their CSC positions (warp scan per group).
__global__ void lookup_count_kernel(int64_t nnz, const uint32_t *__restrict__ mask, int MW,
                                    int64_t *__restrict__ group_count) {
    const int lane = (int)lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g * 32 < nnz; g += warps) {
        const int64_t e = g * 32 + lane;
        int pc = 0;
        if (e < nnz) {
            pc = __popc(mask[e * MW]);
            if (MW == 2) pc += __popc(mask[e * MW + 1]);
        }
        pc = warp_sum(pc);
        if (lane == 0) group_count[g] = pc;
    }
}

__global__ void lookup_fill_kernel(CulshData d, const int32_t *__restrict__ nbr, int K, const uint32_t *__restrict__ mask,
                                   int MW, const int64_t *__restrict__ group_base, int32_t *__restrict__ pos) {
    const int lane = (int)lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g * 32 < d.nnz; g += warps) {
        const int64_t e = g * 32 + lane;
        uint32_t m0 = 0u, m1 = 0u;
        if (e < d.nnz) {
            m0 = mask[e * MW];
            if (MW == 2) m1 = mask[e * MW + 1];
        }
        const int pc = __popc(m0) + __popc(m1);
        int incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (!pc) continue;
        int64_t cur = group_base[g] + incl - pc;
        const int64_t j = column_of(d.col_ptr, d.N, e);
        const int32_t i = d.col_rows[e];
        for (int q = 0; q < MW; ++q) {
            uint32_t m = q == 0 ? m0 : m1;
            while (m) {
                const int k = 32 * q + __ffs(m) - 1;
                m &= m - 1u;
                const int32_t j1 = nbr[j * K + k];
                int64_t lo2 = d.col_ptr[j1], hi2 = d.col_ptr[j1 + 1];
                while (lo2 < hi2) {   // the row is present (the mask says so)
                    const int64_t mid = (lo2 + hi2) >> 1;
                    if (__ldg(d.col_rows + mid) < i) lo2 = mid + 1; else hi2 = mid;
                }
                pos[cur++] = (int32_t)lo2;
            }
        }
    }
}

// ---- the reference's sequential sum of non-negative terms, in parallel -----------------
// S_{k+1} = fl(S_k + x_k), x_k >= 0 (squared errors).  While S stays inside one binade
// [2^e, 2^(e+1)) every S is a multiple of u = ulp(S) = 2^(e-52) (2^-1074 for the subnormal
// range and the first normal binade, which share that grid), and fl(S + x) is S + d*u with
// d = round(x / u) to nearest -- x / u is exact (power-of-two scaling) -- except that an
// exact tie (x / u = k + 1/2) rounds to the even sum, which depends on the parity of S / u.
// So a run of additions inside one binade is an integer sum plus a 1-bit parity state, and
// its effect is the function b -> (D_b, b'_b) of the starting parity b -- associative under
// composition.  The sum then runs as: (1) approximate chunk sums, (2) their exclusive
// prefix (the approximate S at each chunk start, hence its binade), (3) every chunk's
// function on that binade's grid, in parallel, (4) one CTA walks the chunks with the exact S:
// a chunk whose grid matches S's and whose integer sum stays below 2^53 (no binade change
// inside) is applied in O(1); any other chunk (S == 0, a binade change, a huge, negative or
// non-finite term) is added term by term, exactly like the sequential loop.  The result is
// the sequential loop's bits (tests/test_gpu_device_api.py::test_exact_sequential_sum).
constexpr int kSeqChunk = 8192;
constexpr int kSeqItems = kSeqChunk / 1024;

struct SeqFn {
    uint64_t d0, d1;   // integer increments (units of u) for starting parity 0 / 1
    int o0, o1;        // resulting parity
    int uexp;          // log2(u) of the grid the function was built on
    int ok;            // no huge / negative / non-finite term, grid known
};

__device__ __forceinline__ int grid_exp(double S) {   // log2(ulp) of S > 0
    int E;
    frexp(S, &E);                                       // S = m * 2^E, m in [0.5, 1)
    return max(E - 53, -1074);
}

__device__ __forceinline__ SeqFn seq_compose(const SeqFn &a, const SeqFn &b) {
    SeqFn r;
    const uint64_t cap = 1ull << 62;   // saturate: a chunk that large is rejected anyway
    r.d0 = min(cap, a.d0 + (a.o0 ? b.d1 : b.d0));
    r.o0 = a.o0 ? b.o1 : b.o0;
    r.d1 = min(cap, a.d1 + (a.o1 ? b.d1 : b.d0));
    r.o1 = a.o1 ? b.o1 : b.o0;
    r.uexp = a.uexp;
    r.ok = a.ok & b.ok;
    return r;
}

__global__ void __launch_bounds__(1024) seq_chunk_sum_kernel(const double *__restrict__ x, int64_t n,
                                                             double *__restrict__ csum) {
    __shared__ double red[32];
    const int64_t lo = (int64_t)blockIdx.x * kSeqChunk, hi = min64(n, lo + kSeqChunk);
    double s = 0.0;
    for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) s += x[k];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = red[threadIdx.x];
        v = warp_sum(v);
        if (threadIdx.x == 0) csum[blockIdx.x] = v;
    }
}

// exclusive prefix of the chunk sums (approximate chunk-start values; any order is fine)
__global__ void __launch_bounds__(1024) seq_chunk_prefix_kernel(const double *__restrict__ csum, int64_t nch,
                                                                double *__restrict__ cpre) {
    __shared__ double part[1024];
    const int64_t per = (nch + 1023) / 1024;
    const int64_t lo = threadIdx.x * per, hi = min64(nch, lo + per);
    double s = 0.0;
    for (int64_t c = lo; c < hi; ++c) s += csum[c];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        for (int t = 0; t < 1024; ++t) { const double v = part[t]; part[t] = run; run += v; }
    }
    __syncthreads();
    double run = part[threadIdx.x];
    for (int64_t c = lo; c < hi; ++c) { cpre[c] = run; run += csum[c]; }
}

__global__ void __launch_bounds__(1024) seq_chunk_fn_kernel(const double *__restrict__ x, int64_t n,
                                                            const double *__restrict__ cpre, SeqFn *__restrict__ fn) {
    __shared__ SeqFn wred[32];
    const int64_t lo = (int64_t)blockIdx.x * kSeqChunk;
    const double A = cpre[blockIdx.x];
    const bool known = A > 0.0 && isfinite(A);
    const int ue = known ? grid_exp(A) : 0;
    SeqFn f{0, 0, 0, 1, ue, known ? 1 : 0};
    const int64_t k0 = lo + (int64_t)threadIdx.x * kSeqItems;
#pragma unroll
    for (int q = 0; q < kSeqItems; ++q) {
        const int64_t k = k0 + q;
        if (k >= n) break;
        const double xv = x[k];
        const double y = ldexp(xv, -ue);                // exact scaling
        SeqFn e{0, 0, 0, 1, ue, 1};
        if (!(y >= 0.0 && y < 9007199254740992.0)) {   // negative, >= 2^53 units, NaN / inf
            e.ok = 0;
        } else {
            const double fl = floor(y), fr = y - fl;
            const uint64_t di = (uint64_t)fl;
            if (fr == 0.5) {   // tie: the even result
                e.d0 = di + (di & 1u);            // start parity 0: sum parity = di's
                e.d1 = di + ((di & 1u) ^ 1u);
                e.o0 = 0;
                e.o1 = 0;
            } else {
                const uint64_t d = di + (fr > 0.5 ? 1u : 0u);
                e.d0 = d;
                e.d1 = d;
                e.o0 = (int)(d & 1u);
                e.o1 = (int)((d & 1u) ^ 1u);
            }
        }
        f = seq_compose(f, e);
    }
    // ordered reduction: lane order within the warp, then warp order
    const unsigned lane = lane_id();
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        SeqFn g;
        g.d0 = __shfl_down_sync(0xffffffffu, f.d0, off);
        g.d1 = __shfl_down_sync(0xffffffffu, f.d1, off);
        g.o0 = __shfl_down_sync(0xffffffffu, f.o0, off);
        g.o1 = __shfl_down_sync(0xffffffffu, f.o1, off);
        g.ok = __shfl_down_sync(0xffffffffu, f.ok, off);
        g.uexp = ue;
        if ((lane & (2 * off - 1)) == 0) f = seq_compose(f, g);
    }
    if (lane == 0) wred[threadIdx.x >> 5] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
        SeqFn r = wred[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = seq_compose(r, wred[w]);
        r.ok &= known ? 1 : 0;
        fn[blockIdx.x] = r;
    }
}

// one CTA walks the chunks with the exact running sum (dynamic shared: kSeqChunk doubles).
// The chunk functions are staged 1024 at a time; from the current chunk on, the CTA scans
// them (composition in chunk order) and finds the first chunk that is not on S's grid or
// whose sum leaves S's binade; every chunk before it is applied at once (the scanned prefix),
// that one is added term by term, and the scan restarts after it.
__device__ __forceinline__ SeqFn shfl_up_fn(const SeqFn &f, int off) {
    SeqFn g;
    g.d0 = __shfl_up_sync(0xffffffffu, f.d0, off);
    g.d1 = __shfl_up_sync(0xffffffffu, f.d1, off);
    g.o0 = __shfl_up_sync(0xffffffffu, f.o0, off);
    g.o1 = __shfl_up_sync(0xffffffffu, f.o1, off);
    g.ok = __shfl_up_sync(0xffffffffu, f.ok, off);
    g.uexp = f.uexp;
    return g;
}

// inclusive scan over the CTA's 1024 threads (thread order = chunk order)
__device__ SeqFn block_scan_fn(SeqFn f, SeqFn *s_warp) {
    const unsigned lane = lane_id();
    const int w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const SeqFn g = shfl_up_fn(f, off);
        if ((int)lane >= off) f = seq_compose(g, f);
    }
    if (lane == 31) s_warp[w] = f;
    __syncthreads();
    if (w == 0) {
        SeqFn t = s_warp[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const SeqFn g = shfl_up_fn(t, off);
            if ((int)lane >= off) t = seq_compose(g, t);
        }
        s_warp[lane] = t;
    }
    __syncthreads();
    if (w > 0) f = seq_compose(s_warp[w - 1], f);
    __syncthreads();   // s_warp is reused by the next scan
    return f;
}

__global__ void __launch_bounds__(1024) seq_walk_kernel(const double *__restrict__ x, int64_t n, int64_t nch,
                                                        const SeqFn *__restrict__ fn, int as_rmse,
                                                        double *__restrict__ out) {
    extern __shared__ double sbuf[];
    __shared__ SeqFn s_fn[1024];
    __shared__ SeqFn s_warp[32];
    __shared__ double s_S;
    __shared__ int s_k;
    const SeqFn ident{0, 0, 0, 1, 0, 1};
    if (threadIdx.x == 0) s_S = 0.0;
    for (int64_t base = 0; base < nch; base += 1024) {
        const int cnt = (int)min64(1024, nch - base);
        __syncthreads();
        if ((int)threadIdx.x < cnt) s_fn[threadIdx.x] = fn[base + threadIdx.x];
        if (threadIdx.x == 0) s_k = 1 << 30;
        __syncthreads();
        int idx = 0;
        while (idx < cnt) {
            const double S = s_S;
            int k;   // chunks [idx, idx + k) are applied at once; chunk idx + k term by term
            if (isnan(S)) {
                k = cnt - idx;   // NaN stays NaN
            } else if (!(S > 0.0) || isinf(S)) {
                k = 0;           // S == 0 (or inf): term by term
            } else {
                const int ue = grid_exp(S);
                const uint64_t Si0 = (uint64_t)ldexp(S, -ue);   // exact: S is on its grid
                const int c = idx + (int)threadIdx.x;
                const SeqFn f = c < cnt ? s_fn[c] : ident;
                const bool valid = c >= cnt || (f.ok && f.uexp == ue);
                const SeqFn P = block_scan_fn(f, s_warp);
                const uint64_t D = (Si0 & 1u) ? P.d1 : P.d0;   // through chunk c, from S
                const bool bad = c < cnt && (!valid || !P.ok || Si0 + D >= (1ull << 53));
                if (bad) atomicMin(&s_k, (int)threadIdx.x);
                __syncthreads();
                k = min(s_k, cnt - idx);
                if ((int)threadIdx.x == k - 1) s_S = ldexp((double)(Si0 + D), ue);   // exact
                __syncthreads();
                if (threadIdx.x == 0) s_k = 1 << 30;
            }
            idx += k;
            __syncthreads();
            if (idx < cnt) {   // term by term, staged so the adds run at add latency
                const int64_t lo = (base + idx) * kSeqChunk;
                const int m = (int)min64(kSeqChunk, n - lo);
                for (int q = threadIdx.x; q < m; q += blockDim.x) sbuf[q] = x[lo + q];
                __syncthreads();
                if (threadIdx.x == 0) {
                    double T = s_S;
                    for (int q = 0; q < m; ++q) T = __dadd_rn(T, sbuf[q]);
                    s_S = T;
                }
                ++idx;
                __syncthreads();
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = as_rmse ? sqrt(s_S / (double)n) : s_S;
}

// the one-thread loop's result as a plain sum (small n)
__global__ void seq_to_sum_kernel(const double *__restrict__ x, int64_t n, double *__restrict__ out) {
    double S = 0.0;
    for (int64_t k = 0; k < n; ++k) S = __dadd_rn(S, x[k]);
    *out = S;
}

// exact sequential sum for any n (the parallel form above; the one-thread loop for small n)
int seq_sum_exact(const double *sq, int64_t n, double *out, cudaStream_t st, bool as_rmse = true) {
    if (n <= 4 * kSeqChunk) {
        if (as_rmse) seq_sum_kernel<<<1, 1024, 0, st>>>(sq, n, out);
        else seq_to_sum_kernel<<<1, 1, 0, st>>>(sq, n, out);
        return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
    }
    const int64_t nch = (n + kSeqChunk - 1) / kSeqChunk;
    void *scratch = nullptr;
    const size_t bytes = (size_t)nch * (2 * sizeof(double) + sizeof(SeqFn));
    CULSH_CHECK(cudaMallocAsync(&scratch, bytes, st));
    double *csum = static_cast<double *>(scratch), *cpre = csum + nch;
    SeqFn *fn = reinterpret_cast<SeqFn *>(cpre + nch);
    seq_chunk_sum_kernel<<<(unsigned)nch, 1024, 0, st>>>(sq, n, csum);
    seq_chunk_prefix_kernel<<<1, 1024, 0, st>>>(csum, nch, cpre);
    seq_chunk_fn_kernel<<<(unsigned)nch, 1024, 0, st>>>(sq, n, cpre, fn);
    // (set on every call: the attribute is per device)
    CULSH_CHECK(cudaFuncSetAttribute(seq_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(kSeqChunk * sizeof(double))));
    seq_walk_kernel<<<1, 1024, kSeqChunk * sizeof(double), st>>>(sq, n, nch, fn, as_rmse ? 1 : 0, out);
    const cudaError_t e = cudaGetLastError();
    CULSH_CHECK(cudaFreeAsync(scratch, st));
    return e == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

int reduce_rmse(const double *sq, int64_t n, double *out, double *scratch_partials, bool sequential,
                cudaStream_t st) {
    if (sequential) {
        return seq_sum_exact(sq, n, out, st);
    } else {
        const int np = 256;
        tree_sum_kernel<<<np, 1024, 0, st>>>(sq, n, scratch_partials);
        finish_kernel<<<1, 1, 0, st>>>(scratch_partials, np, n, out);
    }
    return cudaGetLastError() == cudaSuccess ? CULSH_OK : CULSH_ECUDA;
}

}  // namespace culsh

using namespace culsh;

// fl(...fl(fl(0 + x[0]) + x[1]) ... + x[n-1]) -- numpy's np.add.accumulate(x)[-1] -- for
// non-negative x (any other term is added one by one), n >= 1
extern "C" int culsh_sequential_sum(const double *x, int64_t n, double *out, void *stream) {
    CULSH_REQUIRE(n >= 1, "empty input");
    return seq_sum_exact(x, n, out, (cudaStream_t)stream, false);
}

// sqerr_scratch must hold n + 256 doubles.  The sum is the reference's sequential one, bit
// for bit, at any n (seq_sum_exact).
extern "C" int culsh_rmse(const CulshData *d, const CulshModel64 *m, const int32_t *t_rows,
                          const int32_t *t_cols, const double *t_vals, int64_t n, int do_clamp,
                          double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                          double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 63) / 64, (int64_t)num_sms() * 24);
    pred_tile_kernel<double, false><<<blocks, 64, 0, st>>>(*d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                            m->nbr, m->F, m->F, m->K, t_rows, t_cols, t_vals, n,
                                                            PreLookup{}, 0, do_clamp, clamp_lo, clamp_hi, unscale,
                                                            sqerr_scratch);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, true, st);
}

extern "C" int culsh_train_lookup(const CulshData *d, const int32_t *nbr, int K, const uint32_t *mask,
                                  int64_t *group_count, const int64_t *group_base, int32_t *pos, void *stream) {
    CULSH_REQUIRE(K >= 1 && K <= 64, "K must be in [1, 64]");
    if (d->nnz <= 0) return CULSH_OK;
    const int MW = K <= 32 ? 1 : 2;
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = num_sms() * 16;
    if (group_count)
        lookup_count_kernel<<<blocks, 256, 0, st>>>(d->nnz, mask, MW, group_count);
    else
        lookup_fill_kernel<<<blocks, 256, 0, st>>>(*d, nbr, K, mask, MW, group_base, pos);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_rmse_train(const CulshData *d, const CulshModel64 *m, const uint32_t *mask,
                                const int64_t *group_base, const int32_t *pos, const int64_t *perm, int do_clamp,
                                double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                                double *rmse_out, void *stream) {
    const int64_t n = d->nnz;
    CULSH_REQUIRE(n > 0, "empty training set");
    CULSH_REQUIRE(m->K == 0 || (mask && group_base && pos), "lookup cache missing");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 127) / 128, (int64_t)num_sms() * 12);
    PreLookup pre{mask, group_base, pos, perm, m->K <= 32 ? 1 : 2};
    pred_tile_kernel<double, true><<<blocks, 128, 0, st>>>(*d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                           m->nbr, m->F, m->F, m->K, nullptr, nullptr, nullptr, n, pre, 0,
                                                           do_clamp, clamp_lo, clamp_hi, unscale, sqerr_scratch);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, true, st);
}

extern "C" int culsh_rmse32(const CulshData *d, const CulshModel32 *m, const int32_t *nbr,
                            const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                            double *sqerr_scratch, double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 63) / 64, (int64_t)num_sms() * 24);
    pred_tile_kernel<float, false><<<blocks, 64, 0, st>>>(*d, (double)m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                           nbr, m->F, m->F, m->K, t_rows, t_cols, t_vals, n, PreLookup{},
                                                           0, 0, 0.0, 0.0, 1.0, sqerr_scratch);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, true, st);
}

extern "C" int culsh_predict(const CulshData *d, const CulshModel64 *m, const int32_t *rows,
                             const int32_t *cols, int64_t n, double *out, void *stream) {
    if (n <= 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 63) / 64, (int64_t)num_sms() * 24);
    pred_tile_kernel<double, false><<<blocks, 64, 0, st>>>(*d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                            m->nbr, m->F, m->F, m->K, rows, cols, nullptr, n, PreLookup{},
                                                            1, 0, 0.0, 0.0, 1.0, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// rmse / rmse_train on an fp32 model (a Hogwild fit) without widening it: the kernel loads
// the fp32 values and computes in fp64 exactly as on the widened copy (every fp32 value is
// an fp64 value), so the result is the same bytes; F = logical factors, the model's row
// stride is m->F (zero-padded widths).  nbr: the model's J^K.
extern "C" int culsh_rmse_m32(const CulshData *d, const CulshModel32 *m, double mu, int F, const int32_t *nbr,
                              const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                              int do_clamp, double clamp_lo, double clamp_hi, double unscale,
                              double *sqerr_scratch, double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    CULSH_REQUIRE(F >= 1 && F <= m->F, "logical F exceeds the model's row stride");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 63) / 64, (int64_t)num_sms() * 24);
    pred_tile_kernel<float, false><<<blocks, 64, 0, st>>>(*d, mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                           nbr, F, m->F, m->K, t_rows, t_cols, t_vals, n,
                                                           PreLookup{}, 0, do_clamp, clamp_lo, clamp_hi, unscale,
                                                           sqerr_scratch);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, true, st);
}

extern "C" int culsh_rmse_train_m32(const CulshData *d, const CulshModel32 *m, double mu, int F,
                                    const int32_t *nbr,
                                    const uint32_t *mask, const int64_t *group_base, const int32_t *pos,
                                    const int64_t *perm, int do_clamp, double clamp_lo, double clamp_hi,
                                    double unscale, double *sqerr_scratch, double *rmse_out, void *stream) {
    const int64_t n = d->nnz;
    CULSH_REQUIRE(n > 0, "empty training set");
    CULSH_REQUIRE(F >= 1 && F <= m->F, "logical F exceeds the model's row stride");
    CULSH_REQUIRE(m->K == 0 || (mask && group_base && pos), "lookup cache missing");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (int)min64((n + 127) / 128, (int64_t)num_sms() * 12);
    PreLookup pre{mask, group_base, pos, perm, m->K <= 32 ? 1 : 2};
    pred_tile_kernel<float, true><<<blocks, 128, 0, st>>>(*d, mu, m->b, m->bhat, m->U, m->V, m->W, m->C,
                                                          nbr, F, m->F, m->K, nullptr, nullptr, nullptr, n, pre, 0,
                                                          do_clamp, clamp_lo, clamp_hi, unscale, sqerr_scratch);
    CULSH_LAUNCH_CHECK();
    return reduce_rmse(sqerr_scratch, n, rmse_out, sqerr_scratch + n, true, st);
}

// factorization.py:559-579 rmse in row order (pred_row_kernel; N <= 65,536, no lookup
// cache).  Targets: the training set itself (culsh_rmse_train_rows: the ratings' CSR,
// csr_entry = entry index of each CSR position, NULL: identity) or any test set grouped by
// row (culsh_rmse_rows: t_ptr (M+1), t_cols, t_vals, t_index = each target's position in
// the test set).  The sum runs in entry order like culsh_rmse / culsh_rmse_train.
static int rows_finish(int rc, const double *sq, int64_t n, double *out, double *scratch, cudaStream_t st) {
    if (rc != CULSH_OK) return rc;
    return reduce_rmse(sq, n, out, scratch, true, st);
}

extern "C" int culsh_rmse_train_rows(const CulshData *d, const CulshModel64 *m, const int32_t *csr_entry,
                                     int do_clamp, double clamp_lo, double clamp_hi, double unscale,
                                     double *sqerr_scratch, double *rmse_out, void *stream) {
    const int64_t n = d->nnz;
    CULSH_REQUIRE(n > 0, "empty training set");
    cudaStream_t st = (cudaStream_t)stream;
    const RowTargets tg{d->row_ptr, d->row_cols, d->row_vals, csr_entry};
    return rows_finish(launch_pred_rows<double>(d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C, m->nbr, m->F,
                                                m->F, m->K, tg, do_clamp, clamp_lo, clamp_hi, unscale,
                                                sqerr_scratch, st),
                       sqerr_scratch, n, rmse_out, sqerr_scratch + n, st);
}

extern "C" int culsh_rmse_train_rows_m32(const CulshData *d, const CulshModel32 *m, double mu, int F,
                                         const int32_t *nbr, const int32_t *csr_entry, int do_clamp,
                                         double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                                         double *rmse_out, void *stream) {
    const int64_t n = d->nnz;
    CULSH_REQUIRE(n > 0, "empty training set");
    CULSH_REQUIRE(F >= 1 && F <= m->F, "logical F exceeds the model's row stride");
    cudaStream_t st = (cudaStream_t)stream;
    const RowTargets tg{d->row_ptr, d->row_cols, d->row_vals, csr_entry};
    return rows_finish(launch_pred_rows<float>(d, mu, m->b, m->bhat, m->U, m->V, m->W, m->C, nbr, F, m->F, m->K,
                                               tg, do_clamp, clamp_lo, clamp_hi, unscale, sqerr_scratch, st),
                       sqerr_scratch, n, rmse_out, sqerr_scratch + n, st);
}

extern "C" int culsh_rmse_rows(const CulshData *d, const CulshModel64 *m, const int64_t *t_ptr,
                               const int32_t *t_cols, const double *t_vals, const int32_t *t_index, int64_t n,
                               int do_clamp, double clamp_lo, double clamp_hi, double unscale,
                               double *sqerr_scratch, double *rmse_out, void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    cudaStream_t st = (cudaStream_t)stream;
    const RowTargets tg{t_ptr, t_cols, t_vals, t_index};
    return rows_finish(launch_pred_rows<double>(d, m->mu, m->b, m->bhat, m->U, m->V, m->W, m->C, m->nbr, m->F,
                                                m->F, m->K, tg, do_clamp, clamp_lo, clamp_hi, unscale,
                                                sqerr_scratch, st),
                       sqerr_scratch, n, rmse_out, sqerr_scratch + n, st);
}

extern "C" int culsh_rmse_rows_m32(const CulshData *d, const CulshModel32 *m, double mu, int F, const int32_t *nbr,
                                   const int64_t *t_ptr, const int32_t *t_cols, const double *t_vals,
                                   const int32_t *t_index, int64_t n, int do_clamp, double clamp_lo,
                                   double clamp_hi, double unscale, double *sqerr_scratch, double *rmse_out,
                                   void *stream) {
    CULSH_REQUIRE(n > 0, "empty test set");
    CULSH_REQUIRE(F >= 1 && F <= m->F, "logical F exceeds the model's row stride");
    cudaStream_t st = (cudaStream_t)stream;
    const RowTargets tg{t_ptr, t_cols, t_vals, t_index};
    return rows_finish(launch_pred_rows<float>(d, mu, m->b, m->bhat, m->U, m->V, m->W, m->C, nbr, F, m->F, m->K,
                                               tg, do_clamp, clamp_lo, clamp_hi, unscale, sqerr_scratch, st),
                       sqerr_scratch, n, rmse_out, sqerr_scratch + n, st);
}
