// simLSH signature build: row-hash table, ordered
// +/-psi accumulation per (column, group, map, bit), threshold and group-key
// pack, all fused in one column-resident kernel.
//
// Reference semantics (bit-exact):
//   bits[i,g,m,t] = (splitmix64(map_key(seed,g,m) ^ i) >> t) & 1     lsh.py:68-78
//   acc[j,g,m,t]  = sum over column j in ascending row of +/-psi(v)   lsh.py:161-179
//   sig = acc >= 0                                                      lsh.py:182-183
//   key[g,j] bit (m*G+t) = sig[j,g,m,t]                                 lsh.py:246-260
//
// HBM layout: the row-hash table stores, per row, q*p*ns bytes (ns = ceil(G/8)
// byte "slices" per map), i.e. the reference's (M,q,p,G) u8 bit tensor packed 8x.
// One CTA owns one column; thread s owns slice s of the column's q*p*ns slices
// and keeps its <= 8 accumulators in registers for the whole column.  Column
// entries (row, psi) are staged through shared memory in chunks.
#include "common.cuh"

namespace culsh {

// Row record of the packed table: q*p*ceil(G/8) bytes padded to 16 (bulk-copy unit).
__host__ __device__ __forceinline__ int64_t table_stride(int qp, int ns) {
    return ((int64_t)qp * ns + 15) & ~15LL;
}

__global__ void map_keys_kernel(uint64_t seed, int q, int p, uint64_t *keys) {
    int gm = blockIdx.x * blockDim.x + threadIdx.x;
    if (gm < q * p) keys[gm] = map_key(seed, gm / p, gm % p);
}

// table[i][g][m][s] = byte s of the low G bits of splitmix64(key(g,m) ^ i)
__global__ void row_hash_kernel(const uint64_t *__restrict__ keys, int qp, int G, int ns,
                                int64_t row_lo, int64_t row_hi, uint8_t *__restrict__ table) {
    const int64_t rec = table_stride(qp, ns);
    const int64_t total = (row_hi - row_lo) * (int64_t)qp;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = row_lo + x / qp;
        const int gm = (int)(x % qp);
        uint64_t h = splitmix64(keys[gm] ^ (uint64_t)i);
        if (G < 64) h &= (1ULL << G) - 1ULL;
        uint8_t *dst = table + i * rec + (int64_t)gm * ns;
        for (int s = 0; s < ns; ++s) dst[s] = (uint8_t)(h >> (8 * s));
    }
}

// (M,q,p,G) u8 bits -> packed table (for injected RowHashes, lsh.py:231-239 `hashes`)
__global__ void pack_bits_kernel(const uint8_t *__restrict__ bits, int64_t M, int qp, int G, int ns,
                                 uint8_t *__restrict__ table) {
    const int64_t total = M * (int64_t)qp * ns;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t igm = x / ns;
        const int s = (int)(x % ns);
        const uint8_t *src = bits + igm * G + 8 * s;
        const int nb = min(8, G - 8 * s);
        uint8_t v = 0;
        for (int t = 0; t < nb; ++t) v |= (uint8_t)((src[t] != 0) << t);
        const int64_t i = igm / qp;
        table[i * table_stride(qp, ns) + (igm % qp) * ns + s] = v;
    }
}

__global__ void unpack_bits_kernel(const uint8_t *__restrict__ table, int64_t M, int qp, int G, int ns,
                                   uint8_t *__restrict__ bits) {
    const int64_t total = M * (int64_t)qp * G;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t igm = x / G;
        const int t = (int)(x % G);
        const int64_t i = igm / qp;
        bits[x] = (table[i * table_stride(qp, ns) + (igm % qp) * ns + t / 8] >> (t % 8)) & 1;
    }
}

constexpr int kChunk = 512;

// AccT = double: the reference's ordered fp64 sum (bit-exact for any values).
// AccT = int:    exact integer sum, used only when every psi is an integer and the
//                per-column sum of |psi| is < 2^31 (then every fp64 partial sum of
//                the reference is an exact integer, so the results are identical).
template <typename AccT>
__global__ void __launch_bounds__(1024)
hash_accumulate_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                       const double *__restrict__ col_vals, int64_t col_begin, int64_t n_cols,
                       const int32_t *__restrict__ col_list, const uint8_t *__restrict__ table,
                       int qp, int p, int G, int ns, int e, int into,
                       double *__restrict__ acc, uint8_t *__restrict__ sig,
                       uint64_t *__restrict__ keys, int64_t keys_ld) {
    __shared__ int32_t s_rows[kChunk];
    __shared__ double s_psi[kChunk];
    extern __shared__ uint8_t s_sigbyte[];  // qp * ns bytes

    const int64_t j = col_list ? (int64_t)col_list[blockIdx.x] : col_begin + blockIdx.x;
    const int W8 = qp * ns;
    const int64_t rec = table_stride(qp, ns);
    const int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
    const int64_t accW = (int64_t)qp * G;

    for (int base = 0; base < W8; base += blockDim.x) {
        const int s = base + threadIdx.x;
        const bool active = s < W8;
        const int gm = active ? s / ns : 0;
        const int sl = active ? s % ns : 0;
        const int nbits = active ? min(8, G - 8 * sl) : 0;
        double *a_out = acc + j * accW + (int64_t)gm * G + 8 * sl;
        AccT a[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = AccT(0);
        if constexpr (sizeof(AccT) == sizeof(double)) {
            if (into && active) {
#pragma unroll
                for (int t = 0; t < 8; ++t) a[t] = t < nbits ? a_out[t] : 0.0;
            }
        }
        for (int64_t c0 = lo; c0 < hi; c0 += kChunk) {
            const int n = (int)min64(kChunk, hi - c0);
            __syncthreads();
            for (int x = threadIdx.x; x < n; x += blockDim.x) {
                s_rows[x] = col_rows[c0 + x];
                s_psi[x] = psi_of(col_vals[c0 + x], e);
            }
            __syncthreads();
            if (active) {
                for (int x = 0; x < n; ++x) {
                    const uint32_t byte = table[(int64_t)s_rows[x] * rec + s];
                    if constexpr (sizeof(AccT) == sizeof(double)) {
                        const double ps = s_psi[x];
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            a[t] = __dadd_rn(a[t], ((byte >> t) & 1u) ? ps : -ps);
                    } else {
                        const int ps = (int)s_psi[x];
#pragma unroll
                        for (int t = 0; t < 8; ++t) a[t] += ((byte >> t) & 1u) ? ps : -ps;
                    }
                }
            }
        }
        if (active) {
            uint32_t sb = 0;
            double out[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                out[t] = (double)a[t];
                if (t < nbits) sb |= (out[t] >= 0.0 ? 1u : 0u) << t;
            }
            if (nbits == 8 && ((reinterpret_cast<uintptr_t>(a_out) & 15) == 0)) {
                double2 *o2 = reinterpret_cast<double2 *>(a_out);
                o2[0] = make_double2(out[0], out[1]);
                o2[1] = make_double2(out[2], out[3]);
                o2[2] = make_double2(out[4], out[5]);
                o2[3] = make_double2(out[6], out[7]);
            } else {
                for (int t = 0; t < nbits; ++t) a_out[t] = out[t];
            }
            if (sig) {
                uint8_t *sg = sig + j * accW + (int64_t)gm * G + 8 * sl;
                for (int t = 0; t < nbits; ++t) sg[t] = (sb >> t) & 1u;
            }
            s_sigbyte[s] = (uint8_t)sb;
        }
    }
    if (keys) {
        __syncthreads();
        const int q = qp / p;
        for (int g = threadIdx.x; g < q; g += blockDim.x) {
            uint64_t k = 0;
            for (int m = 0; m < p; ++m)
                for (int sl = 0; sl < ns; ++sl)
                    k |= (uint64_t)s_sigbyte[(g * p + m) * ns + sl] << (m * G + 8 * sl);
            keys[(int64_t)g * keys_ld + j] = k;
        }
    }
}

// Per-column sum of |psi| and integrality check for the exact-integer fast path.
__global__ void psi_int_check_kernel(const int64_t *__restrict__ col_ptr,
                                     const double *__restrict__ col_vals, int64_t col_begin,
                                     int64_t n_cols, const int32_t *__restrict__ col_list, int e,
                                     int *__restrict__ bad) {
    const int64_t c = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    if (c >= n_cols) return;
    const int64_t j = col_list ? (int64_t)col_list[c] : col_begin + c;
    double s = 0.0;
    int nonint = 0;
    for (int64_t x = col_ptr[j] + lane_id(); x < col_ptr[j + 1]; x += 32) {
        const double ps = psi_of(col_vals[x], e);
        if (!(ps == floor(ps)) || fabs(ps) > 1048576.0) nonint = 1;
        s += fabs(ps);
    }
    s = warp_sum(s);
    nonint = __any_sync(0xffffffffu, nonint);
    if (lane_id() == 0 && (nonint || s >= 2147483647.0)) atomicOr(bad, 1);
}

// ---------------------------------------------------------------------------
// Exact-integer fast path by bit counting (Harley-Seal carry-save adders).
//
// When the ratings take a few distinct values v (e.g. 1..5 stars) every psi is
// an integer, and acc[j,g,m,t] = sum_v psi(v) * (2 * n_v[t] - N_v) where n_v[t]
// counts the column's class-v ratings whose row hash has bit t set and N_v is the
// class size -- exact integer arithmetic, so the fp64 result equals the
// reference's ordered sum bit for bit.  Counting is done bit-sliced: a thread
// owns 32 hash bits (4 consecutive byte slices of the row record), loads one
// 32-bit word per rating and feeds 16 words at a time through a Harley-Seal CSA
// tree (15 x 2 LOP3 ops) into a bit-sliced vertical counter -- ~3 ops per 32 bits
// per rating instead of ~3 ops per bit.  Ratings are pre-partitioned by value
// class per column (class_partition_kernel) so each class streams contiguously.

constexpr int kHsDepth = 14;         // vertical counter bits: 16*(2^14-1) ratings per flush
constexpr int kHsMaxClasses = 16;
constexpr int kHsChunk = 1024;   // multiple of 16

// Per column: entries grouped by value class (order inside a class is irrelevant to
// integer counts).  One warp per column, two passes over the column; per-class counts
// and running offsets live in lanes 0..NC-1 (ballots + shuffles, no shared atomics).
__global__ void class_partition_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                                       const double *__restrict__ col_vals, int64_t N,
                                       const double *__restrict__ class_vals, int NC,
                                       int32_t *__restrict__ rows_by_class, int32_t *__restrict__ class_off) {
    __shared__ double s_cv[kHsMaxClasses];
    if (threadIdx.x < NC) s_cv[threadIdx.x] = class_vals[threadIdx.x];
    __syncthreads();
    const int w = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int64_t j = blockIdx.x * 8LL + w;
    if (j >= N) return;
    const int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
    const unsigned lt = (1u << lane) - 1u;
    // class of a value: its first match among class_vals[0..NC-2], else NC-1 (a uniform
    // NC-1-step loop over a shared copy: no divergent search, no global loads)
    auto cls = [&](double v) {
        int c = NC - 1;
        for (int k = NC - 2; k >= 0; --k) c = s_cv[k] == v ? k : c;
        return c;
    };
    int cnt = 0;   // lane c: entries of class c
    constexpr int U = 4;   // 4 x 32 entries per step: their loads are in flight together
    for (int64_t b0 = lo; b0 < hi; b0 += 32 * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t x = b0 + 32 * u + lane;
            v[u] = x < hi ? col_vals[x] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = b0 + 32 * u + lane < hi ? cls(v[u]) : -1;
            for (int cc = 0; cc < NC; ++cc) {
                const unsigned bal = __ballot_sync(0xffffffffu, c == cc);
                if ((int)lane == cc) cnt += __popc(bal);
            }
        }
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
    }
    int run = incl - cnt;   // lane c: next slot of class c (rows stay ascending within a class)
    if ((int)lane < NC) class_off[j * (NC + 1) + lane] = run;
    if ((int)lane == NC - 1) class_off[j * (NC + 1) + NC] = incl;
    for (int64_t b0 = lo; b0 < hi; b0 += 32 * U) {
        double v[U];
        int32_t rw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t x = b0 + 32 * u + lane;
            v[u] = x < hi ? col_vals[x] : 0.0;
            rw[u] = x < hi ? col_rows[x] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = b0 + 32 * u + lane < hi ? cls(v[u]) : -1;
            for (int cc = 0; cc < NC; ++cc) {
                const unsigned bal = __ballot_sync(0xffffffffu, c == cc);
                if (!bal) continue;
                const int base = __shfl_sync(0xffffffffu, run, cc);
                if (c == cc) rows_by_class[lo + base + __popc(bal & lt)] = rw[u];
                if ((int)lane == cc) run += __popc(bal);
            }
        }
    }
}

// Distinct rating values (up to kHsMaxClasses): per-block sets in shared memory
// (warp leaders found with __match_any_sync), merged by a one-block pass.
// out layout per block: [count or -1 on overflow, v0..v15] as doubles.
// Lock-free set of up to kHsMaxClasses distinct values per block: slots start
// EMPTY (a NaN payload; ratings are finite) and are claimed with atomicCAS, so a
// value can never be inserted twice.  Each thread loads 4 values up front.
__global__ void value_set_kernel(const double *__restrict__ vals, int64_t n, double *__restrict__ out) {
    constexpr unsigned long long EMPTY = 0x7FF4DEADBEEF0001ULL;
    __shared__ unsigned long long s_set[kHsMaxClasses];
    __shared__ int s_over;
    if (threadIdx.x < kHsMaxClasses) s_set[threadIdx.x] = EMPTY;
    if (threadIdx.x == 0) s_over = 0;
    __syncthreads();
    // each thread first collects its own distinct values in registers (compares only, no
    // shared-memory round trips per element), then merges them into the block set once
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    unsigned long long own[kHsMaxClasses];
    int n_own = 0;
    bool over = false;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += 4 * step) {
        unsigned long long v4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t x = base + u * step + threadIdx.x;
            v4[u] = x < n ? (unsigned long long)__double_as_longlong(vals[x]) : EMPTY;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned long long v = v4[u];
            bool found = v == EMPTY;
#pragma unroll
            for (int k = 0; k < kHsMaxClasses; ++k) found |= (k < n_own) && own[k] == v;
            if (!found) {
                if (n_own == kHsMaxClasses) {
                    over = true;
                } else {
#pragma unroll
                    for (int k = 0; k < kHsMaxClasses; ++k)
                        if (k == n_own) own[k] = v;
                    ++n_own;
                }
            }
        }
    }
    if (over) s_over = 1;
#pragma unroll
    for (int q = 0; q < kHsMaxClasses; ++q) {
        if (q >= n_own) break;
        const unsigned long long v = own[q];
        bool found = false;
        for (int k = 0; k < kHsMaxClasses && !found; ++k)
            found = ((volatile unsigned long long *)s_set)[k] == v;
        if (found) continue;
        int k = 0;
        for (; k < kHsMaxClasses; ++k) {
            const unsigned long long old = atomicCAS(&s_set[k], EMPTY, v);
            if (old == EMPTY || old == v) break;
        }
        if (k == kHsMaxClasses) s_over = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double *o = out + blockIdx.x * (kHsMaxClasses + 1);
        int cnt = 0;
        for (int k = 0; k < kHsMaxClasses; ++k)
            if (s_set[k] != EMPTY) o[1 + cnt++] = __longlong_as_double((long long)s_set[k]);
        for (int k = cnt; k < kHsMaxClasses; ++k) o[1 + k] = 0.0;
        o[0] = s_over ? -1.0 : (double)cnt;
    }
}

__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}

// bit-sliced count of position t: sum_k ((V[k] >> t) & 1) << k
__device__ __forceinline__ int sliced_count(const uint32_t *V, int D, int t) {
    int c = 0;
#pragma unroll
    for (int k = 0; k < kHsDepth; ++k) c |= (int)((V[k] >> t) & 1u) << k;
    (void)D;
    return c;
}

constexpr int kHsRing = 4;        // 16-row groups in flight per CTA (64 row records)

// CTA per column.  Thread 0 gathers whole row records (stride bytes, 16-aligned) of
// the next groups into a shared-memory ring with the bulk-copy engine
// (cp.async.bulk + mbarrier transaction counts); every thread then reads its own
// 32-bit word of each record from shared memory and runs the CSA tree.
// (128, 7): 72 registers instead of 96 (a few bytes of spill) so 7 CTAs fit per SM instead
// of 6 — the kernel is gather-latency-bound — with the shared-memory carveout at its maximum:
// 7.84 -> 7.13 ms at C3 (A/B, tools/gpu_ab_lsh.sh)
template <bool kTma>
__global__ void __launch_bounds__(128, 7)
hash_count_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ rows_by_class,
                  const int32_t *__restrict__ class_off, int NC, const int *__restrict__ class_psi,
                  int64_t col_begin, const uint8_t *__restrict__ table, int stride, int W4, int qp, int p,
                  int G, int ns, int pad_row, int row_lo, int row_hi, int first, int last,
                  double *__restrict__ acc, uint8_t *__restrict__ sig, uint64_t *__restrict__ keys,
                  int64_t keys_ld) {
    __shared__ int32_t s_rows[kHsChunk];
    __shared__ __align__(8) uint64_t s_bar[kHsRing];
    extern __shared__ __align__(16) uint8_t s_dyn[];
    uint8_t *s_ring = s_dyn;                                        // kHsRing * 16 * stride (TMA)
    uint8_t *s_sigbyte = s_dyn + (kTma ? (size_t)kHsRing * 16 * stride : 0);   // W4*4 bytes (padded)
    int *a32 = reinterpret_cast<int *>(s_sigbyte + ((W4 * 4 + 15) & ~15)) + threadIdx.x;
    const int astr = blockDim.x;
    const int64_t j = col_begin + blockIdx.x;
    const int lw = threadIdx.x;              // word lane: slices 4*lw .. 4*lw+3
    const bool active = lw < W4;
    const int64_t lo = col_ptr[j];
    const int32_t *coff = class_off + j * (NC + 1);
    const int64_t accW = (int64_t)qp * G;
    const unsigned gbytes = 16u * (unsigned)stride;

    if (threadIdx.x == 0) {
        for (int k = 0; k < kHsRing; ++k) mbar_init(&s_bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // running sums of earlier row-range passes come back from acc (exact integers)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int s = 4 * lw + b;
        const bool ok = active && s < qp * ns;
        const int gm = ok ? s / ns : 0, sl = ok ? s % ns : 0;
        const int nbits = ok ? min(8, G - 8 * sl) : 0;
        const double *a_in = acc + j * accW + (int64_t)gm * G + 8 * sl;
#pragma unroll
        for (int t = 0; t < 8; ++t) a32[(8 * b + t) * astr] = (!first && t < nbits) ? (int)a_in[t] : 0;
    }
    __syncthreads();
    unsigned issued = 0, consumed = 0;   // group counters (identical in every thread)

    for (int c = 0; c < NC; ++c) {
        int c_lo = coff[c], c_hi = coff[c + 1];
        if (c_hi <= c_lo) continue;          // uniform across the CTA
        {   // this pass's rows [row_lo, row_hi): the class segment is row-sorted
            const int32_t *seg = rows_by_class + lo;
            int l = c_lo, h = c_hi;
            while (l < h) { const int m = (l + h) >> 1; if (seg[m] < row_lo) l = m + 1; else h = m; }
            const int a = l;
            h = c_hi;
            while (l < h) { const int m = (l + h) >> 1; if (seg[m] < row_hi) l = m + 1; else h = m; }
            c_lo = a;
            c_hi = l;
        }
        if (c_hi <= c_lo) continue;
        const int psi = class_psi[c];
        uint32_t ones = 0, twos = 0, fours = 0, eights = 0;
        uint32_t V[kHsDepth];
#pragma unroll
        for (int k = 0; k < kHsDepth; ++k) V[k] = 0;
        int groups = 0, done_since_flush = 0;
        auto flush = [&](int n_done) {
            // class contribution psi * (2 * count - n_done), count from the sliced state
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                const int cnt = 16 * sliced_count(V, kHsDepth, t) + 8 * (int)((eights >> t) & 1u) +
                                4 * (int)((fours >> t) & 1u) + 2 * (int)((twos >> t) & 1u) +
                                (int)((ones >> t) & 1u);
                a32[t * astr] += psi * (2 * cnt - n_done);
            }
            ones = twos = fours = eights = 0;
#pragma unroll
            for (int k = 0; k < kHsDepth; ++k) V[k] = 0;
        };
        for (int c0 = c_lo; c0 < c_hi; c0 += kHsChunk) {
            const int n = min(kHsChunk, c_hi - c0);
            const int n16 = (n + 15) & ~15;   // tail padded with the all-zero row
            __syncthreads();                  // previous chunk fully consumed
            for (int x = threadIdx.x; x < n16; x += blockDim.x)
                s_rows[x] = x < n ? rows_by_class[lo + c0 + x] : pad_row;
            __syncthreads();
            const int ng = n16 / 16;
            // lanes 0..15 of warp 0 each gather one row record of the group
            auto issue = [&](int g) {
                const unsigned slot = issued % kHsRing;
                uint64_t *bar = &s_bar[slot];
                if (threadIdx.x == 0) mbar_expect_tx(bar, gbytes);
                __syncwarp();
                if (threadIdx.x < 16) {
                    uint8_t *dst = s_ring + (size_t)slot * gbytes + threadIdx.x * stride;
                    bulk_g2s(dst, table + (int64_t)s_rows[16 * g + threadIdx.x] * stride, stride, bar);
                }
            };
            if (kTma && threadIdx.x < 32) {
                for (int g = 0; g < min(kHsRing, ng); ++g) { issue(g); ++issued; }
            } else {
                issued += min(kHsRing, ng);
            }
            const uint32_t *tab32 = reinterpret_cast<const uint32_t *>(table) + lw;
            const int sw = stride >> 2;
            uint32_t wn[16];
            if (!kTma && active) {
#pragma unroll
                for (int q = 0; q < 16; ++q) wn[q] = __ldg(tab32 + (int64_t)s_rows[q] * sw);
            }
            for (int g = 0; g < ng; ++g) {
                const unsigned slot = consumed % kHsRing;
                if (kTma) mbar_wait(&s_bar[slot], (consumed / kHsRing) & 1u);
                if (active) {
                    uint32_t w[16];
                    if (kTma) {
                        const uint32_t *src = reinterpret_cast<const uint32_t *>(s_ring + (size_t)slot * gbytes) + lw;
#pragma unroll
                        for (int q = 0; q < 16; ++q) w[q] = src[q * sw];
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q) w[q] = wn[q];
                        if (g + 1 < ng) {   // next group's loads in flight during this group's CSA tree
#pragma unroll
                            for (int q = 0; q < 16; ++q) wn[q] = __ldg(tab32 + (int64_t)s_rows[16 * (g + 1) + q] * sw);
                        }
                    }
                    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
                    csa(twosA, ones, ones, w[0], w[1]);
                    csa(twosB, ones, ones, w[2], w[3]);
                    csa(foursA, twos, twos, twosA, twosB);
                    csa(twosA, ones, ones, w[4], w[5]);
                    csa(twosB, ones, ones, w[6], w[7]);
                    csa(foursB, twos, twos, twosA, twosB);
                    csa(eightsA, fours, fours, foursA, foursB);
                    csa(twosA, ones, ones, w[8], w[9]);
                    csa(twosB, ones, ones, w[10], w[11]);
                    csa(foursA, twos, twos, twosA, twosB);
                    csa(twosA, ones, ones, w[12], w[13]);
                    csa(twosB, ones, ones, w[14], w[15]);
                    csa(foursB, twos, twos, twosA, twosB);
                    csa(eightsB, fours, fours, foursA, foursB);
                    csa(sixteens, eights, eights, eightsA, eightsB);
                    uint32_t carry = sixteens;
#pragma unroll
                    for (int k = 0; k < kHsDepth; ++k) {
                        const uint32_t t2 = V[k] & carry;
                        V[k] ^= carry;
                        carry = t2;
                    }
                    ++groups;
                    done_since_flush += min(16, n - 16 * g);
                    if (groups == (1 << kHsDepth) - 1) {   // counter full: fold into a32
                        flush(done_since_flush);
                        groups = 0;
                        done_since_flush = 0;
                    }
                }
                ++consumed;
                if (kTma) {
                    __syncthreads();               // slot free for the producer
                    if (g + kHsRing < ng) {
                        if (threadIdx.x < 32) issue(g + kHsRing);
                        ++issued;
                    }
                }
            }
        }
        if (active) flush(done_since_flush);
    }
    if (active && !last) {   // park the partial sums for the next pass
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int s = 4 * lw + b;
            if (s >= qp * ns) break;
            const int gm = s / ns, sl = s % ns;
            const int nbits = min(8, G - 8 * sl);
            double *a_out = acc + j * accW + (int64_t)gm * G + 8 * sl;
            for (int t = 0; t < nbits; ++t) a_out[t] = (double)a32[(8 * b + t) * astr];
        }
    }
    if (!last) return;
    if (active) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int s = 4 * lw + b;
            if (s >= qp * ns) break;
            const int gm = s / ns, sl = s % ns;
            const int nbits = min(8, G - 8 * sl);
            double *a_out = acc + j * accW + (int64_t)gm * G + 8 * sl;
            uint32_t sb = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const double v = (double)a32[(8 * b + t) * astr];
                if (t < nbits) {
                    a_out[t] = v;
                    sb |= (v >= 0.0 ? 1u : 0u) << t;
                }
            }
            if (sig) {
                uint8_t *sg = sig + j * accW + (int64_t)gm * G + 8 * sl;
                for (int t = 0; t < nbits; ++t) sg[t] = (sb >> t) & 1u;
            }
            s_sigbyte[s] = (uint8_t)sb;
        }
    }
    if (keys) {
        __syncthreads();
        const int q = qp / p;
        for (int g = threadIdx.x; g < q; g += blockDim.x) {
            uint64_t k = 0;
            for (int m = 0; m < p; ++m)
                for (int sl = 0; sl < ns; ++sl)
                    k |= (uint64_t)s_sigbyte[(g * p + m) * ns + sl] << (m * G + 8 * sl);
            keys[(int64_t)g * keys_ld + j] = k;
        }
    }
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_class_partition(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                                     int64_t N, const double *class_vals, int NC, int32_t *rows_by_class,
                                     int32_t *class_off, void *stream) {
    CULSH_REQUIRE(NC >= 1 && NC <= kHsMaxClasses, "1..16 value classes supported");
    if (N <= 0) return CULSH_OK;
    class_partition_kernel<<<(unsigned)((N + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
        col_ptr, col_rows, col_vals, N, class_vals, NC, rows_by_class, class_off);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_hash_count(const int64_t *col_ptr, const int32_t *rows_by_class, const int32_t *class_off,
                                int NC, const int *class_psi, int64_t M, int max_slice_mb, int variant,
                                int64_t col_begin, int64_t n_cols, const uint8_t *table, int q, int p, int G,
                                double *acc, uint8_t *sig, uint64_t *keys, int64_t keys_ld, void *stream) {
    CULSH_REQUIRE(q >= 1 && p >= 1 && G >= 1 && G <= 64 && p * G <= 64, "bad LSH config");
    CULSH_REQUIRE(NC >= 1 && NC <= kHsMaxClasses, "1..16 value classes supported");
    const int ns = (G + 7) / 8;
    const int W8 = q * p * ns;
    CULSH_REQUIRE(W8 % 4 == 0, "bit-count path needs q*p*ceil(G/8) divisible by 4");
    CULSH_REQUIRE((reinterpret_cast<uintptr_t>(table) & 15) == 0, "row-hash table must be 16-byte aligned");
    if (n_cols <= 0) return CULSH_OK;
    const int W4 = W8 / 4;
    const int stride = (int)table_stride(q * p, ns);
    int threads = ((W4 + 31) / 32) * 32;
    CULSH_REQUIRE(threads <= 128, "q*p*ceil(G/8) > 512 bytes: use culsh_hash_accumulate");
    const size_t smem = (size_t)kHsRing * 16 * stride + (size_t)((W4 * 4 + 15) & ~15) +
                        sizeof(int) * 32 * threads;
    {   // per device and cheap: set on every launch (a once-per-process flag breaks on a 2nd GPU)
        cudaFuncSetAttribute(hash_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(hash_count_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(hash_count_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    const bool use_tma = variant == 0;
    const size_t smem_k = use_tma ? smem : smem - (size_t)kHsRing * 16 * stride;
    CULSH_REQUIRE(smem <= 96 * 1024, "row record too large for the staging ring");
    int passes = 1;
    if (max_slice_mb > 0) {
        const int64_t slice_bytes = (int64_t)max_slice_mb << 20;
        passes = (int)((M * (int64_t)stride + slice_bytes - 1) / slice_bytes);
        if (passes < 1) passes = 1;
        if (passes > 64) passes = 64;
    }
    for (int ps = 0; ps < passes; ++ps) {
        const int r0 = (int)((M * ps) / passes), r1 = (int)((M * (ps + 1)) / passes);
        if (use_tma)
            hash_count_kernel<true><<<(unsigned)n_cols, threads, smem_k, (cudaStream_t)stream>>>(
                col_ptr, rows_by_class, class_off, NC, class_psi, col_begin, table, stride, W4, q * p, p, G,
                ns, (int)M, r0, r1, ps == 0, ps == passes - 1, acc, sig, keys, keys_ld);
        else
            hash_count_kernel<false><<<(unsigned)n_cols, threads, smem_k, (cudaStream_t)stream>>>(
                col_ptr, rows_by_class, class_off, NC, class_psi, col_begin, table, stride, W4, q * p, p, G,
                ns, (int)M, r0, r1, ps == 0, ps == passes - 1, acc, sig, keys, keys_ld);
        CULSH_LAUNCH_CHECK();
    }
    return CULSH_OK;
}

extern "C" int culsh_row_hash_table(uint64_t seed, int q, int p, int G, int64_t row_lo, int64_t row_hi,
                                    uint8_t *table, void *stream) {
    CULSH_REQUIRE(q >= 1 && p >= 1 && G >= 1 && G <= 64 && p * G <= 64, "bad LSH config");
    if (row_hi <= row_lo) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *keys = nullptr;
    keep_pool_memory();
    CULSH_CHECK(cudaMallocAsync(&keys, sizeof(uint64_t) * q * p, st));
    map_keys_kernel<<<(q * p + 255) / 256, 256, 0, st>>>(seed, q, p, keys);
    const int ns = (G + 7) / 8;
    const int64_t total = (row_hi - row_lo) * (int64_t)q * p;
    const int blocks = (int)min64((total + 255) / 256, (int64_t)num_sms() * 16);
    row_hash_kernel<<<blocks, 256, 0, st>>>(keys, q * p, G, ns, row_lo, row_hi, table);
    CULSH_LAUNCH_CHECK();
    CULSH_CHECK(cudaFreeAsync(keys, st));
    return CULSH_OK;
}

extern "C" int culsh_pack_bits(const uint8_t *bits, int64_t M, int q, int p, int G, uint8_t *table,
                               void *stream) {
    CULSH_REQUIRE(G >= 1 && G <= 64, "bad G");
    const int ns = (G + 7) / 8;
    const int64_t total = M * (int64_t)q * p * ns;
    if (total == 0) return CULSH_OK;
    const int blocks = (int)min64((total + 255) / 256, (int64_t)num_sms() * 16);
    pack_bits_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, M, q * p, G, ns, table);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_unpack_bits(const uint8_t *table, int64_t M, int q, int p, int G, uint8_t *bits,
                                 void *stream) {
    CULSH_REQUIRE(G >= 1 && G <= 64, "bad G");
    const int ns = (G + 7) / 8;
    const int64_t total = M * (int64_t)q * p * G;
    if (total == 0) return CULSH_OK;
    const int blocks = (int)min64((total + 255) / 256, (int64_t)num_sms() * 16);
    unpack_bits_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(table, M, q * p, G, ns, bits);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_psi_int_check(const int64_t *col_ptr, const double *col_vals, int64_t col_begin,
                                   int64_t n_cols, const int32_t *col_list, int e, int *bad_out,
                                   void *stream) {
    if (n_cols <= 0) return CULSH_OK;
    const int wpb = 8;
    psi_int_check_kernel<<<(unsigned)((n_cols + wpb - 1) / wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
        col_ptr, col_vals, col_begin, n_cols, col_list, e, bad_out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_hash_accumulate(const int64_t *col_ptr, const int32_t *col_rows,
                                     const double *col_vals, int64_t col_begin, int64_t n_cols,
                                     const int32_t *col_list, const uint8_t *table, int q, int p,
                                     int G, int e, int into, int int_path, double *acc,
                                     uint8_t *sig, uint64_t *keys, int64_t keys_ld, void *stream) {
    CULSH_REQUIRE(q >= 1 && p >= 1 && G >= 1 && G <= 64 && p * G <= 64, "bad LSH config");
    CULSH_REQUIRE(e == 1 || e == 2 || e == 4, "psi exponent must be 1, 2 or 4");
    CULSH_REQUIRE(!(into && int_path), "incremental accumulation runs the ordered fp64 path");
    if (n_cols <= 0) return CULSH_OK;
    CULSH_REQUIRE(n_cols < (1LL << 31), "too many columns for one launch");
    const int ns = (G + 7) / 8;
    const int W8 = q * p * ns;
    int threads = ((W8 + 31) / 32) * 32;
    if (threads > 512) threads = 512;
    const size_t smem = (size_t)W8;
    CULSH_REQUIRE(smem <= 48 * 1024, "q*p*ceil(G/8) exceeds the per-column key staging buffer");
    cudaStream_t st = (cudaStream_t)stream;
    if (int_path)
        hash_accumulate_kernel<int><<<(unsigned)n_cols, threads, smem, st>>>(
            col_ptr, col_rows, col_vals, col_begin, n_cols, col_list, table, q * p, p, G, ns, e, into,
            acc, sig, keys, keys_ld);
    else
        hash_accumulate_kernel<double><<<(unsigned)n_cols, threads, smem, st>>>(
            col_ptr, col_rows, col_vals, col_begin, n_cols, col_list, table, q * p, p, G, ns, e, into,
            acc, sig, keys, keys_ld);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// Per-block distinct-value sets of `vals` (out: n_blocks x 17 doubles, see
// value_set_kernel); the caller merges them.  n_blocks <= 4096.
extern "C" int culsh_value_set(const double *vals, int64_t n, double *out, int n_blocks, void *stream) {
    CULSH_REQUIRE(n_blocks >= 1 && n_blocks <= 4096, "n_blocks must be in [1, 4096]");
    value_set_kernel<<<n_blocks, 256, 0, (cudaStream_t)stream>>>(vals, n, out);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// lsh.py:246-260 _pack_group_keys for a given signature tensor sig (N, q, p, G) u8:
// keys[g, j] bit (m*G + t) = sig[j, g, m, t] != 0.
__global__ void pack_keys_kernel(const uint8_t *__restrict__ sig, int64_t N, int q, int p, int G,
                                 uint64_t *__restrict__ keys) {
    const int64_t total = N * (int64_t)q;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = x / q;
        const int g = (int)(x % q);
        const uint8_t *s = sig + (j * q + g) * (int64_t)p * G;
        uint64_t k = 0;
        for (int b = 0; b < p * G; ++b) k |= (uint64_t)(s[b] != 0) << b;
        keys[(int64_t)g * N + j] = k;
    }
}

extern "C" int culsh_pack_keys(const uint8_t *sig, int64_t N, int q, int p, int G, uint64_t *keys, void *stream) {
    CULSH_REQUIRE(q >= 1 && p >= 1 && G >= 1 && p * G <= 64, "p*G exceeds the 64-bit bucket key");
    if (N <= 0) return CULSH_OK;
    const int64_t total = N * (int64_t)q;
    const int blocks = (int)min64((total + 255) / 256, (int64_t)num_sms() * 8);
    pack_keys_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sig, N, q, p, G, keys);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
