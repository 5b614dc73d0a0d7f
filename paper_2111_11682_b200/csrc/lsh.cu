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

__global__ void map_keys_kernel(uint64_t seed, int q, int p, uint64_t *keys) {
    int gm = blockIdx.x * blockDim.x + threadIdx.x;
    if (gm < q * p) keys[gm] = map_key(seed, gm / p, gm % p);
}

// table[i][g][m][s] = byte s of the low G bits of splitmix64(key(g,m) ^ i)
__global__ void row_hash_kernel(const uint64_t *__restrict__ keys, int qp, int G, int ns,
                                int64_t row_lo, int64_t row_hi, uint8_t *__restrict__ table) {
    const int64_t rec = (int64_t)qp * ns;
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
        table[x] = v;
    }
}

__global__ void unpack_bits_kernel(const uint8_t *__restrict__ table, int64_t M, int qp, int G, int ns,
                                   uint8_t *__restrict__ bits) {
    const int64_t total = M * (int64_t)qp * G;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t igm = x / G;
        const int t = (int)(x % G);
        bits[x] = (table[igm * ns + t / 8] >> (t % 8)) & 1;
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
    const int64_t rec = (int64_t)W8;
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

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_row_hash_table(uint64_t seed, int q, int p, int G, int64_t row_lo, int64_t row_hi,
                                    uint8_t *table, void *stream) {
    CULSH_REQUIRE(q >= 1 && p >= 1 && G >= 1 && G <= 64 && p * G <= 64, "bad LSH config");
    if (row_hi <= row_lo) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *keys = nullptr;
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
