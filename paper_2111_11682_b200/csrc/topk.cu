// Bucket build and frequency top-K.
//
// Reference semantics (bit-exact):
//   per group g: stable argsort of keys[g] -> runs of equal keys      lsh.py:263-287
//   candidates of column j: bucket mates != j concatenated over g      lsh.py:308-328
//   rank by (occurrence count desc, column asc); if fewer than K
//   distinct candidates, supplement c = splitmix64(key ^ t) % N_total
//   skipping j and repeats, key = sm(sm(seed ^ 0xC0FFEE) ^ j)          lsh.py:331-374
//   insertion with strict compares (ties -> lower index)               similarity.py:137-161
//
// Device plan: one segmented radix sort of the (q, N) key matrix (one segment
// per group, only the p*G significant bits), a run-walk that writes each
// column's bucket [start, end) per group, a per-target-column count + scan,
// candidate gather, a segmented sort of each column's candidate list, then a
// per-column selection thread that replays the reference's insertion logic.
#include <cub/cub.cuh>

#include "common.cuh"

namespace culsh {

__global__ void iota_cols_kernel(int32_t *vals, int q, int64_t N, int *seg) {
    const int64_t total = (int64_t)q * N;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x)
        vals[x] = (int32_t)(x % N);
    if (blockIdx.x == 0)
        for (int g = threadIdx.x; g <= q; g += blockDim.x) seg[g] = (int)(g * N);
}

// One thread per run head: writes [start, end) of its run for every member column.
__global__ void runs_kernel(const uint64_t *__restrict__ skeys, const int32_t *__restrict__ scols,
                            int q, int64_t N, int32_t *__restrict__ rs, int32_t *__restrict__ re) {
    const int64_t total = (int64_t)q * N;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = x / N, pos = x % N;
        const uint64_t *kg = skeys + g * N;
        if (pos > 0 && kg[pos] == kg[pos - 1]) continue;
        int64_t end = pos + 1;
        while (end < N && kg[end] == kg[pos]) ++end;
        for (int64_t y = pos; y < end; ++y) {
            const int32_t c = scols[g * N + y];
            rs[g * N + c] = (int32_t)pos;
            re[g * N + c] = (int32_t)end;
        }
    }
}

__global__ void cand_count_kernel(const int32_t *__restrict__ rs, const int32_t *__restrict__ re,
                                  int q, int64_t N, int64_t j_base, int64_t n_cols,
                                  int64_t *__restrict__ counts) {
    for (int64_t jj = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; jj < n_cols;
         jj += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = j_base + jj;
        int64_t c = 0;
        for (int g = 0; g < q; ++g) c += re[g * N + j] - rs[g * N + j] - 1;
        counts[jj] = c;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) counts[n_cols] = 0;
}

__global__ void cand_fill_kernel(const int32_t *__restrict__ scols, const int32_t *__restrict__ rs,
                                 const int32_t *__restrict__ re, int q, int64_t N, int64_t j_base,
                                 int64_t n_cols, const int64_t *__restrict__ offsets,
                                 int32_t *__restrict__ cand) {
    for (int64_t jj = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; jj < n_cols;
         jj += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = j_base + jj;
        int64_t o = offsets[jj];
        for (int g = 0; g < q; ++g) {
            const int32_t *sg = scols + g * N;
            for (int32_t pos = rs[g * N + j]; pos < re[g * N + j]; ++pos) {
                const int32_t c = sg[pos];
                if (c != j) cand[o++] = c;
            }
        }
    }
}

constexpr int kMaxK = 128;

// similarity.py:137-161 _topk_insert, unchanged control flow.
__device__ __forceinline__ int topk_insert(int *best_cnt, int32_t *best_idx, int count, int K, int s,
                                           int32_t j2) {
    if (count < K) {
        int pos = count;
        while (pos > 0 && best_cnt[pos - 1] < s) {
            best_cnt[pos] = best_cnt[pos - 1];
            best_idx[pos] = best_idx[pos - 1];
            --pos;
        }
        best_cnt[pos] = s;
        best_idx[pos] = j2;
        return count + 1;
    }
    if (s > best_cnt[K - 1]) {
        int pos = K - 1;
        while (pos > 0 && best_cnt[pos - 1] < s) {
            best_cnt[pos] = best_cnt[pos - 1];
            best_idx[pos] = best_idx[pos - 1];
            --pos;
        }
        best_cnt[pos] = s;
        best_idx[pos] = j2;
    }
    return count;
}

__global__ void select_kernel(const int32_t *__restrict__ cand, const int64_t *__restrict__ offsets,
                              int64_t j_base, int64_t n_cols, int K, uint64_t seed, int64_t N_total,
                              int32_t *__restrict__ entries) {
    int best_cnt[kMaxK];
    int32_t best_idx[kMaxK];
    for (int64_t jj = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; jj < n_cols;
         jj += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = j_base + jj;
        const int64_t lo = offsets[jj], hi = offsets[jj + 1];
        int count = 0;
        int64_t a = lo;
        while (a < hi) {
            int64_t b = a;
            const int32_t v = cand[a];
            while (b < hi && cand[b] == v) ++b;
            count = topk_insert(best_cnt, best_idx, count, K, (int)(b - a), v);
            a = b;
        }
        if (count < K) {
            const uint64_t key = splitmix64(splitmix64(seed ^ 0xC0FFEEULL) ^ (uint64_t)j);
            uint64_t t = 0;
            while (count < K) {
                const uint64_t h = splitmix64(key ^ t);
                t += 1;
                const int32_t c = (int32_t)(h % (uint64_t)N_total);
                if (c == j) continue;
                bool dup = false;
                for (int x = 0; x < count; ++x)
                    if (best_idx[x] == c) { dup = true; break; }
                if (!dup) {
                    best_idx[count] = c;
                    best_cnt[count] = 0;
                    ++count;
                }
            }
        }
        for (int k = 0; k < K; ++k) entries[jj * K + k] = best_idx[k];
    }
}

struct DevBuf {
    void *p = nullptr;
    cudaStream_t st;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    cudaError_t alloc(size_t n) {
        keep_pool_memory();
        return cudaMallocAsync(&p, n ? n : 16, st);
    }
    ~DevBuf() { if (p) cudaFreeAsync(p, st); }
    template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};

// ---- host-side stages -------------------------------------------------------

// Buckets of every group: per (g, column) the [start, end) of its run of equal keys
// in the group's key-sorted order (scols).  rs/re/scols are (q, N_total) int32.
static int build_runs(const uint64_t *keys, int q, int64_t N_total, int key_bits, DevBuf &scols, DevBuf &rs,
                      DevBuf &re, cudaStream_t st) {
    const int64_t QN = (int64_t)q * N_total;
    const int grid = (int)min64((QN + 255) / 256, (int64_t)num_sms() * 8);
    DevBuf skeys(st), vals_in(st), seg(st), tmp(st);
    CULSH_CHECK(skeys.alloc(sizeof(uint64_t) * QN));
    CULSH_CHECK(vals_in.alloc(sizeof(int32_t) * QN));
    CULSH_CHECK(scols.alloc(sizeof(int32_t) * QN));
    CULSH_CHECK(seg.alloc(sizeof(int) * (q + 1)));
    iota_cols_kernel<<<grid, 256, 0, st>>>(vals_in.as<int32_t>(), q, N_total, seg.as<int>());
    CULSH_LAUNCH_CHECK();
    size_t tb = 0;
    CULSH_CHECK(cub::DeviceSegmentedRadixSort::SortPairs(
        nullptr, tb, keys, skeys.as<uint64_t>(), vals_in.as<int32_t>(), scols.as<int32_t>(), (int)QN, q,
        seg.as<int>(), seg.as<int>() + 1, 0, key_bits, st));
    CULSH_CHECK(tmp.alloc(tb));
    CULSH_CHECK(cub::DeviceSegmentedRadixSort::SortPairs(
        tmp.p, tb, keys, skeys.as<uint64_t>(), vals_in.as<int32_t>(), scols.as<int32_t>(), (int)QN, q,
        seg.as<int>(), seg.as<int>() + 1, 0, key_bits, st));
    CULSH_CHECK(rs.alloc(sizeof(int32_t) * QN));
    CULSH_CHECK(re.alloc(sizeof(int32_t) * QN));
    runs_kernel<<<grid, 256, 0, st>>>(skeys.as<uint64_t>(), scols.as<int32_t>(), q, N_total, rs.as<int32_t>(),
                                      re.as<int32_t>());
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// offsets (n_cols+1, device int64) = exclusive prefix of per-target candidate counts;
// returns the total through *total_host (one small D2H).
static int candidate_offsets(const DevBuf &rs, const DevBuf &re, int q, int64_t N_total, int64_t j_base,
                             int64_t n_cols, int64_t *offsets, int64_t *total_host, cudaStream_t st) {
    DevBuf counts(st), tmp(st);
    CULSH_CHECK(counts.alloc(sizeof(int64_t) * (n_cols + 1)));
    const int gridc = (int)min64((n_cols + 127) / 128, (int64_t)num_sms() * 8);
    cand_count_kernel<<<gridc, 128, 0, st>>>(rs.as<int32_t>(), re.as<int32_t>(), q, N_total, j_base, n_cols,
                                             counts.as<int64_t>());
    CULSH_LAUNCH_CHECK();
    size_t tb = 0;
    CULSH_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.as<int64_t>(), offsets, (int)(n_cols + 1), st));
    CULSH_CHECK(tmp.alloc(tb));
    CULSH_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, counts.as<int64_t>(), offsets, (int)(n_cols + 1), st));
    CULSH_CHECK(cudaMemcpyAsync(total_host, offsets + n_cols, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CULSH_CHECK(cudaStreamSynchronize(st));
    return CULSH_OK;
}

static int sort_segments(const int32_t *in, int32_t *out, int64_t total, int64_t n_cols, const int64_t *offsets,
                         cudaStream_t st) {
    if (total <= 0) return CULSH_OK;
    size_t tb = 0;
    CULSH_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, in, out, (int)total, (int)n_cols, offsets,
                                                   offsets + 1, st));
    DevBuf tmp(st);
    CULSH_CHECK(tmp.alloc(tb));
    CULSH_CHECK(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, in, out, (int)total, (int)n_cols, offsets,
                                                   offsets + 1, st));
    return CULSH_OK;
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_candidates(const uint64_t *keys, int q, int64_t N_total, int key_bits, int64_t j_base,
                                int64_t n_cols, int64_t *offsets, int32_t *cand, int64_t cand_capacity,
                                int64_t *n_candidates_out, void *stream) {
    CULSH_REQUIRE(q >= 1 && N_total >= 1, "empty key matrix");
    CULSH_REQUIRE((int64_t)q * N_total < (1LL << 31), "q*N too large for one sort");
    CULSH_REQUIRE(j_base >= 0 && j_base + n_cols <= N_total, "target columns out of range");
    if (key_bits <= 0 || key_bits > 64) key_bits = 64;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf scols(st), rs(st), re(st);
    int r = build_runs(keys, q, N_total, key_bits, scols, rs, re, st);
    if (r != CULSH_OK) return r;
    int64_t total = 0;
    if (n_cols > 0) {
        r = candidate_offsets(rs, re, q, N_total, j_base, n_cols, offsets, &total, st);
        if (r != CULSH_OK) return r;
    }
    if (n_candidates_out) *n_candidates_out = total;
    if (!cand || total == 0) return CULSH_OK;
    CULSH_REQUIRE(cand_capacity >= total, "candidate buffer too small");
    CULSH_REQUIRE(total < (1LL << 31), "candidate list exceeds 2^31 entries");
    DevBuf raw(st);
    CULSH_CHECK(raw.alloc(sizeof(int32_t) * total));
    const int gridc = (int)min64((n_cols + 127) / 128, (int64_t)num_sms() * 8);
    cand_fill_kernel<<<gridc, 128, 0, st>>>(scols.as<int32_t>(), rs.as<int32_t>(), re.as<int32_t>(), q, N_total,
                                            j_base, n_cols, offsets, raw.as<int32_t>());
    CULSH_LAUNCH_CHECK();
    return sort_segments(raw.as<int32_t>(), cand, total, n_cols, offsets, st);
}

extern "C" int culsh_select_topk(const int32_t *cand, const int64_t *offsets, int64_t total, int64_t j_base,
                                 int64_t n_cols, int K, uint64_t seed, int64_t N_total, int32_t *entries,
                                 void *stream) {
    CULSH_REQUIRE(K >= 0 && K <= kMaxK, "K out of supported range [0, 128]");
    CULSH_REQUIRE(K <= N_total - 1 || n_cols == 0, "K exceeds N-1");
    if (n_cols <= 0 || K == 0) return CULSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf sorted(st);
    CULSH_CHECK(sorted.alloc(sizeof(int32_t) * (total > 0 ? total : 1)));
    int r = sort_segments(cand, sorted.as<int32_t>(), total, n_cols, offsets, st);
    if (r != CULSH_OK) return r;
    const int gridc = (int)min64((n_cols + 127) / 128, (int64_t)num_sms() * 8);
    select_kernel<<<gridc, 128, 0, st>>>(sorted.as<int32_t>(), offsets, j_base, n_cols, K, seed, N_total, entries);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_topk(const uint64_t *keys, int q, int64_t N_total, int key_bits, int64_t j_base,
                          int64_t n_cols, int K, uint64_t seed, int32_t *entries,
                          int64_t *n_candidates_out, void *stream) {
    CULSH_REQUIRE(q >= 1 && N_total >= 1, "empty key matrix");
    CULSH_REQUIRE(K >= 0 && K <= kMaxK, "K out of supported range [0, 128]");
    CULSH_REQUIRE(K <= N_total - 1 || n_cols == 0, "K exceeds N-1");
    CULSH_REQUIRE((int64_t)q * N_total < (1LL << 31), "q*N too large for one sort");
    CULSH_REQUIRE(j_base >= 0 && j_base + n_cols <= N_total, "target columns out of range");
    if (key_bits <= 0 || key_bits > 64) key_bits = 64;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf scols(st), rs(st), re(st), offsets(st), cand(st), cand_sorted(st);
    int r = build_runs(keys, q, N_total, key_bits, scols, rs, re, st);
    if (r != CULSH_OK) return r;
    if (n_cols == 0) {
        if (n_candidates_out) *n_candidates_out = 0;
        return CULSH_OK;
    }
    CULSH_CHECK(offsets.alloc(sizeof(int64_t) * (n_cols + 1)));
    int64_t total = 0;
    r = candidate_offsets(rs, re, q, N_total, j_base, n_cols, offsets.as<int64_t>(), &total, st);
    if (r != CULSH_OK) return r;
    if (n_candidates_out) *n_candidates_out = total;
    CULSH_REQUIRE(total < (1LL << 31), "candidate list exceeds 2^31 entries");
    CULSH_CHECK(cand.alloc(sizeof(int32_t) * total));
    CULSH_CHECK(cand_sorted.alloc(sizeof(int32_t) * total));
    const int gridc = (int)min64((n_cols + 127) / 128, (int64_t)num_sms() * 8);
    if (total > 0) {
        cand_fill_kernel<<<gridc, 128, 0, st>>>(scols.as<int32_t>(), rs.as<int32_t>(), re.as<int32_t>(), q,
                                                N_total, j_base, n_cols, offsets.as<int64_t>(), cand.as<int32_t>());
        CULSH_LAUNCH_CHECK();
        r = sort_segments(cand.as<int32_t>(), cand_sorted.as<int32_t>(), total, n_cols, offsets.as<int64_t>(), st);
        if (r != CULSH_OK) return r;
    }
    if (K > 0) {
        select_kernel<<<gridc, 128, 0, st>>>(cand_sorted.as<int32_t>(), offsets.as<int64_t>(), j_base, n_cols, K,
                                             seed, N_total, entries);
        CULSH_LAUNCH_CHECK();
    }
    return CULSH_OK;
}
