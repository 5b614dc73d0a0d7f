// GSM count route, step 2 (reference similarity.py:57-90, 164-185):
// the four co-rating statistic products of the dense int8 column panels
//
//     g_xx += X X',  g_rx += R X',  g_rr += R R',  g_qx += Q X'      (ld x ld, int32)
//
// as ONE hand-written sm_100a tensor-core kernel (tcgen05.mma kind::i8, exact int32
// accumulation in TMEM), replacing four separate library GEMMs.  X / R / Q are rows of
// one (3, ld, w) int8 array (row j of a panel = column j of the ratings over w rating
// rows, i.e. K-major), so the fused kernel loads each operand tile once for all the
// products that use it:
//
//   per 128 x 128 output tile (a, b) and per 64-byte K block:
//     smem  Xa Ra Qa (A, 128 rows each) | Xb Rb (B, contiguous = one 256-row operand)
//     TMEM  cols   0..127  D_xx += Xa . Xb'         (N = 128)
//           cols 128..383  D_rx|D_rr += Ra . [Xb;Rb]'   (N = 256, one instruction)
//           cols 384..511  D_qx += Qa . Xb'         (N = 128)
//
// 4 products share 5 tile loads (a plain GEMM pays 2 per product).
//
// Panel layout in HBM ("tiled"): the panels are stored as tile groups, one per (128-row
// block rb, 64-byte K block kb), kb-major: group = [X | R | Q], 3 x 8 KB, each 8 KB tile
// already in the tcgen05 K-major SWIZZLE_64B layout (row r at r*64 bytes, 16-byte chunk c
// at chunk c ^ ((r >> 1) & 3)).  A stage is then TWO contiguous bulk copies (24 KB of
// A = [Xa|Ra|Qa], 16 KB of B = [Xb|Rb]) instead of five 2D tensor boxes of 64-byte rows:
// measured with the boxes, the copy engine delivered only ~24 B/clk per SM (tensor pipe
// 30 % busy, L2 and DRAM far from saturated).  The densify kernel writes this layout
// directly (culsh_gsm_densify_tiled); culsh_gsm_tile_panels converts a plain (3, ld, w)
// array.
//
// Warp-specialised, persistent (one CTA per SM): warp 0 = bulk-copy producer (5-stage
// mbarrier ring), warp 1 = TMEM owner + single-thread MMA issuer
// (tcgen05.commit frees a stage / publishes the accumulator), warps 2..5 = epilogue
// (tcgen05.ld 32x32b -> int32 stores, += when accumulating over row passes).  Every
// product entry is an exact integer (|sum| <= 121 * rows < 2^31), so the statistics --
// and the fp64 similarities the select kernel derives from them -- are bit-identical to
// the reference's ordered fp64 sums.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace culsh {
namespace gsm_tc {

constexpr int kBM = 128;                     // output tile rows (a) = MMA M
constexpr int kBN = 128;                     // output tile cols (b)
constexpr int kBK = 64;                      // K bytes per stage (64-byte swizzle rows)
constexpr int kStages = 5;
constexpr int kTile = kBM * kBK;             // 8 KB per 128-row operand tile
constexpr int kStageBytes = 5 * kTile;       // Xa Ra Qa Xb Rb = 40 KB
constexpr int kThreads = 192;                // 6 warps
constexpr int kTmemCols = 512;
constexpr int kGroupA = 8;                   // tile raster: 8 a-blocks per band (L2 reuse)
constexpr int kSyncEvery = 512;              // producer checkpoint every 512 K blocks ...
constexpr int kSyncLag = 4;                  // ... at most 4 checkpoints ahead of the slowest CTA
                                             // (CULSH_GSM_SYNC="every,lag" overrides; 0 = off)

// Byte offset of panel p (0 = X, 1 = R, 2 = Q), column j, K position k in the tiled layout.
// Groups are K-block-major (group = kb * nrb + rb): the blocks the co-resident tiles read at
// one K step are contiguous (rb-major placed them nkb * 24 KB apart -- a 2^17-multiple
// stride at C3 -- and C3 runs varied 0.37-1.37 s with the panel's base address).
__host__ __device__ __forceinline__ int64_t tiled_off(int p, int64_t j, int64_t k, int64_t nrb) {
    const int64_t r = j & 127, kk = k & 63;
    const int64_t grp = (k >> 6) * nrb + (j >> 7);
    const int64_t chunk = (kk >> 4) ^ ((r >> 1) & 3);
    return (grp * 3 + p) * (int64_t)kTile + r * 64 + chunk * 16 + (kk & 15);
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// K-major operand in shared memory, 64-byte swizzle: 8-row atoms of 512 bytes, stride
// byte offset 512, descriptor version 1 (sm_100), layout type 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);          // start address
    d |= (uint64_t)1 << 16;                          // leading byte offset (unused, swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;                 // stride byte offset
    d |= (uint64_t)1 << 46;                          // version
    d |= (uint64_t)4 << 61;                          // SWIZZLE_64B
    return d;
}

// kind::i8 instruction descriptor: s32 accumulator, signed A/B, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tile_of(int64_t t, int nA, int nB, int &a, int &b) {
    const int64_t band = (int64_t)kGroupA * nB;
    const int first = (int)(t / band) * kGroupA;
    const int gsz = min(nA - first, kGroupA);
    const int64_t r = t % band;
    a = first + (int)(r % gsz);
    b = (int)(r / gsz);
}

// Drift control.  The concurrently running CTAs share operand tiles through L2 only while
// they stream the same K blocks: the band of 148 tiles reads ~0.5 MB per K block, but L2
// turns over in ~20 us under the panel stream, so CTAs that drift more than ~20 K blocks
// apart re-read their tiles from DRAM (measured: 3.6 TB of DRAM reads at C2 for 3.8 TB of
// tile loads, DRAM-bound).  Every kSyncEvery K blocks the producer publishes its
// checkpoint in prog[cta] and waits until the slowest CTA is at most kSyncLag checkpoints
// behind; a CTA out of tiles publishes INT_MAX.  The grid is one CTA per SM, so all CTAs
// are normally co-resident; if a wait ever exceeds 5 ms (CTAs not co-resident, e.g. SMs
// taken by another context), the CTA stops synchronising instead of deadlocking -- the
// products are unaffected either way, only the L2 reuse.
__device__ __forceinline__ bool drift_wait(int *prog, int ncta, int cp, int lane, int lag) {
    // relaxed (volatile) accesses: no data is handed over, only progress, and an acquire
    // load would invalidate the SM's L1 (CCTL.IVALL) on every poll
    if (lane == 0) *(volatile int *)(prog + blockIdx.x) = cp;
    const uint64_t t0 = global_ns();
    for (;;) {
        int lo = INT_MAX;
        for (int c = lane; c < ncta; c += 32) lo = min(lo, ld_volatile(prog + c));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        if (lo >= cp - lag) return true;
        if (global_ns() - t0 > 5000000ull) return false;
        __nanosleep(200);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
gsm_stats_tc_kernel(const int8_t *__restrict__ tiles, int64_t ld, int nk, int accumulate,
                    int32_t *__restrict__ g_xx, int32_t *__restrict__ g_rx, int32_t *__restrict__ g_rr,
                    int32_t *__restrict__ g_qx, int32_t *__restrict__ g_xr, int32_t *__restrict__ g_xq,
                    int *__restrict__ prog, int sync_every, int sync_lag) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    uint64_t *tmem_full = empty + kStages;
    uint64_t *tmem_empty = tmem_full + 1;
    uint32_t *tmem_slot = (uint32_t *)(tmem_empty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nA = (int)(ld / kBM), nB = (int)(ld / kBN);
    const int64_t ntiles = (int64_t)nA * nB;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (lane 0; the warp joins the drift checkpoints) ----------------
        int stage = 0;
        uint32_t phase = 0;
        int cp = 0;
        bool sync = sync_every > 0;
        int64_t step = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int a, b;
            tile_of(t, nA, nB, a, b);
            for (int kb = 0; kb < nk; ++kb, ++step) {
                if (sync && step % sync_every == 0) {
                    __syncwarp();
                    sync = drift_wait(prog, gridDim.x, ++cp, lane, sync_lag);
                    sync = __shfl_sync(0xffffffffu, sync, 0);
                    if (!sync && lane == 0) {
                        *(volatile int *)(prog + blockIdx.x) = INT_MAX;   // stop holding others
                        atomicAdd(prog + gridDim.x, 1);                   // timeouts (CULSH_GSM_DEBUG)
                    }
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char *st = smem + stage * kStageBytes;
                    mbar_expect_tx(&full[stage], kStageBytes);
                    const int64_t kbase = (int64_t)kb * nA;   // K-block-major groups
                    bulk_load(smem_u32(st), tiles + (kbase + a) * (3 * kTile), 3 * kTile, &full[stage]);
                    bulk_load(smem_u32(st + 3 * kTile), tiles + (kbase + b) * (3 * kTile), 2 * kTile, &full[stage]);
                }
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        __syncwarp();
        if (lane == 0) *(volatile int *)(prog + blockIdx.x) = INT_MAX;
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread) ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            constexpr uint32_t id128 = idesc_i8(128), id256 = idesc_i8(256);
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(tmem_empty, acc_phase ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t base = smem_u32(smem + stage * kStageBytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk) {
                        const uint32_t off = kk * 32;
                        const uint64_t dXa = smem_desc(base + 0 * kTile + off);
                        const uint64_t dRa = smem_desc(base + 1 * kTile + off);
                        const uint64_t dQa = smem_desc(base + 2 * kTile + off);
                        const uint64_t dXb = smem_desc(base + 3 * kTile + off);   // [Xb; Rb] for N = 256
                        const uint32_t acc = (kb | kk) ? 1u : 0u;
                        mma_i8(tmem + 0, dXa, dXb, id128, acc);
                        mma_i8(tmem + 128, dRa, dXb, id256, acc);
                        mma_i8(tmem + 384, dQa, dXb, id128, acc);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(tmem_full);
                acc_phase ^= 1;
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> global ----------------
        const int quarter = warp & 3;            // TMEM lanes this warp may access
        const int row_in_tile = quarter * 32 + lane;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int a, b;
            tile_of(t, nA, nB, a, b);
            mbar_wait(tmem_full, acc_phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t row = (int64_t)a * kBM + row_in_tile;
            const int64_t col0 = (int64_t)b * kBN;
#pragma unroll 1
            for (int c = 0; c < kTmemCols; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c, v);
                int32_t *g = c < 128 ? g_xx : c < 256 ? g_rx : c < 384 ? g_rr : g_qx;
                int4 *dst = reinterpret_cast<int4 *>(g + row * ld + col0 + (c & 127));
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    int4 o = make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2], (int)v[4 * q + 3]);
                    if (accumulate) {
                        const int4 p = dst[q];
                        o.x += p.x;
                        o.y += p.y;
                        o.z += p.z;
                        o.w += p.w;
                    }
                    dst[q] = o;
                }
                // transposed copies of R X' and Q X' (g_xr = X R', g_xq = X Q': the s2 / q2
                // statistics read row-wise by the select kernel): for a fixed column the
                // warp's 32 rows are consecutive, so each of these stores is one 128-byte line
                int32_t *gt = (c >= 128 && c < 256) ? g_xr : (c >= 384 ? g_xq : nullptr);
                if (gt) {
#pragma unroll 8
                    for (int q = 0; q < 32; ++q) {
                        int32_t *p = gt + (col0 + (c & 127) + q) * ld + row;
                        *p = accumulate ? *p + (int)v[q] : (int)v[q];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(tmem_empty);
            acc_phase ^= 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols)
                     : "memory");
}

constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 + 256;

// Dense int8 panels for the count route in the tiled layout: 1 / r / r*r at (j, i - row_lo)
// for every rating (i, j) with row_lo <= i < row_hi (zeros elsewhere, memset by the caller).
// *status |= 1 when a value is not an integer in [-11, 11].
__global__ void densify_tiled_kernel(const int64_t *__restrict__ col_ptr, const int32_t *__restrict__ col_rows,
                                     const double *__restrict__ col_vals, int64_t N, int64_t row_lo,
                                     int64_t row_hi, int64_t nrb, int8_t *__restrict__ tiles,
                                     int *__restrict__ status) {
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
            const int64_t k = i - row_lo;
            tiles[tiled_off(0, j, k, nrb)] = 1;
            tiles[tiled_off(1, j, k, nrb)] = (int8_t)iv;
            tiles[tiled_off(2, j, k, nrb)] = (int8_t)(iv * iv);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1);
    }
}

// plain (3, ld, w) -> tiled, one thread per 16-byte chunk.
__global__ void tile_panels_kernel(const int8_t *__restrict__ plain, int64_t ld, int64_t w,
                                   int8_t *__restrict__ tiles) {
    const int64_t nchunk = 3 * ld * (w / 16), nrb = ld / kBM;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunk;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = c / (w / 16), k = (c % (w / 16)) * 16;
        const int p = (int)(row / ld);
        const int64_t j = row % ld;
        *reinterpret_cast<int4 *>(tiles + tiled_off(p, j, k, nrb)) =
            *reinterpret_cast<const int4 *>(plain + row * w + k);
    }
}

}  // namespace gsm_tc
}  // namespace culsh

using namespace culsh;

extern "C" int culsh_gsm_densify_tiled(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                                       int64_t N, int64_t row_lo, int64_t row_hi, int64_t ld, int64_t w,
                                       int8_t *tiles, int *status, void *stream) {
    using namespace culsh::gsm_tc;
    CULSH_REQUIRE(ld >= N && ld % kBM == 0 && w % kBK == 0 && row_hi - row_lo <= w,
                  "tiled panels need ld >= N, ld % 128 == 0, w % 64 == 0, row range <= w");
    if (N <= 0) return CULSH_OK;
    const int64_t blocks = min64((N + 7) / 8, (int64_t)num_sms() * 16);
    densify_tiled_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(col_ptr, col_rows, col_vals, N, row_lo,
                                                                              row_hi, ld / kBM, tiles, status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_gsm_tile_panels(const int8_t *plain, int64_t ld, int64_t w, int8_t *tiles, void *stream) {
    using namespace culsh::gsm_tc;
    CULSH_REQUIRE(ld > 0 && ld % kBM == 0 && w > 0 && w % kBK == 0, "ld % 128 == 0 and w % 64 == 0");
    CULSH_REQUIRE((reinterpret_cast<uintptr_t>(plain) & 15) == 0 && (reinterpret_cast<uintptr_t>(tiles) & 15) == 0,
                  "16-byte aligned arrays");
    const int64_t blocks = min64((3 * ld * (w / 16) + 255) / 256, (int64_t)num_sms() * 32);
    tile_panels_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(plain, ld, w, tiles);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

extern "C" int culsh_gsm_stats_tc(const int8_t *tiles, int64_t ld, int64_t w, int accumulate, int32_t *g_xx,
                                  int32_t *g_rx, int32_t *g_rr, int32_t *g_qx, int32_t *g_xr, int32_t *g_xq,
                                  void *stream) {
    using namespace culsh::gsm_tc;
    CULSH_REQUIRE(ld > 0 && ld % kBM == 0, "ld must be a positive multiple of 128");
    CULSH_REQUIRE(w > 0 && w % kBK == 0, "w must be a positive multiple of 64");
    CULSH_REQUIRE(w / kBK < (1ll << 31), "panel too long");
    CULSH_REQUIRE((reinterpret_cast<uintptr_t>(tiles) & 15) == 0, "tiles must be 16-byte aligned");
    CULSH_CHECK(cudaFuncSetAttribute(gsm_stats_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSmemBytes));
    const int64_t ntiles = (ld / kBM) * (ld / kBN);
    const int grid = (int)min64(ntiles, (int64_t)num_sms());
    cudaStream_t st = (cudaStream_t)stream;
    int *prog = nullptr;
    CULSH_CHECK(cudaMallocAsync((void **)&prog, sizeof(int) * (size_t)(grid + 1), st));
    CULSH_CHECK(cudaMemsetAsync(prog, 0, sizeof(int) * (size_t)(grid + 1), st));
    int every = kSyncEvery, lag = kSyncLag;
    if (const char *e = getenv("CULSH_GSM_SYNC")) sscanf(e, "%d,%d", &every, &lag);
    gsm_stats_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(tiles, ld, (int)(w / kBK), accumulate, g_xx, g_rx,
                                                            g_rr, g_qx, g_xr, g_xq, prog, every, lag);
    CULSH_LAUNCH_CHECK();
    if (getenv("CULSH_GSM_DEBUG")) {
        int timeouts = 0;
        CULSH_CHECK(cudaMemcpyAsync(&timeouts, prog + grid, sizeof(int), cudaMemcpyDeviceToHost, st));
        CULSH_CHECK(cudaStreamSynchronize(st));
        fprintf(stderr, "culsh_gsm_stats_tc: ld=%lld w=%lld grid=%d sync=%d,%d timeouts=%d\n", (long long)ld,
                (long long)w, grid, every, lag, timeouts);
    }
    CULSH_CHECK(cudaFreeAsync(prog, st));
    return CULSH_OK;
}
