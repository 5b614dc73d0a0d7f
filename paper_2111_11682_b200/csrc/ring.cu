// DSGD ring shift over peer memory (reference parallel.py:166-227 moves blocks
// between workers at the stage barrier): the block a rank trained is written by ITS OWN
// kernel straight into the next rank's receive buffer (NVLink P2P stores when the ranks are
// on different GPUs, CUDA IPC-mapped device memory), followed by a system-scope release flag;
// the next rank's pull kernel waits on that flag on the device, copies the block into its
// parameter arrays and acknowledges with a release flag back in the sender's memory.  No
// NCCL call, no host synchronisation between stages: stage kernel -> push -> pull -> next
// stage kernel are stream-ordered on every rank, and the only cross-GPU dependencies are the
// device-side flags.
//
// Buffer layout of every rank (one cudaMalloc, exported as one IPC handle):
//   [flags: 64 x u64 (ready[2] at 0..1, ack[2] at 8..9, counters at 16..17)]
//   [data parity 0 | data parity 1] (each `slot_bytes`)
// The sender of rank q writes q.data[seq & 1] and q.ready[seq & 1] = seq; rank q, after
// copying, writes sender.ack[seq & 1] = seq; the sender's next write into the same parity
// (seq + 2) first waits for ack >= seq.
#include <cstring>

#include "common.cuh"

namespace culsh {

constexpr int kRingFlagWords = 64;
constexpr int kRingMaxTensors = 8;
constexpr int kRingGrid = 32;

struct RingTensors {
    const char *src[kRingMaxTensors];   // push: block start in the local arrays; pull: unused
    char *dst[kRingMaxTensors];         // pull: block start in the local arrays; push: unused
    int64_t bytes[kRingMaxTensors];     // bytes of the block of each tensor (multiples of 4)
    int64_t off[kRingMaxTensors];       // offset of each tensor's block inside a data slot
    int n;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Thread 0 of every CTA waits for *flag >= want (20 s watchdog -> *status |= 4).
__device__ __forceinline__ bool wait_flag(const uint64_t *flag, uint64_t want, int *status) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        const uint64_t t0 = global_ns();
        int ok = 1;
        while (ld_acquire_sys(flag) < want) {
            if (global_ns() - t0 > 20000000000ull) {
                atomicOr(status, 4);
                ok = 0;
                break;
            }
            __nanosleep(500);
        }
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// Grid-wide "all CTAs done": the last CTA to arrive (after a system fence of its writes)
// publishes `value` to `flag` (release, system scope) and resets the counter.
__device__ __forceinline__ void publish_when_all_done(unsigned long long *counter, uint64_t *flag,
                                                      uint64_t value) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long prev = atomicAdd(counter, 1ull);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            *counter = 0ull;
            st_release_sys(flag, value);
        }
    }
}

__device__ __forceinline__ void copy_bytes(char *dst, const char *src, int64_t bytes) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)bytes) & 15) == 0) {
        const int4 *s = reinterpret_cast<const int4 *>(src);
        int4 *d = reinterpret_cast<int4 *>(dst);
        for (int64_t k = tid; k < bytes / 16; k += nth) d[k] = s[k];
    } else {
        const int *s = reinterpret_cast<const int *>(src);
        int *d = reinterpret_cast<int *>(dst);
        for (int64_t k = tid; k < bytes / 4; k += nth) d[k] = s[k];
    }
}

// Push the trained block into the receiver's slot (seq & 1) once the receiver acknowledged
// the previous use of that slot (seq - 2), then publish receiver.ready[seq & 1] = seq.
__global__ void ring_push_kernel(RingTensors t, char *peer_buf, int64_t slot_bytes, uint64_t seq,
                                 const uint64_t *my_ack, unsigned long long *my_counter, int *status) {
    const int par = (int)(seq & 1);
    if (seq > 2 && !wait_flag(my_ack + par, seq - 2, status)) return;
    char *slot = peer_buf + kRingFlagWords * 8 + par * slot_bytes;
    for (int k = 0; k < t.n; ++k) copy_bytes(slot + t.off[k], t.src[k], t.bytes[k]);
    publish_when_all_done(my_counter, reinterpret_cast<uint64_t *>(peer_buf) + par, seq);
}

// Wait for my.ready[seq & 1] >= seq, copy the slot into the local arrays, then publish
// sender.ack[seq & 1] = seq.
__global__ void ring_pull_kernel(RingTensors t, char *my_buf, int64_t slot_bytes, uint64_t seq,
                                 uint64_t *sender_buf, unsigned long long *my_counter, int *status) {
    const int par = (int)(seq & 1);
    if (!wait_flag(reinterpret_cast<const uint64_t *>(my_buf) + par, seq, status)) return;
    const char *slot = my_buf + kRingFlagWords * 8 + par * slot_bytes;
    for (int k = 0; k < t.n; ++k) copy_bytes(t.dst[k], slot + t.off[k], t.bytes[k]);
    publish_when_all_done(my_counter, sender_buf + 8 + par, seq);
}

}  // namespace culsh

using namespace culsh;

extern "C" int culsh_ring_alloc(int64_t slot_bytes, void **buf, void *ipc_handle_out) {
    CULSH_REQUIRE(slot_bytes >= 0 && (slot_bytes & 15) == 0, "slot_bytes must be a multiple of 16");
    const size_t total = (size_t)kRingFlagWords * 8 + 2 * (size_t)slot_bytes;
    CULSH_CHECK(cudaMalloc(buf, total));
    CULSH_CHECK(cudaMemset(*buf, 0, total));
    CULSH_CHECK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(ipc_handle_out), *buf));
    return CULSH_OK;
}

extern "C" int culsh_ring_open(const void *ipc_handle, void **buf) {
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    CULSH_CHECK(cudaIpcOpenMemHandle(buf, h, cudaIpcMemLazyEnablePeerAccess));
    return CULSH_OK;
}

extern "C" int culsh_ring_close(void *peer_buf) {
    CULSH_CHECK(cudaIpcCloseMemHandle(peer_buf));
    return CULSH_OK;
}

extern "C" int culsh_ring_free(void *buf) {
    CULSH_CHECK(cudaFree(buf));
    return CULSH_OK;
}

extern "C" int culsh_ring_handle_bytes() { return (int)sizeof(cudaIpcMemHandle_t); }

static int fill_tensors(RingTensors &t, int n, void *const *ptrs, const int64_t *bytes, const int64_t *offs,
                        bool push) {
    CULSH_REQUIRE(n >= 0 && n <= kRingMaxTensors, "at most 8 moving tensors");
    t.n = n;
    for (int k = 0; k < n; ++k) {
        CULSH_REQUIRE((bytes[k] & 3) == 0 && (offs[k] & 15) == 0, "4-byte blocks at 16-byte slot offsets");
        t.src[k] = push ? static_cast<const char *>(ptrs[k]) : nullptr;
        t.dst[k] = push ? nullptr : static_cast<char *>(ptrs[k]);
        t.bytes[k] = bytes[k];
        t.off[k] = offs[k];
    }
    return CULSH_OK;
}

// my_buf: this rank's ring buffer (its ack flags and counter live there); peer_buf: the
// receiver's buffer (IPC-mapped).  ptrs / bytes / offs: the n block pieces to send.
extern "C" int culsh_ring_push(int n, void *const *ptrs, const int64_t *bytes, const int64_t *offs, void *my_buf,
                               void *peer_buf, int64_t slot_bytes, uint64_t seq, int *status, void *stream) {
    RingTensors t;
    const int rc = fill_tensors(t, n, ptrs, bytes, offs, true);
    if (rc != CULSH_OK) return rc;
    uint64_t *mine = static_cast<uint64_t *>(my_buf);
    ring_push_kernel<<<kRingGrid, 256, 0, (cudaStream_t)stream>>>(
        t, static_cast<char *>(peer_buf), slot_bytes, seq, mine + 8,
        reinterpret_cast<unsigned long long *>(mine + 16), status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}

// sender_buf: the sending rank's buffer (IPC-mapped; its ack flags are written here).
extern "C" int culsh_ring_pull(int n, void *const *ptrs, const int64_t *bytes, const int64_t *offs, void *my_buf,
                               void *sender_buf, int64_t slot_bytes, uint64_t seq, int *status, void *stream) {
    RingTensors t;
    const int rc = fill_tensors(t, n, ptrs, bytes, offs, false);
    if (rc != CULSH_OK) return rc;
    uint64_t *mine = static_cast<uint64_t *>(my_buf);
    ring_pull_kernel<<<kRingGrid, 256, 0, (cudaStream_t)stream>>>(
        t, static_cast<char *>(my_buf), slot_bytes, seq, static_cast<uint64_t *>(sender_buf),
        reinterpret_cast<unsigned long long *>(mine + 17), status);
    CULSH_LAUNCH_CHECK();
    return CULSH_OK;
}
