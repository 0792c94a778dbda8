// exchange.cu -- the per-layer row exchange of the row-partitioned trainer
// done over NVLink peer memory instead of a separate
// all-gather: the GEMM (and softmax) epilogues store each owned output row into
// every peer's gathered buffer (CUDA IPC mappings, plain st.global over NVLink),
// then signal the peers; a peer waits on a device-side counter before it
// gathers remote rows.  Helpers here: allocation / IPC plumbing and the
// signal / wait kernels.  All device-side state (counters) is monotonic, so the
// sequence is safe inside a replayed CUDA graph.
#include <cstring>

#include "gdx_common.cuh"

namespace gdx {
namespace {

// Release our stores to the peers, then bump our slot in each peer's arrival array.
__global__ void peer_signal_kernel(unsigned long long* const* peer_slots, uint32_t npeers) {
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (uint32_t r = 0; r < npeers; ++r) atomicAdd_system(peer_slots[r], 1ull);
    }
}

struct PushPeers {
    uint32_t n;
    int64_t delta[7];
};

// SM push of a contiguous block to the same offset in every peer buffer (NVLink
// stores, 16 B per lane, 4 vectors in flight), fused with the arrival signal: the
// last CTA to finish (device-scope counter) releases all CTAs' stores system-wide
// and bumps our slot in every peer's arrival array, then re-arms the counter.
__global__ void __launch_bounds__(512) push_peers_kernel(const uint4* __restrict__ src, uint64_t n16,
                                                         PushPeers pp,
                                                         unsigned long long* const* peer_slots,
                                                         unsigned int* done) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(src + i + u * stride);
        for (uint32_t r = 0; r < pp.n; ++r) {
            uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<char*>(const_cast<uint4*>(src)) + pp.delta[r]);
#pragma unroll
            for (int u = 0; u < 4; ++u) d[i + u * stride] = v[u];
        }
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldg(src + i);
        for (uint32_t r = 0; r < pp.n; ++r)
            reinterpret_cast<uint4*>(reinterpret_cast<char*>(const_cast<uint4*>(src)) + pp.delta[r])[i] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (uint32_t r = 0; r < pp.n; ++r) atomicAdd_system(peer_slots[r], 1ull);
            *done = 0;
        }
    }
}

struct PushRows {
    uint32_t n;
    int64_t delta[7];
    uint64_t off[8];  // rows idx[off[r] .. off[r+1]) go to peer r
};

// Sparse push: only the rows each peer's CSR references (cooperative batches on
// low-degree subgraphs need about half of a block).  Row k of the list for peer r is
// copied to the same offset in peer r's buffer; 16-byte vectors, consecutive threads
// cover one row, so every row is one coalesced burst.  Fused signal as above.
__global__ void __launch_bounds__(512) push_rows_kernel(const char* __restrict__ base, uint32_t vpr,
                                                        uint64_t row_bytes, const uint32_t* __restrict__ idx,
                                                        PushRows pr, unsigned long long* const* peer_slots,
                                                        unsigned int* done) {
    // lane group of vpr lanes per row (rpw rows per warp), 4 rows in flight per group
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rpw = vpr >= 32 ? 1 : 32 / vpr;
    const uint32_t sub = vpr >= 32 ? 0 : lane / vpr;
    const uint32_t v0 = vpr >= 32 ? lane : lane - sub * vpr;
    const bool on = sub < rpw;
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * rpw;
    const uint64_t g0 = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * rpw + sub;
    // all peers at once (one GPU pair alone gets well under the NVLink ingress): item t
    // copies row t of every peer's list
    uint64_t tmax = 0;
    for (uint32_t r = 0; r < pr.n; ++r) tmax = max(tmax, pr.off[r + 1] - pr.off[r]);
    for (uint64_t t = g0; on && t < tmax; t += groups) {
        uint64_t o[7];
        bool ok[7];
#pragma unroll
        for (int r = 0; r < 7; ++r) {
            ok[r] = r < static_cast<int>(pr.n) && t < pr.off[r + 1] - pr.off[r];
            o[r] = ok[r] ? static_cast<uint64_t>(__ldg(idx + pr.off[r] + t)) * row_bytes : 0;
        }
        for (uint32_t v = v0; v < vpr; v += 32) {
#pragma unroll
            for (int r = 0; r < 7; ++r)
                if (ok[r])
                    *reinterpret_cast<uint4*>(const_cast<char*>(base) + o[r] + pr.delta[r] + 16 * v) =
                        __ldg(reinterpret_cast<const uint4*>(base + o[r] + 16 * v));
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (uint32_t r = 0; r < pr.n; ++r) atomicAdd_system(peer_slots[r], 1ull);
            *done = 0;
        }
    }
}

// NVSwitch multicast push: every 16-byte vector of the block is read once locally
// and stored ONCE to the multicast address (multimem.st); the switch replicates it
// into every GPU's copy of the buffer, so the sender's NVLink egress is the block
// size, not (world-1) x it.  Fused with the arrival signal like push_peers_kernel.
__global__ void __launch_bounds__(512) push_multicast_kernel(const uint4* __restrict__ src, uint64_t n16,
                                                             char* mc_dst, uint32_t npeers,
                                                             unsigned long long* const* peer_slots,
                                                             unsigned int* done) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + 16 * (i + u * stride)),
                         "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                         : "memory");
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldg(src + i);
        asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + 16 * i), "r"(v.x),
                     "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
    }
    asm volatile("fence.proxy.alias;" ::: "memory");
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (uint32_t r = 0; r < npeers; ++r) atomicAdd_system(peer_slots[r], 1ull);
            *done = 0;
        }
    }
}

// Round k of the exchange is complete when every other rank's slot reached k:
// *expected += 1, then spin (acquire, system scope) on each slot; traps after
// timeout_ns instead of hanging.
__global__ void peer_wait_kernel(unsigned long long* slots, unsigned long long* expected, uint32_t world,
                                 uint32_t self, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    const unsigned long long want = *expected + 1;
    *expected = want;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t r = 0; r < world; ++r) {
        if (r == self) continue;
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + r) : "memory");
            if (v >= want) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) __trap();
            __nanosleep(32);
        }
    }
    __threadfence_system();
}

// Per-source wait (pipelined exchange): the round number lives in *expected; with
// advance the round is started (*expected += 1) before waiting on slots[src].
__global__ void peer_wait_src_kernel(unsigned long long* slots, unsigned long long* expected, uint32_t src,
                                     int advance, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    unsigned long long want = *expected;
    if (advance) {
        want += 1;
        *expected = want;
    }
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + src) : "memory");
        if (v >= want) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) __trap();
        __nanosleep(64);
    }
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" int gdx_device_alloc(uint64_t bytes, void** out) {
    GDX_REQUIRE(out != nullptr, GDX_INPUT, "gdx_device_alloc: null out");
    GDX_CUDA(cudaMalloc(out, bytes ? bytes : 16));
    GDX_CUDA(cudaMemset(*out, 0, bytes ? bytes : 16));
    return GDX_OK;
}

extern "C" int gdx_device_free(void* p) {
    if (p) GDX_CUDA(cudaFree(p));
    return GDX_OK;
}

extern "C" int gdx_ipc_get_handle(const void* base, void* handle64) {
    GDX_REQUIRE(base && handle64, GDX_INPUT, "gdx_ipc_get_handle: null pointer");
    cudaIpcMemHandle_t h;
    GDX_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
    return GDX_OK;
}

extern "C" int gdx_ipc_open(const void* handle64, void** out) {
    GDX_REQUIRE(handle64 && out, GDX_INPUT, "gdx_ipc_open: null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    GDX_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return GDX_OK;
}

extern "C" int gdx_ipc_close(void* p) {
    if (p) GDX_CUDA(cudaIpcCloseMemHandle(p));
    return GDX_OK;
}

extern "C" int gdx_peer_wait_src(unsigned long long* slots, unsigned long long* expected, uint32_t src,
                                 int advance, uint64_t timeout_ns, gdx_stream stream) {
    GDX_REQUIRE(slots && expected, GDX_INPUT, "gdx_peer_wait_src: null pointer");
    peer_wait_src_kernel<<<1, 32, 0, as_cuda(stream)>>>(slots, expected, src, advance, timeout_ns);
    note_launch();
    return check_launch("gdx_peer_wait_src");
}

extern "C" int gdx_peer_signal(unsigned long long* const* peer_slots_dev, uint32_t npeers, gdx_stream stream) {
    GDX_REQUIRE(npeers == 0 || peer_slots_dev, GDX_INPUT, "gdx_peer_signal: null slots");
    if (!npeers) return GDX_OK;
    peer_signal_kernel<<<1, 32, 0, as_cuda(stream)>>>(peer_slots_dev, npeers);
    note_launch();
    return check_launch("gdx_peer_signal");
}

extern "C" int gdx_peer_wait(unsigned long long* slots, unsigned long long* expected, uint32_t world,
                             uint32_t self, uint64_t timeout_ns, gdx_stream stream) {
    GDX_REQUIRE(slots && expected, GDX_INPUT, "gdx_peer_wait: null pointer");
    GDX_REQUIRE(self < world, GDX_INPUT, "gdx_peer_wait: self >= world");
    if (world <= 1) return GDX_OK;
    peer_wait_kernel<<<1, 32, 0, as_cuda(stream)>>>(slots, expected, world, self, timeout_ns);
    note_launch();
    return check_launch("gdx_peer_wait");
}

// Copy-engine push of a contiguous block to a peer's IPC-mapped buffer (NVLink).
extern "C" int gdx_memcpy_async(void* dst, const void* src, uint64_t bytes, gdx_stream stream) {
    GDX_REQUIRE((dst && src) || bytes == 0, GDX_INPUT, "gdx_memcpy_async: null pointer");
    if (!bytes) return GDX_OK;
    GDX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_cuda(stream)));
    return GDX_OK;
}

extern "C" int gdx_memset2d_async(void* dst, uint64_t pitch_bytes, int value, uint64_t width_bytes, uint64_t rows,
                                  gdx_stream stream) {
    GDX_REQUIRE(dst || rows == 0 || width_bytes == 0, GDX_INPUT, "gdx_memset2d_async: null pointer");
    GDX_REQUIRE(rows <= 1 || pitch_bytes >= width_bytes, GDX_INPUT, "gdx_memset2d_async: pitch < width");
    if (!rows || !width_bytes) return GDX_OK;
    if (rows == 1 || pitch_bytes == width_bytes)
        GDX_CUDA(cudaMemsetAsync(dst, value, width_bytes * rows, as_cuda(stream)));
    else
        GDX_CUDA(cudaMemset2DAsync(dst, pitch_bytes, value, width_bytes, rows, as_cuda(stream)));
    return GDX_OK;
}

// SM-driven push + signal (see push_peers_kernel); `done` is a zeroed device counter.
extern "C" int gdx_push_peers(const void* src, uint64_t bytes, const int64_t* peer_delta, uint32_t npeers,
                              unsigned long long* const* peer_slots_dev, unsigned int* done, uint32_t ctas,
                              gdx_stream stream) {
    GDX_REQUIRE(npeers <= 7, GDX_INPUT, "gdx_push_peers: at most 7 peers");
    GDX_REQUIRE(npeers == 0 || (peer_slots_dev && done && peer_delta), GDX_INPUT, "gdx_push_peers: null pointer");
    GDX_REQUIRE(bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0, GDX_INPUT,
                "gdx_push_peers: 16-byte aligned whole vectors only");
    if (!npeers) return GDX_OK;
    PushPeers pp{npeers, {}};
    for (uint32_t r = 0; r < npeers; ++r) {
        GDX_REQUIRE(peer_delta[r] % 16 == 0, GDX_INPUT, "gdx_push_peers: peer offsets must be 16-byte aligned");
        pp.delta[r] = peer_delta[r];
    }
    push_peers_kernel<<<ctas ? ctas : 1, 512, 0, as_cuda(stream)>>>(
        reinterpret_cast<const uint4*>(src), bytes / 16, pp, peer_slots_dev, done);
    note_launch();
    return check_launch("gdx_push_peers");
}

// Multicast push + signal (see push_multicast_kernel).  mc_dst: the block's address in
// the buffer's multicast mapping (same offset as src in the local mapping).
extern "C" int gdx_push_multicast(const void* src, uint64_t bytes, void* mc_dst, uint32_t npeers,
                                  unsigned long long* const* peer_slots_dev, unsigned int* done,
                                  uint32_t ctas, gdx_stream stream) {
    GDX_REQUIRE(src && mc_dst && done && (npeers == 0 || peer_slots_dev), GDX_INPUT,
                "gdx_push_multicast: null pointer");
    GDX_REQUIRE(bytes % 16 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(mc_dst)) & 15) == 0,
                GDX_INPUT, "gdx_push_multicast: 16-byte aligned whole vectors only");
    push_multicast_kernel<<<ctas ? ctas : 1, 512, 0, as_cuda(stream)>>>(
        reinterpret_cast<const uint4*>(src), bytes / 16, static_cast<char*>(mc_dst), npeers, peer_slots_dev, done);
    note_launch();
    return check_launch("gdx_push_multicast");
}

// Sparse push + signal (see push_rows_kernel).  base: this rank's block; idx: row
// indices within it, concatenated per peer with offsets off[0..npeers].
extern "C" int gdx_push_rows(const void* base, uint64_t row_bytes, const uint32_t* idx, const uint64_t* off,
                             const int64_t* peer_delta, uint32_t npeers, unsigned long long* const* peer_slots_dev,
                             unsigned int* done, uint32_t ctas, gdx_stream stream) {
    GDX_REQUIRE(npeers <= 7, GDX_INPUT, "gdx_push_rows: at most 7 peers");
    GDX_REQUIRE(npeers == 0 || (base && off && peer_delta && peer_slots_dev && done), GDX_INPUT,
                "gdx_push_rows: null pointer");
    GDX_REQUIRE(row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0, GDX_INPUT,
                "gdx_push_rows: rows must be whole 16-byte vectors");
    if (!npeers) return GDX_OK;
    PushRows pr{npeers, {}, {}};
    for (uint32_t r = 0; r < npeers; ++r) {
        GDX_REQUIRE(peer_delta[r] % 16 == 0, GDX_INPUT, "gdx_push_rows: peer offsets must be 16-byte aligned");
        pr.delta[r] = peer_delta[r];
    }
    for (uint32_t r = 0; r <= npeers; ++r) pr.off[r] = off[r];
    GDX_REQUIRE(pr.off[npeers] == 0 || idx, GDX_INPUT, "gdx_push_rows: null index list");
    push_rows_kernel<<<ctas ? ctas : 1, 512, 0, as_cuda(stream)>>>(
        static_cast<const char*>(base), static_cast<uint32_t>(row_bytes / 16), row_bytes, idx, pr,
        peer_slots_dev, done);
    note_launch();
    return check_launch("gdx_push_rows");
}
