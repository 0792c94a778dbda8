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
