// TMEM load-shape probe (diagnostic, not part of the engine): stores lane*1000+col into
// TMEM with the known 32x32b shape, reads it back with tcgen05.ld.16x256b / 16x128b /
// 16x64b and records which (lane, col) every (thread, register) received.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t slot;
    const int t = threadIdx.x;
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    if (t < 32) {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = t * 1000 + j;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        uint32_t a[4];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(tm));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int r = 0; r < 4; ++r) out[t * 4 + r] = a[r];
        uint32_t b[2];
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(tm));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int r = 0; r < 2; ++r) out[128 + t * 2 + r] = b[r];
        uint32_t c;
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(c) : "r"(tm));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        out[192 + t] = c;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 256 * 4);
    cudaMemset(d, 0xff, 256 * 4);
    probe<<<1, 128>>>(d);
    uint32_t h[256];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    printf("16x256b (thread: lane.col per reg)\n");
    for (int t = 0; t < 32; ++t) {
        printf("t%02d:", t);
        for (int r = 0; r < 4; ++r) printf(" %u.%u", h[t * 4 + r] / 1000, h[t * 4 + r] % 1000);
        printf("\n");
    }
    printf("16x128b\n");
    for (int t = 0; t < 32; ++t) printf("t%02d: %u.%u %u.%u\n", t, h[128 + 2 * t] / 1000, h[128 + 2 * t] % 1000,
                                        h[129 + 2 * t] / 1000, h[129 + 2 * t] % 1000);
    printf("16x64b\n");
    for (int t = 0; t < 32; ++t) printf("t%02d: %u.%u\n", t, h[192 + t] / 1000, h[192 + t] % 1000);
    return 0;
}
