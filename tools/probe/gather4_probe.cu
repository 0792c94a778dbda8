// Probe of the TMA gather4 mode (cp.async.bulk.tensor.2d ... tile::gather4) on sm_100a:
// which tensor-map box height it wants, whether a 512-byte-aligned destination keeps
// the 128B swizzle, and what an out-of-range row index loads. Prints PASS/FAIL lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/gather4_probe tools/probe/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, const int32_t* idx, int nrows, uint16_t* out,
                      int dst_off) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sbar = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    uint8_t* dst0 = smem + dst_off;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) smem[i] = 0xAB;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(nrows * 128)
                     : "memory");
        for (int g = 0; g < nrows / 4; ++g) {
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst0 + g * 512));
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(idx[4 * g]), "r"(idx[4 * g + 1]),
                "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3]), "r"(sbar)
                : "memory");
        }
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sbar)
            : "memory");
    }
    __syncthreads();
    // un-swizzle: logical row r (128 B = 64 u16), 16-byte chunk c sits at chunk c ^ (addr bits [9:7])
    for (int i = threadIdx.x; i < nrows * 64; i += blockDim.x) {
        const int r = i / 64, e = i % 64, c = e / 8;
        const uintptr_t rowaddr = reinterpret_cast<uintptr_t>(dst0) + r * 128;
        const uint32_t sw = static_cast<uint32_t>((__cvta_generic_to_shared(reinterpret_cast<void*>(rowaddr)) >> 7) & 7);
        out[i] = reinterpret_cast<const uint16_t*>(dst0 + r * 128 + ((c ^ sw) * 16))[e % 8];
    }
}

int main() {
    const int R = 1000, C = 64, NR = 16;
    std::vector<uint16_t> h(R * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = static_cast<uint16_t>(r * 64 + c + 1);
    uint16_t* dsrc;
    cudaMalloc(&dsrc, h.size() * 2);
    cudaMemcpy(dsrc, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    std::vector<int32_t> idx = {5, 999, 0, 17, 400, 3, 3, 250, 998, 1, 2, 777, -1, 1000, 123, 66};
    int32_t* didx;
    cudaMallocManaged(&didx, NR * 4);
    for (int i = 0; i < NR; ++i) didx[i] = idx[i];
    uint16_t* dout;
    cudaMalloc(&dout, NR * C * 2);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    int fails = 0;
    for (uint32_t boxh : {1u, 4u}) {
        CUtensorMap map;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(R)};
        cuuint64_t strides[1] = {C * 2};
        cuuint32_t box[2] = {64, boxh};
        cuuint32_t es[2] = {1, 1};
        CUresult rc = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsrc, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) {
            printf("box height %u: encode failed %d\n", boxh, static_cast<int>(rc));
            continue;
        }
        for (int off : {0, 512}) {
            cudaMemset(dout, 0, NR * C * 2);
            probe<<<1, 128, 16384 + 2048>>>(map, didx, NR, dout, off);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("box height %u dst offset %d: launch error %s\n", boxh, off, cudaGetErrorString(e));
                return 1;
            }
            std::vector<uint16_t> o(NR * C);
            cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
            int bad = 0, zero_oob = 1;
            for (int i = 0; i < NR; ++i)
                for (int c = 0; c < C; ++c) {
                    const bool oob = idx[i] < 0 || idx[i] >= R;
                    const uint16_t want = oob ? 0 : h[idx[i] * C + c];
                    if (o[i * C + c] != want) {
                        if (oob) zero_oob = 0;
                        else ++bad;
                    }
                }
            printf("box height %u dst offset %d: %s (%d wrong in-range elements; out-of-range rows %s)\n", boxh, off,
                   bad == 0 ? "PASS" : "FAIL", bad, zero_oob ? "zero-filled" : "NOT zero");
            fails += bad != 0;
        }
    }
    return 0;
}
