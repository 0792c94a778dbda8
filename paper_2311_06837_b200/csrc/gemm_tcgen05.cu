// gemm_tcgen05.cu -- K2: the dense feature transform on 5th-gen tensor cores.
//
// Replaces apply_layer (reference_gnn.cpp:53-60) -- out = W * agg for every
// vertex -- by one GEMM over all rows,  C[m][n] = sum_k A(m,k) B(n,k),
// and serves the backward GEMMs of the training extension (dW = G^T H with
// split-K over vertices, dH = G W).  A and B are each K-major (A[m][k]) or
// MN-major (A stored [k][m]); the MN-major forms let dW = G^T H read G and H
// in place, with no transposes.
//
// Precision: the path must stay within 1e-4 (scaled) of an fp64 oracle, which
// TF32 or plain BF16 cannot.  Operands are stored "split bf16" (x = hi + lo,
// hi = bf16(x), lo = bf16(x - hi); |x - hi - lo| <= 2^-17 |x|) and each k-step
// issues three tcgen05.mma kind::f16 (hi*hi + hi*lo + lo*hi) into one fp32 TMEM
// accumulator: ~2^-16 relative per product, fp32 accumulation, at 1/3 of the
// bf16 tensor rate -- the GEMMs here are skinny (N <= 256) and HBM-bound anyway.
//
// Persistent structure: one CTA per SM loops over output tiles (128 x BN, and
// K ranges for split-K); 320 threads:
//   warp 0 / lane 0 : TMA producer   (cp.async.bulk.tensor, 128B swizzle, mbarrier tx)
//   warp 1 / lane 0 : MMA issuer     (tcgen05.mma, tcgen05.commit releases stages / accumulators)
//   warps 2-9       : epilogue       (tcgen05.ld 32x32b.x32 -> scale/ReLU -> vector stores);
//                     two warps per 32-lane TMEM quarter, each taking half the columns
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the TMA + MMA of tile i+1.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "gdx_common.cuh"

// the MT instantiation leaves the generic epilogue loop unreachable by design
#pragma nv_diag_suppress 128

namespace gdx {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
// Epilogue warps per CTA (template EW): 8 = two per 32-lane TMEM quarter, each half the
// columns, with a 20 KB store-transpose buffer; 16 = four per quarter, no buffer.
// Measured (tools/gemm_bench.py): 16 warps hide the fused dH epilogue's mask loads
// (Reddit 0.127 -> 0.092 ms, products 1.10 -> 0.90 ms) but lose on plain stores
// (products L2 forward 0.28 -> 0.32 ms), so EW = 16 is used when a mask is fused.
constexpr int kThreadsFor(int ew) { return 64 + 32 * ew; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c_inner, int32_t c_outer) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c_inner), "r"(c_outer), "r"(smem_u32(bar))
        : "memory");
}

// 128B-swizzled smem operand descriptor (tcgen05 "matrix descriptor"):
// start>>4 [0,14) | LBO>>4 [16,30) | SBO>>4 [32,46) | version 1 [46,48) | swizzle 2 [61,64)
//   K-major : rows of 64 k-elements (128 B), 8-row groups at SBO = 1024 B (LBO unused)
//   MN-major: 64 mn-elements contiguous, 8 k-rows per 1 KB atom (SBO = 1024 B between
//             k-groups), 64-wide mn blocks LBO apart
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}

// split-bf16 copy of 16 values at hp/lp: 8-byte vector stores when aligned
__device__ __forceinline__ void store_split16(const float* vv, uint16_t* hp, uint16_t* lp, uint32_t col0,
                                              uint32_t n) {
    if (col0 + 16 <= n && (reinterpret_cast<uintptr_t>(hp) & 7) == 0 && (reinterpret_cast<uintptr_t>(lp) & 7) == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
            ushort4 h, l;
            split_bf16(vv[j], h.x, l.x);
            split_bf16(vv[j + 1], h.y, l.y);
            split_bf16(vv[j + 2], h.z, l.z);
            split_bf16(vv[j + 3], h.w, l.w);
            *reinterpret_cast<ushort4*>(hp + j) = h;
            *reinterpret_cast<ushort4*>(lp + j) = l;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (col0 + j < n) split_bf16(vv[j], hp[j], lp[j]);
    }
}

struct Epi {
    uint32_t m, n;
    float* c0;
    uint64_t ldc0;
    float* c1;
    uint64_t ldc1;
    uint32_t split;
    const float* row_scale;
    int relu;
    uint16_t* out_hi;
    uint16_t* out_lo;
    uint64_t ld_split;
    uint32_t split_k;
    uint32_t kblocks;   // total k blocks
    uint32_t m_tiles, n_tiles;
    const float* mask;
    uint64_t ld_mask;
    int split_unscaled;
    uint32_t npeers;        // fused exchange: peer copies of output `peer_target`
    int peer_target;
    int64_t peer_delta[7];
    int stage_stores;       // row-contiguous (smem-transposed) fp32 stores
    int tma_store;          // ... leaving smem through TMA bulk tensor stores (map_c0 / map_c1)
    const uint32_t* a_rows; // row gather of a K-major A (m index) / an MN-major B (k index):
    const uint32_t* b_rows; // TMA gather4, 4 source rows per instruction
    uint32_t k;
    uint16_t* p24_hi;       // packed-24 form of output p24_target (its fp32 pointer is null)
    uint8_t* p24_lo;
    uint64_t ld_p24_hi, ld_p24_lo;
    int p24_target;
};

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c_inner,
                                            const uint4& rows) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c_inner), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w),
        "r"(smem_u32(bar))
        : "memory");
}

// four consecutive entries of a row index (out of range -> 0xFFFFFFFF: TMA zero-fills)
__device__ __forceinline__ uint4 gather_rows4(const uint32_t* idx, uint32_t r0, uint32_t count) {
    uint4 v;
    v.x = r0 < count ? __ldg(idx + r0) : 0xFFFFFFFFu;
    v.y = r0 + 1 < count ? __ldg(idx + r0 + 1) : 0xFFFFFFFFu;
    v.z = r0 + 2 < count ? __ldg(idx + r0 + 2) : 0xFFFFFFFFu;
    v.w = r0 + 3 < count ? __ldg(idx + r0 + 3) : 0xFFFFFFFFu;
    return v;
}

// Store transpose buffers, 4 KB per epilogue warp (32 KB at EW = 8):
//  * TMA stores: two 32 rows x 16 fp32 boxes (2 KB each, 64-byte rows in the SWIZZLE_64B
//    layout, so the row-per-thread float4 writes of a quarter-warp hit 8 distinct bank
//    groups); one elected lane issues cp.async.bulk.tensor per box and the warp moves on,
//    double-buffered on bulk_group completion;
//  * register stores (peer copies): one 32 x 16 box at row pitch 20 floats.
constexpr uint32_t kStgPitch = 20;
constexpr uint32_t kStgWarpFloats = 1024;
constexpr uint32_t kStgBytesFor(int ew) { return ew <= 8 ? ew * kStgWarpFloats * 4 : 0; }

__device__ __forceinline__ void tma_store_2d_nc(const CUtensorMap* map, const void* src, int32_t c_inner,
                                                int32_t c_outer) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c_inner), "r"(c_outer)
                 : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c_inner,
                                             int32_t c_outer) {
    tma_store_2d_nc(map, src, c_inner, c_outer);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Fused ReLU-backward (MT) variant, BN = 64 only: the producer warp also TMA-loads the
// tile's 128 x 64 fp32 mask (two 128B-swizzled 128 x 32 boxes, double-buffered with the
// accumulators), and every output -- the scaled fp32 c0 and the split hi/lo copy --
// leaves through TMA stores. Per epilogue warp and store buffer: fp32 box 2 KB
// (SWIZZLE_64B) + hi 1 KB + lo 1 KB (32 x 16 u16, SWIZZLE_32B), two buffers.
constexpr uint32_t kMaskTile = BM * 64 * 4;       // 32 KB
constexpr uint32_t kMtWarpBytes = 2 * 4096;       // per epilogue warp

// store one float4 locally and, for the exchanged output, into every peer buffer
__device__ __forceinline__ void store4x(float* p, const float4& v, const Epi& ep, bool xchg) {
    *reinterpret_cast<float4*>(p) = v;
    if (xchg)
        for (uint32_t r = 0; r < ep.npeers; ++r)
            *reinterpret_cast<float4*>(reinterpret_cast<char*>(p) + ep.peer_delta[r]) = v;
}
__device__ __forceinline__ void store1x(float* p, float v, const Epi& ep, bool xchg) {
    *p = v;
    if (xchg)
        for (uint32_t r = 0; r < ep.npeers; ++r) *reinterpret_cast<float*>(reinterpret_cast<char*>(p) + ep.peer_delta[r]) = v;
}

template <int BN, int STAGES, int EW, bool MT = false>
struct Smem {
    static constexpr uint32_t kA = BM * BK * 2;  // bytes per A operand tile (hi or lo)
    static constexpr uint32_t kB = BN * BK * 2;
    static constexpr uint32_t kStage = 2 * kA + 2 * kB;
    static constexpr uint32_t kStaging = MT ? EW * kMtWarpBytes : kStgBytesFor(EW);  // epilogue store transposes
    static constexpr uint32_t kMask = MT ? 2 * kMaskTile : 0;
    static constexpr uint32_t kBytes = STAGES * kStage + kStaging + kMask + 1024 /*align*/ + 512 /*barriers*/;
    static_assert(kBytes <= 232448, "227 KB shared memory per CTA");
};

// Load one operand tile (rows x BK of a K-major matrix, or BK x rows of an
// MN-major one) into smem as the canonical SW128 layout.
template <int ROWS, bool MN>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                             int32_t row0, int32_t k0) {
    if constexpr (!MN) {
        tma_load_2d(dst, map, bar, k0, row0);  // box {64 k, ROWS rows}
    } else {
#pragma unroll
        for (int b = 0; b < ROWS / 64; ++b)  // box {64 mn, BK k}, 8 KB each
            tma_load_2d(dst + b * (64 * BK * 2), map, bar, row0 + 64 * b, k0);
    }
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EW, bool MT>
__global__ void __launch_bounds__(kThreadsFor(EW), 1)
    gemm_bf16x3(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                const __grid_constant__ CUtensorMap map_c0, const __grid_constant__ CUtensorMap map_c1,
                const __grid_constant__ CUtensorMap map_mask, const __grid_constant__ CUtensorMap map_shi,
                const __grid_constant__ CUtensorMap map_slo, const __grid_constant__ CUtensorMap map_phi,
                const __grid_constant__ CUtensorMap map_plo, const Epi ep) {
    static_assert(!MT || (BN == 64 && EW == 8), "mask-TMA variant: BN 64, 8 epilogue warps");
    using S = Smem<BN, STAGES, EW, MT>;
    constexpr int kEpiWarps = EW;
    constexpr uint32_t kStgBytes = kStgBytesFor(EW);
    constexpr uint32_t kTmemCols = 2 * BN;  // two accumulators
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* epi_stage = reinterpret_cast<float*>(smem + STAGES * S::kStage);  // store transposes
    float* mask_s = reinterpret_cast<float*>(smem + STAGES * S::kStage + S::kStaging);  // MT: [2] tiles
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage + S::kStaging + S::kMask);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint64_t* mfull = tempty + 2;      // [2] mask tile landed (MT)
    uint64_t* mempty = mfull + 2;      // [2] mask tile consumed (MT)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t total = ep.m_tiles * ep.n_tiles * ep.split_k;
    const uint32_t per = (ep.kblocks + ep.split_k - 1) / ep.split_k;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
            mbar_init(&mfull[a], 1);
            mbar_init(&mempty[a], kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
        if (ep.tma_store) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c0)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c1)) : "memory");
        }
        if constexpr (MT) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_mask)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_shi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_slo)) : "memory");
        }
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    auto tile_coords = [&](uint32_t t, uint32_t& mt, uint32_t& nt, uint32_t& z) {
        z = t % ep.split_k;
        const uint32_t mn = t / ep.split_k;
        nt = mn % ep.n_tiles;
        mt = mn / ep.n_tiles;
    };

    const bool gather_a = !A_MN && ep.a_rows != nullptr;
    const bool gather_b = B_MN && ep.b_rows != nullptr;
    if (warp == 0 && (gather_a || gather_b)) {
        // ---------------- TMA producer, gathered operand(s): the whole warp ----------------
        // Lane l gathers A rows 4l..4l+3 of the tile (K-major A: 32 x gather4 = 128 rows)
        // and B k-rows 4(l & 15).. of 64-wide column block l >> 4 (MN-major B), so one
        // k block's gathers go out from 32 lanes at once. Lane 0 waits/arms the barrier.
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
            uint32_t mt, nt, z;
            tile_coords(t, mt, nt, z);
            const uint32_t kb0 = z * per, kb1 = min(ep.kblocks, kb0 + per);
            uint4 ia = make_uint4(0, 0, 0, 0);
            if (gather_a) ia = gather_rows4(ep.a_rows, mt * BM + 4 * lane, ep.m);
            for (uint32_t kb = kb0; kb < kb1; ++kb, ++it) {
                const int s = it % STAGES;
                uint8_t* st = smem + s * S::kStage;
                const int32_t kc = static_cast<int32_t>(kb * BK);
                uint4 ib = make_uint4(0, 0, 0, 0);
                if (gather_b) ib = gather_rows4(ep.b_rows, kb * BK + 4 * (lane & 15), ep.k);
                if (lane == 0) {
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    mbar_expect_tx(&full[s], S::kStage);
                }
                __syncwarp();
                if (gather_a) {
                    tma_gather4(st + lane * 512, &map_ahi, &full[s], kc, ia);
                    tma_gather4(st + S::kA + lane * 512, &map_alo, &full[s], kc, ia);
                } else if (lane == 0) {
                    load_operand<BM, A_MN>(st, &map_ahi, &full[s], static_cast<int32_t>(mt * BM), kc);
                    load_operand<BM, A_MN>(st + S::kA, &map_alo, &full[s], static_cast<int32_t>(mt * BM), kc);
                }
                if (gather_b) {
#pragma unroll
                    for (int blk = lane >> 4; blk < BN / 64; blk += 2) {
                        const uint32_t off = blk * (64 * BK * 2) + (lane & 15) * 512;
                        const int32_t nc = static_cast<int32_t>(nt * BN + 64 * blk);
                        tma_gather4(st + 2 * S::kA + off, &map_bhi, &full[s], nc, ib);
                        tma_gather4(st + 2 * S::kA + S::kB + off, &map_blo, &full[s], nc, ib);
                    }
                } else if (lane == 0) {
                    load_operand<BN, B_MN>(st + 2 * S::kA, &map_bhi, &full[s], static_cast<int32_t>(nt * BN), kc);
                    load_operand<BN, B_MN>(st + 2 * S::kA + S::kB, &map_blo, &full[s],
                                           static_cast<int32_t>(nt * BN), kc);
                }
                __syncwarp();
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            uint32_t it = 0, tl = 0;
            for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
                uint32_t mt, nt, z;
                tile_coords(t, mt, nt, z);
                const uint32_t kb0 = z * per, kb1 = min(ep.kblocks, kb0 + per);
                if constexpr (MT) {  // the tile's mask, ahead of its operands
                    const uint32_t mb = tl & 1;
                    mbar_wait(&mempty[mb], ((tl >> 1) & 1) ^ 1);
                    mbar_expect_tx(&mfull[mb], kMaskTile);
                    float* dst = mask_s + mb * (kMaskTile / 4);
                    tma_load_2d(dst, &map_mask, &mfull[mb], 0, static_cast<int32_t>(mt * BM));
                    tma_load_2d(dst + BM * 32, &map_mask, &mfull[mb], 32, static_cast<int32_t>(mt * BM));
                }
                for (uint32_t kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* st = smem + s * S::kStage;
                    mbar_expect_tx(&full[s], S::kStage);
                    const int32_t kc = static_cast<int32_t>(kb * BK);
                    load_operand<BM, A_MN>(st, &map_ahi, &full[s], static_cast<int32_t>(mt * BM), kc);
                    load_operand<BM, A_MN>(st + S::kA, &map_alo, &full[s], static_cast<int32_t>(mt * BM), kc);
                    load_operand<BN, B_MN>(st + 2 * S::kA, &map_bhi, &full[s], static_cast<int32_t>(nt * BN), kc);
                    load_operand<BN, B_MN>(st + 2 * S::kA + S::kB, &map_blo, &full[s],
                                           static_cast<int32_t>(nt * BN), kc);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            // kind::f16: D=f32 (bit 4), A=B=bf16 (bits 7, 10), majors (15, 16), N>>3 @17, M>>4 @24
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                                       ((B_MN ? 1u : 0u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                       (static_cast<uint32_t>(BM >> 4) << 24);
            // per 16-wide k step: +32 B inside the swizzle row (K-major) or +16 rows (MN-major)
            constexpr uint32_t a_step = A_MN ? 16 * 128 : 32, b_step = B_MN ? 16 * 128 : 32;
            constexpr uint32_t a_lbo = A_MN ? 64 * BK * 2 : 16, b_lbo = B_MN ? 64 * BK * 2 : 16;
            uint32_t it = 0, tl = 0;
            for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
                uint32_t mt, nt, z;
                tile_coords(t, mt, nt, z);
                const uint32_t kb0 = z * per, kb1 = min(ep.kblocks, kb0 + per);
                const uint32_t acc = tl & 1;
                mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d_tmem = tmem + acc * BN;
                for (uint32_t kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t st = smem_u32(smem + s * S::kStage);
                    const uint32_t ahi = st, alo = st + S::kA, bhi = st + 2 * S::kA, blo = st + 2 * S::kA + S::kB;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t dah = smem_desc_sw128(ahi + kk * a_step, a_lbo);
                        const uint64_t dal = smem_desc_sw128(alo + kk * a_step, a_lbo);
                        const uint64_t dbh = smem_desc_sw128(bhi + kk * b_step, b_lbo);
                        const uint64_t dbl = smem_desc_sw128(blo + kk * b_step, b_lbo);
                        mma_bf16(d_tmem, dah, dbh, idesc, (kb != kb0 || kk) ? 1u : 0u);
                        mma_bf16(d_tmem, dah, dbl, idesc, 1u);
                        mma_bf16(d_tmem, dal, dbh, idesc, 1u);
                    }
                    mma_commit(&empty[s]);  // frees the stage once these MMAs retire
                }
                mma_commit(&tfull[acc]);    // accumulator ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue warps 2..9 ----------------
        const uint32_t lane_base = 32 * (warp & 3);       // TMEM lanes this warp may access
        constexpr int kCols = BN / (kEpiWarps / 4);       // columns per epilogue warp
        constexpr int kChunk = kCols < 32 ? kCols : 32;   // columns per TMEM load
        const uint32_t col_base = (warp - 2) / 4 * kCols;  // which part of the tile
        float* wstage = epi_stage + (warp - 2) * (MT ? kMtWarpBytes / 4 : kStgWarpFloats);
        uint32_t sbuf = 0;  // TMA store buffer toggle
        uint32_t tl = 0;
        for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
            uint32_t mt, nt, z;
            tile_coords(t, mt, nt, z);
            const uint32_t acc = tl & 1;
            const bool has_k = z * per < ep.kblocks;  // an empty split still gets a commit
            mbar_wait(&tfull[acc], (tl >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t row = mt * BM + lane_base + lane;
            const bool row_ok = row < ep.m;
            const float rs = (row_ok && ep.row_scale && ep.split_k <= 1) ? ep.row_scale[row] : 1.f;
            if constexpr (MT) {
                // 32 columns per warp: one TMEM load, two 16-column store groups
                uint32_t raw[32];
                tmem_ld32_nowait(tmem + (lane_base << 16) + acc * BN + col_base, raw);
                mbar_wait(&mfull[acc], (tl >> 1) & 1);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const uint32_t rl = lane_base + lane;  // tile-local row
                const float* mrow = mask_s + acc * (kMaskTile / 4) + (col_base >> 5) * (BM * 32) + rl * 32;
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; j += 4) {  // 128B swizzle: 16-byte chunk ^= row & 7
                    const float4 q = *reinterpret_cast<const float4*>(mrow + (((j >> 2) ^ (rl & 7)) << 2));
                    v[j] = q.x > 0.f ? __uint_as_float(raw[j]) : 0.f;
                    v[j + 1] = q.y > 0.f ? __uint_as_float(raw[j + 1]) : 0.f;
                    v[j + 2] = q.z > 0.f ? __uint_as_float(raw[j + 2]) : 0.f;
                    v[j + 3] = q.w > 0.f ? __uint_as_float(raw[j + 3]) : 0.f;
                }
                // TMEM and the mask tile are consumed: release both
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&tempty[acc]);
                    mbar_arrive(&mempty[acc]);
                }
#pragma unroll
                for (int h = 0; h < 32; h += 16) {
                    const int32_t col0 = static_cast<int32_t>(col_base + h);
                    uint8_t* buf = reinterpret_cast<uint8_t*>(wstage) + sbuf * 4096;
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
                    const float* vv = v + h;
                    if (ep.out_hi) {
                        const uint32_t sw = (lane >> 2) & 1;  // SWIZZLE_32B: chunk ^= row bit 2
                        float sv[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            sv[j] = ep.split_unscaled ? vv[j] : vv[j] * rs;
                            if (!ep.split_unscaled && ep.relu) sv[j] = fmaxf(sv[j], 0.f);
                        }
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            uint32_t hw[4], lw[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                uint16_t h0, l0, h1, l1;
                                split_bf16(sv[8 * c + 2 * j], h0, l0);
                                split_bf16(sv[8 * c + 2 * j + 1], h1, l1);
                                hw[j] = static_cast<uint32_t>(h0) | (static_cast<uint32_t>(h1) << 16);
                                lw[j] = static_cast<uint32_t>(l0) | (static_cast<uint32_t>(l1) << 16);
                            }
                            const uint32_t off = lane * 32 + ((c ^ sw) << 4);
                            *reinterpret_cast<uint4*>(buf + 2048 + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                            *reinterpret_cast<uint4*>(buf + 3072 + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        }
                    }
                    if (ep.p24_hi) {  // packed-24 c0: hi 32 x 32 B (SWIZZLE_32B) at 0, lo 32 x 16 B at 1 KB
                        float o[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) o[j] = ep.relu ? fmaxf(vv[j] * rs, 0.f) : vv[j] * rs;
                        uint4 h0, h1, l0;
                        pack24x16(o, h0, h1, l0);
                        const uint32_t s32 = (lane >> 2) & 1;
                        *reinterpret_cast<uint4*>(buf + lane * 32 + (s32 << 4)) = h0;
                        *reinterpret_cast<uint4*>(buf + lane * 32 + ((1 ^ s32) << 4)) = h1;
                        *reinterpret_cast<uint4*>(buf + 1024 + lane * 16) = l0;
                    }
                    const uint32_t sw = (lane >> 1) & 3;  // SWIZZLE_64B
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (ep.p24_hi) break;
                        float4 o;
                        o.x = vv[4 * j] * rs;
                        o.y = vv[4 * j + 1] * rs;
                        o.z = vv[4 * j + 2] * rs;
                        o.w = vv[4 * j + 3] * rs;
                        if (ep.relu) {
                            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f);
                            o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                        }
                        *reinterpret_cast<float4*>(buf + lane * 64 + ((j ^ sw) << 4)) = o;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        const int32_t r0 = static_cast<int32_t>(mt * BM + lane_base);
                        if (ep.c0) tma_store_2d_nc(&map_c0, buf, col0, r0);
                        if (ep.p24_hi) {
                            tma_store_2d_nc(&map_phi, buf, col0, r0);
                            tma_store_2d_nc(&map_plo, buf + 1024, col0, r0);
                        }
                        if (ep.out_hi) {
                            tma_store_2d_nc(&map_shi, buf + 2048, col0, r0);
                            tma_store_2d_nc(&map_slo, buf + 3072, col0, r0);
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    sbuf ^= 1;
                }
                continue;
            }
#pragma unroll 1
            for (int cb = 0; cb < kCols; cb += kChunk) {
                uint32_t raw[32];
                if constexpr (kChunk == 32) {
                    tmem_ld32_nowait(tmem + (lane_base << 16) + acc * BN + col_base + cb, raw);
                } else {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]),
                          "=r"(raw[6]), "=r"(raw[7]), "=r"(raw[8]), "=r"(raw[9]), "=r"(raw[10]), "=r"(raw[11]),
                          "=r"(raw[12]), "=r"(raw[13]), "=r"(raw[14]), "=r"(raw[15])
                        : "r"(tmem + (lane_base << 16) + acc * BN + col_base + cb));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float v[32];
#pragma unroll
                for (int j = 0; j < kChunk; ++j) v[j] = has_k ? __uint_as_float(raw[j]) : 0.f;
#pragma unroll
                for (int h = 0; h < kChunk; h += 16) {
                    const uint32_t col0 = nt * BN + col_base + cb + h;
                    if (col0 >= ep.n) break;  // warp-uniform
                    float* vv = v + h;
                    // Row-contiguous form of the main fp32 store (warp-uniform test): the
                    // group's 32 rows x 16 columns go through smem and leave as 8 rows x 64 B
                    // per store instruction instead of 32 rows x 16 B.
                    float* fdst = nullptr;
                    uint64_t fld = 0;
                    bool fx = false;
                    const CUtensorMap* fmap = &map_c0;
                    int32_t fcol = static_cast<int32_t>(col0);
                    if (kStgBytes && ep.stage_stores && ep.split_k <= 1 && col0 + 16 <= ep.n) {
                        if (col0 + 16 <= ep.split && ep.c0 && ep.ldc0 % 4 == 0) {
                            fdst = ep.c0 + col0;
                            fld = ep.ldc0;
                            fx = ep.npeers && ep.peer_target == 0;
                        } else if (col0 >= ep.split && ep.c1 && ep.ldc1 % 4 == 0 && (col0 - ep.split) % 4 == 0) {
                            fdst = ep.c1 + (col0 - ep.split);
                            fld = ep.ldc1;
                            fx = ep.npeers && ep.peer_target == 1;
                            fmap = &map_c1;
                            fcol = static_cast<int32_t>(col0 - ep.split);
                        }
                        if (fdst && (reinterpret_cast<uintptr_t>(fdst) & 15) != 0) fdst = nullptr;
                    }
                    if (!row_ok && !fdst) continue;
                    if (ep.split_k > 1) {
                        float* dst = ep.c0 + static_cast<uint64_t>(z) * ep.m * ep.ldc0 +
                                     static_cast<uint64_t>(row) * ep.ldc0 + col0;
                        if (col0 + 16 <= ep.n && (ep.ldc0 % 4) == 0) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                *reinterpret_cast<float4*>(dst + j) = make_float4(vv[j], vv[j + 1], vv[j + 2], vv[j + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (col0 + j < ep.n) dst[j] = vv[j];
                        }
                        continue;
                    }
                    if (ep.mask && row_ok) {  // ReLU backward: zero where the forward activation was not positive
                        const float* mp = ep.mask + static_cast<uint64_t>(row) * ep.ld_mask + col0;
                        if (col0 + 16 <= ep.n && (ep.ld_mask % 4) == 0 &&
                            (reinterpret_cast<uintptr_t>(mp) & 15) == 0) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4) {
                                const float4 q = __ldg(reinterpret_cast<const float4*>(mp + j));
                                if (!(q.x > 0.f)) vv[j] = 0.f;
                                if (!(q.y > 0.f)) vv[j + 1] = 0.f;
                                if (!(q.z > 0.f)) vv[j + 2] = 0.f;
                                if (!(q.w > 0.f)) vv[j + 3] = 0.f;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (col0 + j < ep.n && !(mp[j] > 0.f)) vv[j] = 0.f;
                        }
                    }
                    if (ep.out_hi && ep.split_unscaled && row_ok)
                        store_split16(vv, ep.out_hi + static_cast<uint64_t>(row) * ep.ld_split + col0,
                                      ep.out_lo + static_cast<uint64_t>(row) * ep.ld_split + col0, col0, ep.n);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        vv[j] *= rs;
                        if (ep.relu) vv[j] = fmaxf(vv[j], 0.f);
                    }
                    if (fdst && ep.tma_store && !fx) {
                        float* buf = wstage + sbuf * 512;
                        if (lane == 0)  // the box written two stores ago has been read out
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        __syncwarp();
                        const uint32_t sw = (lane >> 1) & 3;  // SWIZZLE_64B: chunk ^= row bits [2:1]
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<float4*>(buf + lane * 16 + ((j ^ sw) << 2)) =
                                make_float4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) tma_store_2d(fmap, buf, fcol, static_cast<int32_t>(mt * BM + lane_base));
                        sbuf ^= 1;
                        if (ep.out_hi && !ep.split_unscaled && row_ok)
                            store_split16(vv, ep.out_hi + static_cast<uint64_t>(row) * ep.ld_split + col0,
                                          ep.out_lo + static_cast<uint64_t>(row) * ep.ld_split + col0, col0, ep.n);
                        continue;
                    }
                    if (fdst) {
                        float* srow = wstage + lane * kStgPitch;
                        __syncwarp();
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(srow + j) = make_float4(vv[j], vv[j + 1], vv[j + 2], vv[j + 3]);
                        __syncwarp();
                        const uint32_t sr = lane >> 2, sc = (lane & 3) * 4;
                        const float* sbase = wstage;
#pragma unroll
                        for (int pass = 0; pass < 4; ++pass) {
                            const uint32_t r = pass * 8 + sr;
                            const uint32_t orow = mt * BM + lane_base + r;
                            if (orow < ep.m)
                                store4x(fdst + static_cast<uint64_t>(orow) * fld + sc,
                                        *reinterpret_cast<const float4*>(sbase + r * kStgPitch + sc), ep, fx);
                        }
                        if (ep.out_hi && !ep.split_unscaled && row_ok)
                            store_split16(vv, ep.out_hi + static_cast<uint64_t>(row) * ep.ld_split + col0,
                                          ep.out_lo + static_cast<uint64_t>(row) * ep.ld_split + col0, col0, ep.n);
                        continue;
                    }
                    if (!row_ok) continue;
                    if (ep.p24_hi && col0 + 16 <= ep.n &&
                        (ep.p24_target == 0 ? col0 + 16 <= ep.split : col0 >= ep.split)) {
                        const uint32_t pc = ep.p24_target == 0 ? col0 : col0 - ep.split;
                        uint4 h0, h1, l0;
                        pack24x16(vv, h0, h1, l0);
                        uint4* hp = reinterpret_cast<uint4*>(ep.p24_hi + static_cast<uint64_t>(row) * ep.ld_p24_hi + pc);
                        hp[0] = h0;
                        hp[1] = h1;
                        *reinterpret_cast<uint4*>(ep.p24_lo + static_cast<uint64_t>(row) * ep.ld_p24_lo + pc) = l0;
                        if (ep.out_hi && !ep.split_unscaled)
                            store_split16(vv, ep.out_hi + static_cast<uint64_t>(row) * ep.ld_split + col0,
                                          ep.out_lo + static_cast<uint64_t>(row) * ep.ld_split + col0, col0, ep.n);
                        continue;
                    }
                    // a 16-column group entirely on one side of the split: 4 x 16 B stores
                    float* base = nullptr;
                    bool xchg = false;
                    if (col0 + 16 <= ep.n) {
                        if (col0 + 16 <= ep.split && ep.c0 && ep.ldc0 % 4 == 0) {
                            base = ep.c0 + static_cast<uint64_t>(row) * ep.ldc0 + col0;
                            xchg = ep.npeers && ep.peer_target == 0;
                        } else if (col0 >= ep.split && ep.c1 && ep.ldc1 % 4 == 0 && (col0 - ep.split) % 4 == 0) {
                            base = ep.c1 + static_cast<uint64_t>(row) * ep.ldc1 + (col0 - ep.split);
                            xchg = ep.npeers && ep.peer_target == 1;
                        }
                    }
                    if (base && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            store4x(base + j, make_float4(vv[j], vv[j + 1], vv[j + 2], vv[j + 3]), ep, xchg);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const uint32_t col = col0 + j;
                            if (col >= ep.n) continue;
                            if (col < ep.split) {
                                if (ep.c0) store1x(ep.c0 + static_cast<uint64_t>(row) * ep.ldc0 + col, vv[j], ep,
                                                   ep.npeers && ep.peer_target == 0);
                            } else if (ep.c1) {
                                store1x(ep.c1 + static_cast<uint64_t>(row) * ep.ldc1 + (col - ep.split), vv[j], ep,
                                        ep.npeers && ep.peer_target == 1);
                            }
                        }
                    }
                    if (ep.out_hi && !ep.split_unscaled)
                        store_split16(vv, ep.out_hi + static_cast<uint64_t>(row) * ep.ld_split + col0,
                                      ep.out_lo + static_cast<uint64_t>(row) * ep.ld_split + col0, col0, ep.n);
                }
            }
            // accumulator drained: hand it back to the MMA warp
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if ((MT || ep.tma_store) && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---- reference-precision SIMT GEMM (tests / tiny shapes) ----------------------
__global__ void gemm_simt_kernel(const uint16_t* a_hi, const uint16_t* a_lo, uint64_t lda, int a_mn,
                                 const uint16_t* b_hi, const uint16_t* b_lo, uint64_t ldb, int b_mn,
                                 uint32_t k, const Epi ep) {
    const uint32_t row = blockIdx.y * blockDim.y + threadIdx.y;
    const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= ep.m || col >= ep.n) return;
    float acc = 0.f;
    const uint64_t arow = ep.a_rows ? ep.a_rows[row] : row;  // gathered K-major A
    for (uint32_t i = 0; i < k; ++i) {
        const uint64_t ki = ep.b_rows ? ep.b_rows[i] : i;        // gathered MN-major B
        const uint64_t ia = a_mn ? static_cast<uint64_t>(i) * lda + row : arow * lda + i;
        const uint64_t ib = b_mn ? ki * ldb + col : static_cast<uint64_t>(col) * ldb + i;
        const float a = bf2f(a_hi[ia]) + bf2f(a_lo[ia]);
        const float b = bf2f(b_hi[ib]) + bf2f(b_lo[ib]);
        acc = fmaf(a, b, acc);
    }
    if (ep.split_k > 1) {  // single "split": write partial 0, zero the others
        for (uint32_t z = 0; z < ep.split_k; ++z)
            ep.c0[static_cast<uint64_t>(z) * ep.m * ep.ldc0 + row * ep.ldc0 + col] = z == 0 ? acc : 0.f;
        return;
    }
    if (ep.mask && !(ep.mask[row * ep.ld_mask + col] > 0.f)) acc = 0.f;
    if (ep.out_hi && ep.split_unscaled)
        split_bf16(acc, ep.out_hi[row * ep.ld_split + col], ep.out_lo[row * ep.ld_split + col]);
    float x = acc * (ep.row_scale ? ep.row_scale[row] : 1.f);
    if (ep.relu) x = fmaxf(x, 0.f);
    if (col < ep.split) {
        if (ep.c0) store1x(ep.c0 + row * ep.ldc0 + col, x, ep, ep.npeers && ep.peer_target == 0);
    } else if (ep.c1) {
        store1x(ep.c1 + row * ep.ldc1 + col - ep.split, x, ep, ep.npeers && ep.peer_target == 1);
    }
    if (ep.out_hi && !ep.split_unscaled)
        split_bf16(x, ep.out_hi[row * ep.ld_split + col], ep.out_lo[row * ep.ld_split + col]);
}

// ---- host side --------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// inner x outer matrix (inner contiguous, pitch ld elements), box {64, box_outer}
int make_map(CUtensorMap* map, const uint16_t* base, uint64_t inner, uint64_t outer, uint64_t ld,
             uint32_t box_outer) {
    auto fn = encode_fn();
    GDX_REQUIRE(fn != nullptr, GDX_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {64u, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GDX_REQUIRE(r == CUDA_SUCCESS, GDX_INTERNAL,
                "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return GDX_OK;
}

// fp32 output map for the TMA-store epilogue: (cols inner, rows outer), box {16, 32},
// 64-byte rows swizzled as the epilogue writes them.
int make_out_map(CUtensorMap* map, void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                 bool u16 = false, uint32_t box_cols = 16, uint32_t box_rows = 32, bool u8 = false) {
    auto fn = encode_fn();
    GDX_REQUIRE(fn != nullptr, GDX_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    const uint32_t esz = u8 ? 1 : u16 ? 2 : 4;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * esz};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const uint32_t row_bytes = box_cols * esz;
    const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = fn(map, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : u16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GDX_REQUIRE(r == CUDA_SUCCESS, GDX_INTERNAL,
                "cuTensorMapEncodeTiled (output) failed (" + std::to_string(static_cast<int>(r)) + ")");
    return GDX_OK;
}

bool tma_store_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GDX_GEMM_TMA_STORE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Operand maps: K-major = (k inner, rows outer, box {64, rows_per_tile});
// MN-major = (rows inner, k outer, box {64, BK}).
int operand_maps(CUtensorMap* hi, CUtensorMap* lo, const uint16_t* phi, const uint16_t* plo,
                 uint64_t rows, uint64_t k, uint64_t ld, bool mn, uint32_t tile_rows) {
    int rc;
    if (!mn) {
        if ((rc = make_map(hi, phi, k, rows, ld, tile_rows))) return rc;
        return make_map(lo, plo, k, rows, ld, tile_rows);
    }
    if ((rc = make_map(hi, phi, rows, k, ld, BK))) return rc;
    return make_map(lo, plo, rows, k, ld, BK);
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EW, bool MT = false>
int launch_tc(const gdx_gemm_args* g, const Epi& ep, cudaStream_t s) {
    CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
    int rc;
    // gathered operands: maps over the whole source (k inner for A, n inner for B), one
    // row per box -- the tile::gather4 form (tools/probe/gather4_probe.cu)
    if (g->a_rows) {
        if ((rc = make_map(&ma_hi, g->a_hi, g->k, g->a_src_rows, g->lda, 1))) return rc;
        if ((rc = make_map(&ma_lo, g->a_lo, g->k, g->a_src_rows, g->lda, 1))) return rc;
    } else if ((rc = operand_maps(&ma_hi, &ma_lo, g->a_hi, g->a_lo, g->m, g->k, g->lda, A_MN, BM))) {
        return rc;
    }
    if (g->b_rows) {
        if ((rc = make_map(&mb_hi, g->b_hi, g->n, g->b_src_rows, g->ldb, 1))) return rc;
        if ((rc = make_map(&mb_lo, g->b_lo, g->n, g->b_src_rows, g->ldb, 1))) return rc;
    } else if ((rc = operand_maps(&mb_hi, &mb_lo, g->b_hi, g->b_lo, g->n, g->k, g->ldb, B_MN, BN))) {
        return rc;
    }
    // TMA-store epilogue for the staged fp32 outputs (16-byte aligned bases, pitch % 4)
    CUtensorMap mc0{}, mc1{}, mmask{}, mshi{}, mslo{}, mphi{}, mplo{};
    Epi e = ep;
    e.tma_store = 0;
    if constexpr (MT) {  // gdx_gemm_tn checked the shapes and alignments (mask_tma_ok)
        if (ep.c0 && (rc = make_out_map(&mc0, ep.c0, ep.n, ep.m, ep.ldc0))) return rc;
        if ((rc = make_out_map(&mmask, const_cast<float*>(ep.mask), ep.n, ep.m, ep.ld_mask, false, 32, BM)))
            return rc;
        if (ep.out_hi) {
            if ((rc = make_out_map(&mshi, ep.out_hi, ep.n, ep.m, ep.ld_split, true))) return rc;
            if ((rc = make_out_map(&mslo, ep.out_lo, ep.n, ep.m, ep.ld_split, true))) return rc;
        }
        if (ep.p24_hi) {
            if ((rc = make_out_map(&mphi, ep.p24_hi, ep.n, ep.m, ep.ld_p24_hi, true))) return rc;
            if ((rc = make_out_map(&mplo, ep.p24_lo, ep.n, ep.m, ep.ld_p24_lo, false, 16, 32, true))) return rc;
        }
        e.tma_store = ep.c0 != nullptr;
    } else if (kStgBytesFor(EW) && ep.stage_stores && ep.split_k <= 1 && tma_store_enabled() && !ep.p24_hi) {
        const bool ok0 = !ep.c0 || (ep.split >= 16 && ep.ldc0 % 4 == 0 &&
                                    (reinterpret_cast<uintptr_t>(ep.c0) & 15) == 0);
        const bool ok1 = !ep.c1 || ep.split >= ep.n ||
                         (ep.ldc1 % 4 == 0 && (reinterpret_cast<uintptr_t>(ep.c1) & 15) == 0);
        if (ok0 && ok1) {
            if (ep.c0 && ep.split >= 16 && (rc = make_out_map(&mc0, ep.c0, ep.split, ep.m, ep.ldc0))) return rc;
            if (ep.c1 && ep.split < ep.n && (rc = make_out_map(&mc1, ep.c1, ep.n - ep.split, ep.m, ep.ldc1)))
                return rc;
            e.tma_store = 1;
        }
    }
    auto kern = gemm_bf16x3<BN, STAGES, A_MN, B_MN, EW, MT>;
    const int bytes = Smem<BN, STAGES, EW, MT>::kBytes;
    if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), bytes))) return rc;
    const uint64_t sms = static_cast<uint64_t>(device_sms());
    const uint64_t tiles = static_cast<uint64_t>(ep.m_tiles) * ep.n_tiles * ep.split_k;
    const unsigned grid = static_cast<unsigned>(tiles < sms ? tiles : sms);
    kern<<<grid, kThreadsFor(EW), bytes, s>>>(ma_hi, ma_lo, mb_hi, mb_lo, mc0, mc1, mmask, mshi, mslo, mphi, mplo, e);
    note_launch();
    return check_launch("gdx_gemm_tn");
}

template <int BN, int STAGES, int EW>
int launch_majors_ew(const gdx_gemm_args* g, const Epi& ep, cudaStream_t s) {
    if (!g->a_mn_major && !g->b_mn_major) return launch_tc<BN, STAGES, false, false, EW>(g, ep, s);
    if (g->a_mn_major && g->b_mn_major) return launch_tc<BN, STAGES, true, true, EW>(g, ep, s);
    if (g->a_mn_major) return launch_tc<BN, STAGES, true, false, EW>(g, ep, s);
    return launch_tc<BN, STAGES, false, true, EW>(g, ep, s);
}

template <int BN, int STAGES>
int launch_majors(const gdx_gemm_args* g, const Epi& ep, cudaStream_t s) {
    // the fused ReLU-backward epilogue (mask loads) runs with 16 epilogue warps, except on
    // very long GEMMs where 8 warps + the store-transpose staging win (6 M rows: 2.35 ->
    // 2.19 ms; 2.4 M rows: 0.84 -> 0.88, 233 K: 0.092 -> 0.110 -- tools/gemm_bench.py).
    // GDX_MASK_EW=8|16 overrides.
    static const int mask_ew = [] {
        const char* e = std::getenv("GDX_MASK_EW");
        return e ? std::atoi(e) : 0;
    }();
    const bool ew8 = mask_ew ? mask_ew == 8 : g->m >= (4u << 20);
    if (g->mask && !g->a_mn_major && g->b_mn_major && !ew8)
        return launch_tc<BN, STAGES, false, true, 16>(g, ep, s);
    return launch_majors_ew<BN, STAGES, 8>(g, ep, s);
}

// The fused ReLU-backward GEMM with the mask tile TMA-loaded and all outputs TMA-stored:
// n == 64 (one column tile), K-major A x MN-major B, a single fp32 output, no peer
// copies or split-K, 16-byte aligned bases and pitches. GDX_MASK_TMA=0 disables.
bool mask_tma_ok(const gdx_gemm_args* g, const Epi& ep) {
    static const bool on = [] {
        const char* e = std::getenv("GDX_MASK_TMA");
        return !(e && e[0] == '0');
    }();
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return on && g->mask && !g->a_rows && !g->b_rows && g->n == 64 && g->k > 0 && !g->a_mn_major && g->b_mn_major && ep.split_k <= 1 &&
           g->npeers == 0 && ep.split >= g->n && !g->c1 && (!g->c0 || (al(g->c0) && g->ldc0 % 4 == 0)) &&
           (!g->p24_hi || g->p24_target == 0) &&
           al(g->mask) && g->ld_mask % 4 == 0 &&
           (!g->out_hi || (al(g->out_hi) && al(g->out_lo) && g->ld_split % 8 == 0));
}

int validate(const gdx_gemm_args* g) {
    GDX_REQUIRE(g != nullptr, GDX_INPUT, "gdx_gemm_tn: null args");
    GDX_REQUIRE(g->a_hi && g->a_lo && g->b_hi && g->b_lo, GDX_INPUT, "gdx_gemm_tn: null operand");
    GDX_REQUIRE(g->lda >= (g->a_mn_major ? g->m : g->k) && g->ldb >= (g->b_mn_major ? g->n : g->k),
                GDX_INPUT, "gdx_gemm_tn: leading dim too small");
    GDX_REQUIRE(g->lda % 8 == 0 && g->ldb % 8 == 0, GDX_INPUT,
                "gdx_gemm_tn: leading dims must be multiples of 8 elements (16 B TMA pitch)");
    GDX_REQUIRE(g->split <= g->n, GDX_INPUT, "gdx_gemm_tn: split > n");
    GDX_REQUIRE(g->c0 || g->c1 || g->out_hi || g->p24_hi, GDX_INPUT, "gdx_gemm_tn: no output");
    GDX_REQUIRE(!g->out_hi == !g->out_lo, GDX_INPUT, "gdx_gemm_tn: out_hi/out_lo must pair");
    GDX_REQUIRE(g->split_k <= 1 || g->c0, GDX_INPUT, "gdx_gemm_tn: split_k needs c0 workspace");
    GDX_REQUIRE(!g->mask || g->ld_mask >= g->n, GDX_INPUT, "gdx_gemm_tn: ld_mask < n");
    GDX_REQUIRE(g->npeers <= 7, GDX_INPUT, "gdx_gemm_tn: at most 7 peers");
    GDX_REQUIRE(g->npeers == 0 || g->split_k <= 1, GDX_INPUT, "gdx_gemm_tn: peers with split_k");
    if (g->p24_hi) {
        const uint32_t lo = g->p24_target == 0 ? 0 : g->split, hi = g->p24_target == 0 ? g->split : g->n;
        auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        GDX_REQUIRE(g->p24_lo && (g->p24_target == 0 ? !g->c0 : !g->c1), GDX_INPUT,
                    "gdx_gemm_tn: a packed-24 output needs both planes and replaces its fp32 output");
        GDX_REQUIRE(lo % 16 == 0 && (hi - lo) % 16 == 0 && g->ld_p24_hi % 8 == 0 && g->ld_p24_lo % 16 == 0 &&
                        al(g->p24_hi) && al(g->p24_lo) && g->split_k <= 1 && g->npeers == 0,
                    GDX_INPUT, "gdx_gemm_tn: packed-24 output columns, pitches and bases must be 16-aligned");
    }
    GDX_REQUIRE(!g->a_rows || (!g->a_mn_major && g->a_src_rows > 0 && g->a_src_rows < (1ull << 31)), GDX_INPUT,
                "gdx_gemm_tn: a_rows gathers a K-major A from a_src_rows (< 2^31) source rows");
    GDX_REQUIRE(!g->b_rows || (g->b_mn_major && g->b_src_rows > 0 && g->b_src_rows < (1ull << 31)), GDX_INPUT,
                "gdx_gemm_tn: b_rows gathers an MN-major B from b_src_rows (< 2^31) source rows");
    return GDX_OK;
}

// GDX_STAGE_MIN_ROWS overrides the row count from which the staged epilogue is used
uint32_t stage_min_rows() {
    static const uint32_t v = [] {
        const char* e = std::getenv("GDX_STAGE_MIN_ROWS");
        return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : (1u << 20);
    }();
    return v;
}

Epi make_epi(const gdx_gemm_args* g, int bn) {
    Epi ep{g->m, g->n, g->c0, g->ldc0, g->c1, g->ldc1, g->split, g->row_scale, g->relu,
           g->out_hi, g->out_lo, g->ld_split, g->split_k ? g->split_k : 1,
           (g->k + BK - 1) / BK, (g->m + BM - 1) / BM, (g->n + bn - 1) / bn,
           g->mask, g->ld_mask, g->split_unscaled, g->npeers, g->peer_target, {},
           // measured (tools/gemm_bench.py): the transposed stores win on long
           // write-bound GEMMs (6 M rows: 1.2-1.25x) and lose on short ones (233 K rows)
           g->m >= stage_min_rows() && !g->p24_hi ? 1 : 0, 0, g->a_rows, g->b_rows, g->k,
           g->p24_hi, g->p24_lo, g->ld_p24_hi, g->ld_p24_lo, g->p24_target};
    for (int r = 0; r < 7; ++r) ep.peer_delta[r] = g->peer_delta[r];
    return ep;
}

}  // namespace
}  // namespace gdx

extern "C" int gdx_gemm_tn(const gdx_gemm_args* g, gdx_stream stream) {
    using namespace gdx;
    int rc = validate(g);
    if (rc) return rc;
    if (g->m == 0 || g->n == 0) return GDX_OK;
    const int bn = g->n <= 64 ? 64 : (g->n <= 128 ? 128 : 256);
    Epi ep = make_epi(g, bn);
    GDX_REQUIRE(ep.split_k <= ep.kblocks || g->k == 0, GDX_INPUT,
                "gdx_gemm_tn: split_k exceeds the number of 64-wide k blocks");
    cudaStream_t s = as_cuda(stream);
    if (bn == 64 && mask_tma_ok(g, ep)) return launch_tc<64, 2, false, true, 8, true>(g, ep, s);
    if (bn == 64) return launch_majors<64, 4>(g, ep, s);
    if (bn == 128) return launch_majors<128, 3>(g, ep, s);
    return launch_majors<256, 2>(g, ep, s);
}

extern "C" int gdx_gemm_tn_simt(const gdx_gemm_args* g, gdx_stream stream) {
    using namespace gdx;
    int rc = validate(g);
    if (rc) return rc;
    if (g->m == 0 || g->n == 0) return GDX_OK;
    Epi ep = make_epi(g, 64);
    dim3 blk(32, 8), grid((g->n + 31) / 32, (g->m + 7) / 8);
    gemm_simt_kernel<<<grid, blk, 0, as_cuda(stream)>>>(g->a_hi, g->a_lo, g->lda, g->a_mn_major, g->b_hi,
                                                        g->b_lo, g->ldb, g->b_mn_major, g->k, ep);
    note_launch();
    return check_launch("gdx_gemm_tn_simt");
}
