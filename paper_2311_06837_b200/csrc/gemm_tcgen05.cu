// gemm_tcgen05.cu -- K2: the dense feature transform on 5th-gen tensor cores.
//
// Replaces apply_layer (reference_gnn.cpp:53-60) -- out = W * agg for every
// vertex -- by one TN GEMM over all rows,  C[m][n] = sum_k A[m][k] B[n][k],
// and serves the backward GEMMs of the training extension (dW = G^T H with
// split-K over vertices, dH = G W).
//
// Precision: the path must stay within 1e-4 (scaled) of an fp64 oracle, which
// TF32 or plain BF16 cannot.  Operands are stored "split bf16" (x = hi + lo,
// hi = bf16(x), lo = bf16(x - hi); |x - hi - lo| <= 2^-17 |x|) and each k-step
// issues three tcgen05.mma kind::f16 (hi*hi + hi*lo + lo*hi) into one fp32 TMEM
// accumulator: ~2^-16 relative per product, fp32 accumulation, at 1/3 of the
// bf16 tensor rate -- the GEMMs here are skinny (N <= 256) and HBM-bound anyway.
//
// Structure (one 128 x BN output tile per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer  (cp.async.bulk.tensor, 128B swizzle, mbarrier tx)
//   warp 1 / lane 0 : MMA issuer    (tcgen05.mma, tcgen05.commit -> stage release)
//   warp 2          : TMEM allocator (tcgen05.alloc / dealloc, BN fp32 columns)
//   warps 0-3       : epilogue      (tcgen05.ld 32x32b -> scale/ReLU -> fp32 / split stores)
// Operand stages: {A_hi, A_lo, B_hi, B_lo} x BK=64, S stages deep.
#include <cudaTypedefs.h>

#include <mutex>

#include "gdx_common.cuh"

namespace gdx {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row

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

// K-major, 128B-swizzled smem operand descriptor (tcgen05 "matrix descriptor"):
// start>>4 [0,14) | LBO>>4 [16,30) | SBO>>4 [32,46) | version 1 [46,48) | swizzle 2 [61,64)
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;              // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;      // SBO: 8 rows x 128 B
    d |= static_cast<uint64_t>(1) << 46;              // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;              // SWIZZLE_128B
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

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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
    uint32_t kblocks;  // total k blocks
};

template <int BN, int STAGES>
struct Smem {
    static constexpr uint32_t kA = BM * BK * 2;  // bytes per A operand tile
    static constexpr uint32_t kB = BN * BK * 2;
    static constexpr uint32_t kStage = 2 * kA + 2 * kB;
    static constexpr uint32_t kBytes = STAGES * kStage + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tn_bf16x3(const __grid_constant__ CUtensorMap map_ahi,
                   const __grid_constant__ CUtensorMap map_alo,
                   const __grid_constant__ CUtensorMap map_bhi,
                   const __grid_constant__ CUtensorMap map_blo, const Epi ep) {
    using S = Smem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* accum = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t m0 = blockIdx.x * BM;
    const uint32_t n0 = blockIdx.y * BN;

    // split-K range of k blocks
    const uint32_t per = (ep.kblocks + ep.split_k - 1) / ep.split_k;
    const uint32_t kb_begin = blockIdx.z * per;
    const uint32_t kb_end = min(ep.kblocks, kb_begin + per);
    const uint32_t nkb = kb_end > kb_begin ? kb_end - kb_begin : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(static_cast<uint32_t>(BN)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0 && nkb > 0) {
        // ---------------- TMA producer ----------------
        for (uint32_t i = 0; i < nkb; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = (i / STAGES) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * S::kStage;
            mbar_expect_tx(&full[s], S::kStage);
            const int32_t kc = static_cast<int32_t>((kb_begin + i) * BK);
            tma_load_2d(st, &map_ahi, &full[s], kc, static_cast<int32_t>(m0));
            tma_load_2d(st + S::kA, &map_alo, &full[s], kc, static_cast<int32_t>(m0));
            tma_load_2d(st + 2 * S::kA, &map_bhi, &full[s], kc, static_cast<int32_t>(n0));
            tma_load_2d(st + 2 * S::kA + S::kB, &map_blo, &full[s], kc, static_cast<int32_t>(n0));
        }
    } else if (warp == 1 && lane == 0 && nkb > 0) {
        // ---------------- MMA issuer ----------------
        // kind::f16: D=f32 (bit 4), A=B=bf16 (bits 7, 10), K-major both, N>>3 @17, M>>4 @24
        constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                   (static_cast<uint32_t>(BN >> 3) << 17) |
                                   (static_cast<uint32_t>(BM >> 4) << 24);
        for (uint32_t i = 0; i < nkb; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = (i / STAGES) & 1;
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t st = smem_u32(smem + s * S::kStage);
            const uint32_t a_hi = st, a_lo = st + S::kA, b_hi = st + 2 * S::kA,
                           b_lo = st + 2 * S::kA + S::kB;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;  // 16 bf16 along K inside the swizzle row
                const uint64_t dah = smem_desc_sw128(a_hi + off), dal = smem_desc_sw128(a_lo + off);
                const uint64_t dbh = smem_desc_sw128(b_hi + off), dbl = smem_desc_sw128(b_lo + off);
                mma_bf16(tmem, dah, dbh, idesc, (i | kk) != 0);
                mma_bf16(tmem, dah, dbl, idesc, 1);
                mma_bf16(tmem, dal, dbh, idesc, 1);
            }
            mma_commit(&empty[s]);  // frees the stage once these MMAs retire
        }
        mma_commit(accum);
    }
    __syncwarp();

    // ---------------- epilogue: TMEM -> registers -> global ----------------
    if (nkb > 0) {
        mbar_wait(accum, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const uint32_t row = m0 + warp * 32 + lane;
    const bool row_ok = row < ep.m;
    const float rs = (row_ok && ep.row_scale && ep.split_k <= 1) ? ep.row_scale[row] : 1.f;
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 16) {
        float v[16];
        if (nkb > 0) {
            tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        if (!row_ok) continue;
        if (ep.split_k > 1) {
            float* dst = ep.c0 + static_cast<uint64_t>(blockIdx.z) * ep.m * ep.ldc0 +
                         static_cast<uint64_t>(row) * ep.ldc0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t col = n0 + cb + j;
                if (col < ep.n) dst[col] = v[j];
            }
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t col = n0 + cb + j;
            if (col >= ep.n) continue;
            float x = v[j] * rs;
            if (ep.relu) x = fmaxf(x, 0.f);
            if (col < ep.split) {
                if (ep.c0) ep.c0[static_cast<uint64_t>(row) * ep.ldc0 + col] = x;
            } else if (ep.c1) {
                ep.c1[static_cast<uint64_t>(row) * ep.ldc1 + (col - ep.split)] = x;
            }
            if (ep.out_hi) {
                uint16_t h, l;
                split_bf16(x, h, l);
                ep.out_hi[static_cast<uint64_t>(row) * ep.ld_split + col] = h;
                ep.out_lo[static_cast<uint64_t>(row) * ep.ld_split + col] = l;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(static_cast<uint32_t>(BN)));
    }
}

// ---- reference-precision SIMT GEMM (tests / tiny shapes) ----------------------
__global__ void gemm_tn_simt_kernel(const uint16_t* a_hi, const uint16_t* a_lo, uint64_t lda,
                                    const uint16_t* b_hi, const uint16_t* b_lo, uint64_t ldb,
                                    uint32_t k, const Epi ep) {
    const uint32_t row = blockIdx.y * blockDim.y + threadIdx.y;
    const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= ep.m || col >= ep.n) return;
    float acc = 0.f;
    for (uint32_t i = 0; i < k; ++i) {
        const float a = bf2f(a_hi[row * lda + i]) + bf2f(a_lo[row * lda + i]);
        const float b = bf2f(b_hi[col * ldb + i]) + bf2f(b_lo[col * ldb + i]);
        acc = fmaf(a, b, acc);
    }
    if (ep.split_k > 1) {  // single "split": write partial 0, zero the others
        for (uint32_t z = 0; z < ep.split_k; ++z)
            ep.c0[static_cast<uint64_t>(z) * ep.m * ep.ldc0 + row * ep.ldc0 + col] = z == 0 ? acc : 0.f;
        return;
    }
    float x = acc * (ep.row_scale ? ep.row_scale[row] : 1.f);
    if (ep.relu) x = fmaxf(x, 0.f);
    if (col < ep.split) {
        if (ep.c0) ep.c0[row * ep.ldc0 + col] = x;
    } else if (ep.c1) {
        ep.c1[row * ep.ldc1 + col - ep.split] = x;
    }
    if (ep.out_hi) split_bf16(x, ep.out_hi[row * ep.ld_split + col], ep.out_lo[row * ep.ld_split + col]);
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

int make_map(CUtensorMap* map, const uint16_t* base, uint64_t rows, uint64_t k, uint64_t ld,
             uint32_t box_rows) {
    auto fn = encode_fn();
    GDX_REQUIRE(fn != nullptr, GDX_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {k, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GDX_REQUIRE(r == CUDA_SUCCESS, GDX_INTERNAL,
                "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return GDX_OK;
}

template <int BN, int STAGES>
int launch_tc(const gdx_gemm_args* g, const Epi& ep, cudaStream_t s) {
    CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
    int rc;
    if ((rc = make_map(&ma_hi, g->a_hi, g->m, g->k, g->lda, BM))) return rc;
    if ((rc = make_map(&ma_lo, g->a_lo, g->m, g->k, g->lda, BM))) return rc;
    if ((rc = make_map(&mb_hi, g->b_hi, g->n, g->k, g->ldb, BN))) return rc;
    if ((rc = make_map(&mb_lo, g->b_lo, g->n, g->k, g->ldb, BN))) return rc;
    auto kern = gemm_tn_bf16x3<BN, STAGES>;
    const int bytes = Smem<BN, STAGES>::kBytes;
    static bool configured = false;  // per instantiation
    if (!configured) {
        GDX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        configured = true;
    }
    dim3 grid((g->m + BM - 1) / BM, (g->n + BN - 1) / BN, ep.split_k > 1 ? ep.split_k : 1);
    kern<<<grid, 128, bytes, s>>>(ma_hi, ma_lo, mb_hi, mb_lo, ep);
    note_launch();
    return check_launch("gdx_gemm_tn");
}

int validate(const gdx_gemm_args* g) {
    GDX_REQUIRE(g != nullptr, GDX_INPUT, "gdx_gemm_tn: null args");
    GDX_REQUIRE(g->a_hi && g->a_lo && g->b_hi && g->b_lo, GDX_INPUT, "gdx_gemm_tn: null operand");
    GDX_REQUIRE(g->lda >= g->k && g->ldb >= g->k, GDX_INPUT, "gdx_gemm_tn: leading dim < k");
    GDX_REQUIRE(g->lda % 8 == 0 && g->ldb % 8 == 0, GDX_INPUT,
                "gdx_gemm_tn: leading dims must be multiples of 8 elements (16 B TMA pitch)");
    GDX_REQUIRE(g->split <= g->n, GDX_INPUT, "gdx_gemm_tn: split > n");
    GDX_REQUIRE(g->c0 || g->c1 || g->out_hi, GDX_INPUT, "gdx_gemm_tn: no output");
    GDX_REQUIRE(!g->out_hi == !g->out_lo, GDX_INPUT, "gdx_gemm_tn: out_hi/out_lo must pair");
    GDX_REQUIRE(g->split_k <= 1 || g->c0, GDX_INPUT, "gdx_gemm_tn: split_k needs c0 workspace");
    return GDX_OK;
}

Epi make_epi(const gdx_gemm_args* g) {
    Epi ep{g->m, g->n, g->c0, g->ldc0, g->c1, g->ldc1, g->split, g->row_scale, g->relu,
           g->out_hi, g->out_lo, g->ld_split, g->split_k ? g->split_k : 1,
           (g->k + BK - 1) / BK};
    if (ep.split_k > ep.kblocks && ep.kblocks > 0) ep.split_k = ep.kblocks;
    return ep;
}

}  // namespace
}  // namespace gdx

extern "C" int gdx_gemm_tn(const gdx_gemm_args* g, gdx_stream stream) {
    using namespace gdx;
    int rc = validate(g);
    if (rc) return rc;
    if (g->m == 0 || g->n == 0) return GDX_OK;
    Epi ep = make_epi(g);
    GDX_REQUIRE(ep.split_k == (g->split_k ? g->split_k : 1) || g->k == 0, GDX_INPUT,
                "gdx_gemm_tn: split_k exceeds the number of 64-wide k blocks");
    cudaStream_t s = as_cuda(stream);
    if (g->n <= 64) return launch_tc<64, 4>(g, ep, s);
    if (g->n <= 128) return launch_tc<128, 3>(g, ep, s);
    return launch_tc<256, 2>(g, ep, s);
}

extern "C" int gdx_gemm_tn_simt(const gdx_gemm_args* g, gdx_stream stream) {
    using namespace gdx;
    int rc = validate(g);
    if (rc) return rc;
    if (g->m == 0 || g->n == 0) return GDX_OK;
    Epi ep = make_epi(g);
    ep.split_k = g->split_k ? g->split_k : 1;
    dim3 blk(32, 8), grid((g->n + 31) / 32, (g->m + 7) / 8);
    gemm_tn_simt_kernel<<<grid, blk, 0, as_cuda(stream)>>>(g->a_hi, g->a_lo, g->lda, g->b_hi,
                                                           g->b_lo, g->ldb, g->k, ep);
    note_launch();
    return check_launch("gdx_gemm_tn_simt");
}
