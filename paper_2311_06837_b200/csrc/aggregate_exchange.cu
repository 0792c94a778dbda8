// aggregate_exchange.cu -- the per-layer exchange and the aggregation in ONE kernel
// (the a13 exchange of sim.cpp:197-266 fused with the forward_full inner loop,
// reference_gnn.cpp:76-83, and its transposed backward), for the row-partitioned
// multi-GPU trainer.
//
// Separately, a layer's exchange is a push kernel (this rank's rows into every peer's
// copy of the gathered buffer), a local-source aggregation pass into a partial buffer,
// a wait kernel, and a remote-source pass with the epilogue: three launches on two
// streams.  Here one cooperative (co-resident) grid does, per block:
//   0. push its share of this rank's row block to every peer (16-byte NVLink stores);
//   1. the locally owned source segment of each of its rows -> the partial buffer,
//      while its pushes drain;
//   2. release its stores (system fence) and count in; the last block bumps this
//      rank's arrival slot in every peer;
//   3. thread 0 spins (acquire, system scope) until every peer's slot reached the
//      round; then the remote segments + partial + the fused epilogue, with coherent
//      loads (the remote rows were written during this kernel).
// Deadlock-free: a rank's signal depends only on its own blocks (all co-resident by
// the cooperative launch), never on a peer.
#include <cuda_runtime.h>

#include "gdx_common.cuh"

namespace gdx {
namespace {

struct Xchg {
    const uint4* push_src;  // this rank's row block of the gathered buffer
    uint64_t push_n16;
    int64_t delta[7];       // byte offsets to the same address in each peer's copy
    uint32_t npeers;
    unsigned long long* const* peer_slots;  // our slot in each peer's arrival array
    unsigned long long* slots;              // our arrival array (world entries)
    unsigned long long* expected;           // rounds completed by this rank
    uint32_t world, self;
    unsigned int* counters;                 // [0] blocks past phase 2, [1] blocks finished
    unsigned long long timeout_ns;
};

struct Agg {
    const uint64_t* row_ptr;
    const uint64_t* seg_lo;   // per row: the locally owned source sub-range
    const uint64_t* seg_hi;
    const uint32_t* col;
    uint32_t rows;
    const float* src;
    uint32_t ld_bytes;
    uint64_t ld_src;
    float* partial;
    uint64_t ld_partial;
    float self_coef;
    uint64_t self_base;
    const float* post_scale;
    const float* add;
    uint64_t ld_add;
    int relu;
    float* out;
    uint64_t ld_out;
    uint16_t* out_hi;
    uint16_t* out_lo;
    uint64_t ld_split;
};

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 ld_row4_nc(const void* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
// coherent 16-byte row load (rows written by peers during this kernel must not use .nc)
__device__ __forceinline__ float4 ld_row4_coherent(const void* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ const char* row_addr(uint64_t base, uint32_t nb, uint32_t ldb) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(nb), "r"(ldb), "l"(base));
    return reinterpret_cast<const char*>(r);
}
__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

// One warp gathers edges [b, e) of a row: LPE lanes per neighbour row (one float4 each),
// EPW rows per step, UNROLL steps in flight.  Partial sums stay per lane group.
template <int LPE, int UNROLL, bool NC>
__device__ __forceinline__ void gather(const Agg& p, uint64_t b, uint64_t e, int lane, int sub, bool lane_on,
                                       uint64_t base, uint64_t pol_keep, uint64_t pol_stream, float4& acc) {
    constexpr int EPW = 32 / LPE >= 32 ? 32 : (32 / LPE >= 16 ? 16 : (32 / LPE >= 8 ? 8 : (32 / LPE >= 4 ? 4 : (32 / LPE >= 2 ? 2 : 1))));
    constexpr int STEP = EPW * UNROLL;
    uint32_t my = (b + lane < e) ? ld_stream_u32(p.col + b + lane, pol_stream) : 0u;
    for (uint64_t e0 = b; e0 < e; e0 += 32) {
        const uint32_t cnt = static_cast<uint32_t>((e - e0) < 32 ? (e - e0) : 32);
        const uint64_t e1 = e0 + 32;
        const uint32_t nxt = (e1 + lane < e) ? ld_stream_u32(p.col + e1 + lane, pol_stream) : 0u;
        uint32_t j = 0;
        for (; j + STEP <= cnt; j += STEP) {
            float4 v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t nb = __shfl_sync(0xffffffffu, my, (j + u * EPW + sub) & 31);
                const char* rp = row_addr(base, nb, p.ld_bytes);
                v[u] = lane_on ? (NC ? ld_row4_nc(rp, pol_keep) : ld_row4_coherent(rp, pol_keep))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) add4(acc, v[u]);
        }
        for (; j < cnt; j += EPW) {
            const uint32_t slot = j + sub;
            const uint32_t nb = __shfl_sync(0xffffffffu, my, slot & 31);
            if (lane_on && slot < cnt) {
                const char* rp = row_addr(base, nb, p.ld_bytes);
                add4(acc, NC ? ld_row4_nc(rp, pol_keep) : ld_row4_coherent(rp, pol_keep));
            }
        }
        my = nxt;
    }
}

template <int LPE>
__device__ __forceinline__ void combine(float4& acc) {
    constexpr int EPW = 32 / LPE >= 32 ? 32 : (32 / LPE >= 16 ? 16 : (32 / LPE >= 8 ? 8 : (32 / LPE >= 4 ? 4 : (32 / LPE >= 2 ? 2 : 1))));
#pragma unroll
    for (int k = EPW / 2; k >= 1; k >>= 1) {
        acc.x += __shfl_down_sync(0xffffffffu, acc.x, k * LPE);
        acc.y += __shfl_down_sync(0xffffffffu, acc.y, k * LPE);
        acc.z += __shfl_down_sync(0xffffffffu, acc.z, k * LPE);
        acc.w += __shfl_down_sync(0xffffffffu, acc.w, k * LPE);
    }
}

template <int LPE, int UNROLL, bool REMOTE_NC>
__global__ void __launch_bounds__(256, 8) aggregate_exchange(const Agg p, const Xchg x) {
    constexpr int EPW = 32 / LPE >= 32 ? 32 : (32 / LPE >= 16 ? 16 : (32 / LPE >= 8 ? 8 : (32 / LPE >= 4 ? 4 : (32 / LPE >= 2 ? 2 : 1))));
    __shared__ unsigned long long s_target;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    const bool lane_on = sub < EPW;
    if (threadIdx.x == 0) s_target = *x.expected + 1;  // this exchange's round
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t base = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    const uint32_t warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    // 0. push this block's share of our rows into every peer (stores drain during phase 1)
    {
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < x.push_n16; i += stride) {
            const uint4 v = __ldg(x.push_src + i);
#pragma unroll
            for (int r = 0; r < 7; ++r)  // static indices: the deltas stay in the parameter bank
                if (static_cast<uint32_t>(r) < x.npeers)
                    reinterpret_cast<uint4*>(reinterpret_cast<char*>(const_cast<uint4*>(x.push_src)) + x.delta[r])[i] = v;
        }
    }
    // 1. local-source segments -> partial
    for (uint32_t row = warp0; row < p.rows; row += warps_total) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        // our own rows: not written by anyone during this kernel, the read-only path is legal
        gather<LPE, UNROLL, true>(p, p.seg_lo[row], p.seg_hi[row], lane, sub, lane_on, base, pol_keep, pol_stream, acc);
        combine<LPE>(acc);
        if (sub == 0) *reinterpret_cast<float4*>(p.partial + row * p.ld_partial + 4 * lin) = acc;
    }
    // 2. release our pushes; the last block signals every peer
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(&x.counters[0], 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (uint32_t r = 0; r < x.npeers; ++r) atomicAdd_system(x.peer_slots[r], 1ull);  // (once per kernel)
            x.counters[0] = 0;
        }
        // 3. wait for every peer's rows of this round
        const unsigned long long want = s_target;
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (uint32_t r = 0; r < x.world; ++r) {
            if (r == x.self) continue;
            while (true) {
                unsigned long long v;
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(x.slots + r) : "memory");
                if (v >= want) break;
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > x.timeout_ns) __trap();
                __nanosleep(64);
            }
        }
        __threadfence();
    }
    __syncthreads();
    // 4. remote segments + partial + epilogue
    for (uint32_t row = warp0; row < p.rows; row += warps_total) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint64_t rb = p.row_ptr[row], re = p.row_ptr[row + 1];
        gather<LPE, UNROLL, REMOTE_NC>(p, rb, p.seg_lo[row], lane, sub, lane_on, base, pol_keep, pol_stream, acc);
        gather<LPE, UNROLL, REMOTE_NC>(p, p.seg_hi[row], re, lane, sub, lane_on, base, pol_keep, pol_stream, acc);
        combine<LPE>(acc);
        if (sub != 0) continue;
        const uint32_t ch = lin;
        float4 r = acc;
        const float4 q = *reinterpret_cast<const float4*>(p.partial + row * p.ld_partial + 4 * ch);
        add4(r, q);
        if (p.self_coef != 0.f) {
            const float4 s = ld_row4_coherent(p.src + (p.self_base + row) * p.ld_src + 4 * ch, pol_keep);
            r.x += p.self_coef * s.x;
            r.y += p.self_coef * s.y;
            r.z += p.self_coef * s.z;
            r.w += p.self_coef * s.w;
        }
        const float scale = p.post_scale ? p.post_scale[row] : 1.f;
        r.x *= scale;
        r.y *= scale;
        r.z *= scale;
        r.w *= scale;
        if (p.add) add4(r, *reinterpret_cast<const float4*>(p.add + row * p.ld_add + 4 * ch));
        if (p.relu) {
            r.x = fmaxf(r.x, 0.f);
            r.y = fmaxf(r.y, 0.f);
            r.z = fmaxf(r.z, 0.f);
            r.w = fmaxf(r.w, 0.f);
        }
        if (p.out) *reinterpret_cast<float4*>(p.out + row * p.ld_out + 4 * ch) = r;
        if (p.out_hi) {
            ushort4 h, l;
            split_bf16(r.x, h.x, l.x);
            split_bf16(r.y, h.y, l.y);
            split_bf16(r.z, h.z, l.z);
            split_bf16(r.w, h.w, l.w);
            *reinterpret_cast<ushort4*>(p.out_hi + row * p.ld_split + 4 * ch) = h;
            *reinterpret_cast<ushort4*>(p.out_lo + row * p.ld_split + 4 * ch) = l;
        }
    }
    // the last block to finish closes the round (every block read the target first)
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(&x.counters[1], 1u);
        if (prev == gridDim.x - 1) {
            *x.expected = s_target;
            x.counters[1] = 0;
        }
    }
}

template <int LPE>
int launch(const Agg& p, const Xchg& x, cudaStream_t s) {
    // remote rows through the coherent path (reading them via .nc measured no faster)
    auto kern = aggregate_exchange<LPE, 4, false>;
    static int per_sm[64] = {0};  // resident blocks per SM (per device)
    int dev = 0;
    GDX_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && per_sm[dev] == 0) GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], kern, 256, 0));
    const int occ = dev < 64 ? per_sm[dev] : 1;
    uint64_t blocks = static_cast<uint64_t>(device_sms()) * (occ > 0 ? occ : 1);
    const uint64_t need = (static_cast<uint64_t>(p.rows) + 7) / 8;
    if (need < blocks) blocks = need ? need : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all blocks co-resident (the wait needs it)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GDX_CUDA(cudaLaunchKernelEx(&cfg, kern, p, x));
    note_launch();
    return check_launch("gdx_aggregate_exchange");
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" int gdx_aggregate_exchange(const gdx_aggregate_args* a, const uint64_t* seg_lo, const uint64_t* seg_hi,
                                      float* partial, uint64_t ld_partial, const void* push_src, uint64_t push_bytes,
                                      const int64_t* peer_delta, uint32_t npeers,
                                      unsigned long long* const* peer_slots_dev, unsigned long long* slots,
                                      unsigned long long* expected, uint32_t world, uint32_t self,
                                      unsigned int* counters, uint64_t timeout_ns, gdx_stream stream) {
    GDX_REQUIRE(a && seg_lo && seg_hi && partial && slots && expected && counters, GDX_INPUT,
                "gdx_aggregate_exchange: null pointer");
    GDX_REQUIRE(npeers <= 7 && npeers + 1 == world && self < world, GDX_INPUT,
                "gdx_aggregate_exchange: world - 1 peers, at most 7");
    GDX_REQUIRE(npeers == 0 || (peer_delta && peer_slots_dev && push_src), GDX_INPUT,
                "gdx_aggregate_exchange: null peer arguments");
    GDX_REQUIRE(push_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(push_src) & 15) == 0, GDX_INPUT,
                "gdx_aggregate_exchange: 16-byte aligned whole vectors only");
    GDX_REQUIRE(!a->row_end && !a->skip_lo && !a->partial && !a->src_lo8 && !a->out24_hi, GDX_INPUT,
                "gdx_aggregate_exchange: plain CSR rows (the split is given by seg_lo / seg_hi)");
    const uint32_t c4 = a->width / 4;
    GDX_REQUIRE(a->width % 4 == 0 && (c4 == 8 || c4 == 12 || c4 == 16 || c4 == 32) && a->ld_src % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(a->src) & 15) == 0 && ld_partial % 4 == 0 &&
                    (!a->out || a->ld_out % 4 == 0) && (!a->add || a->ld_add % 4 == 0),
                GDX_INPUT, "gdx_aggregate_exchange: widths 32, 48, 64, 128 with 16-byte rows");
    Agg p{a->row_ptr, seg_lo, seg_hi, a->col, a->rows, a->src, static_cast<uint32_t>(a->ld_src * 4), a->ld_src,
          partial, ld_partial, a->self_coef, a->self_base, a->post_scale, a->add, a->ld_add, a->relu, a->out,
          a->ld_out, a->out_hi, a->out_lo, a->ld_split};
    Xchg x{reinterpret_cast<const uint4*>(push_src), push_bytes / 16, {}, npeers, peer_slots_dev, slots, expected,
           world, self, counters, timeout_ns};
    for (uint32_t r = 0; r < npeers; ++r) {
        GDX_REQUIRE(peer_delta[r] % 16 == 0, GDX_INPUT, "gdx_aggregate_exchange: peer offsets must be 16-byte aligned");
        x.delta[r] = peer_delta[r];
    }
    if (a->rows == 0 && push_bytes == 0 && npeers == 0) return GDX_OK;
    cudaStream_t s = as_cuda(stream);
    switch (c4) {
        case 8: return launch<8>(p, x, s);
        case 12: return launch<12>(p, x, s);
        case 16: return launch<16>(p, x, s);
        default: return launch<32>(p, x, s);
    }
}
