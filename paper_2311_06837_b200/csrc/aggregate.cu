// aggregate.cu -- K1/K3: CSR gather-reduce aggregation on sm_100a.
//
// Replaces the reference's per-vertex loop (reference_gnn.cpp:76-83, masked
// variant :123-134) and serves the transposed backward (A is symmetric,
// graph.hpp:14-18, so A^T g is the same pull over the same CSR).
//
// Design (HBM/L2-bound gather, no tensor-core work):
//  * one warp per destination row; the row's column indices are read once,
//    coalesced, with an evict-first streaming hint and broadcast by shuffle;
//  * a gathered row of F fp32 is read with 128-bit loads by LPE = pow2(F/4)
//    lanes, so 32/LPE neighbour rows are in flight per warp step, unrolled 4x
//    for memory-level parallelism;
//  * partial sums of the lane groups are combined with xor-shuffles and the
//    whole epilogue (self term, destination scale, SAGE self path, ReLU,
//    fp32 and split-bf16 stores) is fused, so the output is written once.
#include "gdx_common.cuh"

// Occupancy: 8 resident 256-thread blocks (64 warps, <= 32 registers; the few spills
// sit outside the gather loop) keep more gathers in flight.  Measured: 64-wide rows in
// the HBM regime 2.86 -> 2.60 ms (products pass, 98% of the copy peak), L2 regime 1.50
// -> 1.49 ms, 192-wide low-degree rows 4.46 -> 3.94 ms; the 12-lane warp kernel loses
// (1.51 -> 1.74 ms) and wide rows (several float4 chunks per lane) would spill heavily,
// so those keep the default.
constexpr int agg_min_blocks(int lpe, int nch) { return (lpe == 12 || nch > 1) ? 1 : 8; }

namespace gdx {
namespace {

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(pol));
    return v;
}

// 16-byte gather of a neighbour row chunk: skip L1 (no reuse on structure-free
// graphs) and keep the gathered matrix resident in L2 against the index stream.
__device__ __forceinline__ float4 ld_row4(const void* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// row address = base + nb * ld_bytes in one IMAD.WIDE.U32
__device__ __forceinline__ const char* row_addr(uint64_t base, uint32_t nb, uint32_t ldb) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(nb), "r"(ldb), "l"(base));
    return reinterpret_cast<const char*>(r);
}

__device__ __forceinline__ float4 ld_plain4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// Packed fp32 adds (FADD2 on sm_100): two lanes of a float4 per instruction.
__device__ __forceinline__ void add4(float4& a, const float4& b) {
    unsigned long long lo, hi;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(lo)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a.x)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b.x)));
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(hi)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a.z)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b.z)));
    *reinterpret_cast<unsigned long long*>(&a.x) = lo;
    *reinterpret_cast<unsigned long long*>(&a.z) = hi;
}

struct AggParams {
    const uint64_t* row_ptr;
    const uint64_t* row_end;
    const uint64_t* skip_lo;  // optional excluded sub-range [skip_lo, skip_hi) per row
    const uint64_t* skip_hi;
    const float* partial;     // optional partial sums added before the epilogue
    uint64_t ld_partial;
    const uint32_t* col;
    uint32_t rows;
    uint32_t c4;        // width / 4
    const float* src;
    uint64_t ld_src;    // elements
    uint32_t ld_bytes;  // ld_src * 4 (fits: checked on the host)
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

constexpr int pow2_floor(int x) { return x >= 32 ? 32 : x >= 16 ? 16 : x >= 8 ? 8 : x >= 4 ? 4 : x >= 2 ? 2 : 1; }

// LPE lanes cover one neighbour row (NCH float4 chunks each); EPW = pow2 rows per
// warp step; EXACT: c4 == LPE*NCH (no column masks).
template <int LPE, int NCH, bool EXACT, int UNROLL>
__global__ void __launch_bounds__(256, agg_min_blocks(LPE, NCH)) aggregate_vec4(const AggParams p) {
    constexpr int EPW = pow2_floor(32 / LPE);
    constexpr int STEP = EPW * UNROLL;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    const bool lane_on = sub < EPW;
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t base = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint32_t ldb = p.ld_bytes;
    bool chan_on[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) chan_on[c] = EXACT || (lin + c * LPE) < p.c4;

    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < p.rows;
         row += warps_total) {
        const uint64_t beg = p.row_ptr[row];
        const uint64_t end = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);

        // with a skip range the row is processed as [beg, skip_lo) then [skip_hi, end)
        const int nseg = p.skip_lo ? 2 : 1;
        for (int seg = 0; seg < nseg; ++seg) {
        uint64_t sbeg = beg, send = end;
        if (p.skip_lo) {
            if (seg == 0) send = p.skip_lo[row];
            else sbeg = p.skip_hi[row];
        }
        // index chunks of 32 are software-pipelined: chunk k+1's column ids are in
        // flight while chunk k's rows are gathered.
        uint32_t my = (sbeg + lane < send) ? ld_stream_u32(p.col + sbeg + lane, pol_stream) : 0u;
        for (uint64_t e0 = sbeg; e0 < send; e0 += 32) {
            const uint32_t cnt = static_cast<uint32_t>((send - e0) < 32 ? (send - e0) : 32);
            const uint64_t e1 = e0 + 32;
            const uint32_t nxt = (e1 + lane < send) ? ld_stream_u32(p.col + e1 + lane, pol_stream) : 0u;
            uint32_t j = 0;
            // full steps: no per-edge predicates, UNROLL gathers in flight per lane
            for (; j + STEP <= cnt; j += STEP) {
                float4 v[UNROLL][NCH];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const uint32_t nb = __shfl_sync(0xffffffffu, my, (j + u * EPW + sub) & 31);
                    const char* rp = row_addr(base, nb, ldb);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        v[u][c] = (lane_on && chan_on[c]) ? ld_row4(rp + 16 * LPE * c, pol_keep)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                    for (int c = 0; c < NCH; ++c) add4(acc[c], v[u][c]);
            }
            // tail
            for (; j < cnt; j += EPW) {
                const uint32_t slot = j + sub;
                const uint32_t nb = __shfl_sync(0xffffffffu, my, slot & 31);
                const char* rp = row_addr(base, nb, ldb);
#pragma unroll
                for (int c = 0; c < NCH; ++c)
                    if (lane_on && chan_on[c] && slot < cnt) add4(acc[c], ld_row4(rp + 16 * LPE * c, pol_keep));
            }
            my = nxt;
        }
        }
        // combine the EPW lane groups into group 0
#pragma unroll
        for (int k = EPW / 2; k >= 1; k >>= 1) {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                acc[c].x += __shfl_down_sync(0xffffffffu, acc[c].x, k * LPE);
                acc[c].y += __shfl_down_sync(0xffffffffu, acc[c].y, k * LPE);
                acc[c].z += __shfl_down_sync(0xffffffffu, acc[c].z, k * LPE);
                acc[c].w += __shfl_down_sync(0xffffffffu, acc[c].w, k * LPE);
            }
        }
        if (sub != 0) continue;
        const float scale = p.post_scale ? p.post_scale[row] : 1.f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const uint32_t ch = lin + c * LPE;
            if (!chan_on[c]) continue;
            float4 r = acc[c];
            if (p.partial) {
                const float4 q = ld_plain4(p.partial + row * p.ld_partial + 4 * ch);
                r.x += q.x;
                r.y += q.y;
                r.z += q.z;
                r.w += q.w;
            }
            if (p.self_coef != 0.f) {
                const float4 s = ld_plain4(p.src + (p.self_base + row) * p.ld_src + 4 * ch);
                r.x += p.self_coef * s.x;
                r.y += p.self_coef * s.y;
                r.z += p.self_coef * s.z;
                r.w += p.self_coef * s.w;
            }
            r.x *= scale;
            r.y *= scale;
            r.z *= scale;
            r.w *= scale;
            if (p.add) {
                const float4 q = ld_plain4(p.add + row * p.ld_add + 4 * ch);
                r.x += q.x;
                r.y += q.y;
                r.z += q.z;
                r.w += q.w;
            }
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
    }
}

// Low-degree rows (in-batch subgraphs: a few edges per row): the warp-per-row
// kernel spends most of its time on the per-row dependency chain row_ptr ->
// col -> row.  Here every LPE-lane group owns its own destination row, so a warp
// walks EPW rows at once, and each group keeps UNROLL neighbour gathers in
// flight; no shuffles, so groups diverge freely.
template <int LPE, int NCH, bool EXACT, int UNROLL>
__global__ void __launch_bounds__(256, agg_min_blocks(LPE == 12 ? 16 : LPE, NCH)) aggregate_rows(const AggParams p) {
    constexpr int EPW = pow2_floor(32 / LPE);
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    if (sub >= EPW) return;
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t base = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint32_t ldb = p.ld_bytes;
    bool chan_on[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) chan_on[c] = EXACT || (lin + c * LPE) < p.c4;
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * EPW;
    for (uint64_t r = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * EPW + sub;
         r < p.rows; r += groups) {
        const uint32_t row = static_cast<uint32_t>(r);
        const uint64_t beg = p.row_ptr[row];
        const uint64_t end = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int nseg = p.skip_lo ? 2 : 1;
        for (int seg = 0; seg < nseg; ++seg) {
            uint64_t e = beg, send = end;
            if (p.skip_lo) {
                if (seg == 0) send = p.skip_lo[row];
                else e = p.skip_hi[row];
            }
            for (; e + UNROLL <= send; e += UNROLL) {
                uint32_t nb[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) nb[u] = ld_stream_u32(p.col + e + u, pol_stream);
                float4 v[UNROLL][NCH];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const char* rp = row_addr(base, nb[u], ldb);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        v[u][c] = chan_on[c] ? ld_row4(rp + 16 * LPE * c, pol_keep)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                    for (int c = 0; c < NCH; ++c) add4(acc[c], v[u][c]);
            }
            for (; e < send; ++e) {
                const char* rp = row_addr(base, ld_stream_u32(p.col + e, pol_stream), ldb);
#pragma unroll
                for (int c = 0; c < NCH; ++c)
                    if (chan_on[c]) add4(acc[c], ld_row4(rp + 16 * LPE * c, pol_keep));
            }
        }
        const float scale = p.post_scale ? p.post_scale[row] : 1.f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const uint32_t ch = lin + c * LPE;
            if (!chan_on[c]) continue;
            float4 rr = acc[c];
            if (p.partial) {
                const float4 q = ld_plain4(p.partial + row * p.ld_partial + 4 * ch);
                rr.x += q.x;
                rr.y += q.y;
                rr.z += q.z;
                rr.w += q.w;
            }
            if (p.self_coef != 0.f) {
                const float4 q = ld_plain4(p.src + (p.self_base + row) * p.ld_src + 4 * ch);
                rr.x += p.self_coef * q.x;
                rr.y += p.self_coef * q.y;
                rr.z += p.self_coef * q.z;
                rr.w += p.self_coef * q.w;
            }
            rr.x *= scale;
            rr.y *= scale;
            rr.z *= scale;
            rr.w *= scale;
            if (p.add) {
                const float4 q = ld_plain4(p.add + row * p.ld_add + 4 * ch);
                rr.x += q.x;
                rr.y += q.y;
                rr.z += q.z;
                rr.w += q.w;
            }
            if (p.relu) {
                rr.x = fmaxf(rr.x, 0.f);
                rr.y = fmaxf(rr.y, 0.f);
                rr.z = fmaxf(rr.z, 0.f);
                rr.w = fmaxf(rr.w, 0.f);
            }
            if (p.out) *reinterpret_cast<float4*>(p.out + row * p.ld_out + 4 * ch) = rr;
            if (p.out_hi) {
                ushort4 h, l;
                split_bf16(rr.x, h.x, l.x);
                split_bf16(rr.y, h.y, l.y);
                split_bf16(rr.z, h.z, l.z);
                split_bf16(rr.w, h.w, l.w);
                *reinterpret_cast<ushort4*>(p.out_hi + row * p.ld_split + 4 * ch) = h;
                *reinterpret_cast<ushort4*>(p.out_lo + row * p.ld_split + 4 * ch) = l;
            }
        }
    }
}

// Any width / alignment: one warp per row, lanes stride over columns.
__global__ void __launch_bounds__(256) aggregate_scalar(const AggParams p, uint32_t width) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < p.rows;
         row += warps_total) {
        const uint64_t beg = p.row_ptr[row];
        const uint64_t end = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        const uint64_t s0 = p.skip_lo ? p.skip_lo[row] : end, s1 = p.skip_hi ? p.skip_hi[row] : end;
        const float scale = p.post_scale ? p.post_scale[row] : 1.f;
        for (uint32_t c = lane; c < width; c += 32) {
            float acc = p.self_coef != 0.f ? p.self_coef * p.src[(p.self_base + row) * p.ld_src + c]
                                           : 0.f;
            for (uint64_t e = beg; e < s0; ++e) acc += p.src[static_cast<uint64_t>(p.col[e]) * p.ld_src + c];
            for (uint64_t e = s1; e < end; ++e) acc += p.src[static_cast<uint64_t>(p.col[e]) * p.ld_src + c];
            if (p.partial) acc += p.partial[row * p.ld_partial + c];
            acc *= scale;
            if (p.add) acc += p.add[row * p.ld_add + c];
            if (p.relu) acc = fmaxf(acc, 0.f);
            if (p.out) p.out[row * p.ld_out + c] = acc;
            if (p.out_hi) split_bf16(acc, p.out_hi[row * p.ld_split + c], p.out_lo[row * p.ld_split + c]);
        }
    }
}

// Per-row sub-range of column ids in [lo, hi): rows are sorted, so it is contiguous.
__global__ void row_split_kernel(const uint64_t* row_ptr, const uint32_t* col, uint32_t rows,
                                 uint32_t lo, uint32_t hi, uint64_t* seg_lo, uint64_t* seg_hi) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rows; v += gridDim.x * blockDim.x) {
        auto lower = [&](uint32_t key) {
            uint64_t a = row_ptr[v], b = row_ptr[v + 1];
            while (a < b) {
                const uint64_t m = a + (b - a) / 2;
                if (col[m] < key) a = m + 1;
                else b = m;
            }
            return a;
        };
        seg_lo[v] = lower(lo);
        seg_hi[v] = lower(hi);
    }
}

template <int LPE, int NCH, bool EXACT, int UNROLL = 4>
void launch_vec(const AggParams& p, cudaStream_t s) {
    const uint32_t warps_per_block = 8;
    uint64_t blocks = (static_cast<uint64_t>(p.rows) + warps_per_block - 1) / warps_per_block;
    if (blocks > 65535ull * 64) blocks = 65535ull * 64;
    aggregate_vec4<LPE, NCH, EXACT, UNROLL><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p);
}

// Exact instantiations for the widths the engine uses (8/16/32/48/64/128/256),
// masked power-of-two fallbacks for the rest.
int pick_and_launch(const AggParams& p, cudaStream_t s) {
    switch (p.c4) {
        case 1: launch_vec<1, 1, true>(p, s); return 0;
        case 2: launch_vec<2, 1, true>(p, s); return 0;
        case 4: launch_vec<4, 1, true>(p, s); return 0;
        case 8: launch_vec<8, 1, true>(p, s); return 0;
        case 12: launch_vec<12, 1, true>(p, s); return 0;
        case 16: launch_vec<16, 1, true>(p, s); return 0;
        case 32: launch_vec<32, 1, true>(p, s); return 0;
        case 64: launch_vec<32, 2, true>(p, s); return 0;
        default: break;
    }
    const uint32_t c4 = p.c4;
    if (c4 <= 4) launch_vec<4, 1, false>(p, s);
    else if (c4 <= 8) launch_vec<8, 1, false>(p, s);
    else if (c4 <= 16) launch_vec<16, 1, false>(p, s);
    else if (c4 <= 32) launch_vec<32, 1, false>(p, s);
    else if (c4 <= 64) launch_vec<32, 2, false>(p, s);
    else if (c4 <= 128) launch_vec<32, 4, false>(p, s);
    else launch_vec<32, 8, false>(p, s);
    return 0;
}

template <int LPE, int NCH, bool EXACT>
void launch_rows(const AggParams& p, cudaStream_t s) {
    constexpr int EPW = pow2_floor(32 / LPE);
    uint64_t blocks = (static_cast<uint64_t>(p.rows) + 8 * EPW - 1) / (8 * EPW);
    if (blocks > 65535ull * 64) blocks = 65535ull * 64;
    aggregate_rows<LPE, NCH, EXACT, 4><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p);
}

int launch_rows_any(const AggParams& p, cudaStream_t s) {
    switch (p.c4) {
        case 1: launch_rows<1, 1, true>(p, s); return 0;
        case 2: launch_rows<2, 1, true>(p, s); return 0;
        case 4: launch_rows<4, 1, true>(p, s); return 0;
        case 8: launch_rows<8, 1, true>(p, s); return 0;
        case 12: launch_rows<12, 1, true>(p, s); return 0;
        case 16: launch_rows<16, 1, true>(p, s); return 0;
        case 32: launch_rows<32, 1, true>(p, s); return 0;
        case 48: launch_rows<16, 3, true>(p, s); return 0;
        case 64: launch_rows<32, 2, true>(p, s); return 0;
        default: break;
    }
    const uint32_t c4 = p.c4;
    if (c4 <= 4) launch_rows<4, 1, false>(p, s);
    else if (c4 <= 8) launch_rows<8, 1, false>(p, s);
    else if (c4 <= 16) launch_rows<16, 1, false>(p, s);
    else if (c4 <= 32) launch_rows<32, 1, false>(p, s);
    else if (c4 <= 64) launch_rows<32, 2, false>(p, s);
    else if (c4 <= 128) launch_rows<32, 4, false>(p, s);
    else launch_rows<32, 8, false>(p, s);
    return 0;
}

// variant: 4 / 8 = unroll depth of the exact 12/16-lane warp-per-row kernels
// (tuning); GDX_AGG_ROWS = the lane-group-per-row kernel for low-degree rows.
int launch_variant(const AggParams& p, int variant, cudaStream_t s) {
    if (variant == GDX_AGG_ROWS) return launch_rows_any(p, s);
    const bool u8 = variant == 8;
    if (p.c4 == 16) {
        if (u8) launch_vec<16, 1, true, 8>(p, s);
        else launch_vec<16, 1, true, 4>(p, s);
    } else if (p.c4 == 12) {
        if (u8) launch_vec<12, 1, true, 8>(p, s);
        else launch_vec<12, 1, true, 4>(p, s);
    } else if (p.c4 == 8) {
        if (u8) launch_vec<8, 1, true, 8>(p, s);
        else launch_vec<8, 1, true, 4>(p, s);
    } else {
        return pick_and_launch(p, s);
    }
    return 0;
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; }

}  // namespace
}  // namespace gdx

namespace gdx {
namespace {
int aggregate_impl(const gdx_aggregate_args* a, int variant, gdx_stream stream) {
    GDX_REQUIRE(a != nullptr, GDX_INPUT, "gdx_aggregate: null args");
    GDX_REQUIRE(a->rows == 0 || (a->row_ptr && a->col && a->src), GDX_INPUT,
                "gdx_aggregate: null CSR or source");
    GDX_REQUIRE(a->width > 0, GDX_INPUT, "gdx_aggregate: width must be >= 1");
    GDX_REQUIRE(a->ld_src >= a->width, GDX_INPUT, "gdx_aggregate: ld_src < width");
    GDX_REQUIRE(!a->out || a->ld_out >= a->width, GDX_INPUT, "gdx_aggregate: ld_out < width");
    GDX_REQUIRE(!a->out_hi == !a->out_lo, GDX_INPUT, "gdx_aggregate: out_hi/out_lo must pair");
    if (a->rows == 0) return GDX_OK;
    GDX_REQUIRE(!a->skip_lo == !a->skip_hi, GDX_INPUT, "gdx_aggregate: skip_lo/skip_hi must pair");
    GDX_REQUIRE(!a->partial || a->ld_partial >= a->width, GDX_INPUT, "gdx_aggregate: ld_partial < width");
    AggParams p{a->row_ptr, a->row_end, a->skip_lo, a->skip_hi, a->partial, a->ld_partial, a->col,
                a->rows, a->width / 4, a->src, a->ld_src,
                static_cast<uint32_t>(a->ld_src * 4), a->self_coef, a->self_base, a->post_scale,
                a->add, a->ld_add, a->relu, a->out, a->ld_out, a->out_hi, a->out_lo, a->ld_split};
    const bool vec = a->width % 4 == 0 && a->ld_src % 4 == 0 && aligned16(a->src) && a->width <= 4096 &&
                     a->ld_src * 4 < (1ull << 32) &&
                     (!a->add || (a->ld_add % 4 == 0 && aligned16(a->add))) &&
                     (!a->partial || (a->ld_partial % 4 == 0 && aligned16(a->partial))) &&
                     (!a->out || (a->ld_out % 4 == 0 && aligned16(a->out))) &&
                     (!a->out_hi || (a->ld_split % 4 == 0 && (reinterpret_cast<uintptr_t>(a->out_hi) & 7) == 0 &&
                                     (reinterpret_cast<uintptr_t>(a->out_lo) & 7) == 0));
    cudaStream_t s = as_cuda(stream);
    if (vec) {
        if (variant) launch_variant(p, variant, s);
        else pick_and_launch(p, s);
    } else {
        uint64_t blocks = (static_cast<uint64_t>(a->rows) + 7) / 8;
        if (blocks > 65535ull * 64) blocks = 65535ull * 64;
        aggregate_scalar<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, a->width);
    }
    note_launch();
    return check_launch("gdx_aggregate");
}
}  // namespace
}  // namespace gdx

extern "C" int gdx_aggregate(const gdx_aggregate_args* a, gdx_stream stream) {
    return gdx::aggregate_impl(a, 0, stream);
}

extern "C" int gdx_aggregate_variant(const gdx_aggregate_args* a, int variant, gdx_stream stream) {
    return gdx::aggregate_impl(a, variant, stream);
}

extern "C" int gdx_row_split(const uint64_t* row_ptr, const uint32_t* col, uint32_t rows, uint32_t lo,
                             uint32_t hi, uint64_t* seg_lo, uint64_t* seg_hi, gdx_stream stream) {
    GDX_REQUIRE(row_ptr && seg_lo && seg_hi && (col || rows == 0), GDX_INPUT, "gdx_row_split: null pointer");
    GDX_REQUIRE(lo <= hi, GDX_INPUT, "gdx_row_split: lo > hi");
    if (!rows) return GDX_OK;
    unsigned blocks = (rows + 255) / 256;
    if (blocks > 148u * 32u) blocks = 148u * 32u;
    gdx::row_split_kernel<<<blocks, 256, 0, gdx::as_cuda(stream)>>>(row_ptr, col, rows, lo, hi, seg_lo, seg_hi);
    gdx::note_launch();
    return gdx::check_launch("gdx_row_split");
}
