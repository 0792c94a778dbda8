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
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

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
    const uint32_t* row_list; // optional: the rows to compute (list position -> destination row)
    const uint8_t* src_lo8;   // packed-24 source: src is the u16 high plane, this the u8 low plane
    uint16_t* out24_hi;       // optional packed-24 copy of the output
    uint8_t* out24_lo;
    uint64_t ld_out24;
    uint64_t ld_lo8;          // low-plane pitch of a packed-24 source (u8 elements)
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
    for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < p.rows;
         it += warps_total) {
        const uint32_t row = p.row_list ? p.row_list[it] : it;
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
        const uint32_t row = p.row_list ? p.row_list[r] : static_cast<uint32_t>(r);
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
            if (NCH == 1 && e < send) {
                // the < UNROLL remaining edges as one predicated block: their index and row
                // loads go out together instead of as a serial col -> row chain per edge
                // (low-degree rows are mostly tail). Same edge order. Measured at 6 M rows x
                // 64 (tools/agg_bench.py): degree 3 1.80 -> 1.60 ms, 6 2.65 -> 2.33; with two
                // chunks per lane (GDX_AGG_ROWS2) it loses (2.36 -> 2.50), so NCH 1 only.
                uint32_t nb[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) nb[u] = e + u < send ? ld_stream_u32(p.col + e + u, pol_stream) : 0u;
                float4 v[UNROLL][NCH];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const char* rp = row_addr(base, nb[u], ldb);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        v[u][c] = chan_on[c] && e + u < send ? ld_row4(rp + 16 * LPE * c, pol_keep)
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    if (e + u < send)
#pragma unroll
                        for (int c = 0; c < NCH; ++c) add4(acc[c], v[u][c]);
            } else {
                for (; e < send; ++e) {
                    const char* rp = row_addr(base, ld_stream_u32(p.col + e, pol_stream), ldb);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        if (chan_on[c]) add4(acc[c], ld_row4(rp + 16 * LPE * c, pol_keep));
                }
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

__device__ __forceinline__ void epi4(const AggParams& p, uint32_t row, uint32_t ch, float4 r);

// Epilogue of one destination row for a lane group (lane lin holds columns lin + c LPE).
template <int LPE, int NCH>
__device__ __forceinline__ void group_epilogue(const AggParams& p, uint32_t row, int lin, const bool (&chan_on)[NCH],
                                               const float4 (&acc)[NCH]) {
#pragma unroll
    for (int c = 0; c < NCH; ++c)
        if (chan_on[c]) epi4(p, row, lin + c * LPE, acc[c]);
}

// Low-degree rows, edge-flat (GDX_AGG_FLAT): a lane group owns RG = LPE - 1 consecutive
// rows -- one contiguous edge range -- and walks those edges in order with UNROLL
// gathers in flight across row boundaries, flushing each row's epilogue as the walk
// passes it.  The rows' offsets come in one coalesced load (one per lane) and the
// column ids LPE at a time, so the per-row row_ptr -> col -> row chain of
// aggregate_rows becomes one chain per RG rows.  A row's edges are summed in ascending
// order, as in aggregate_rows.  Plain CSR rows only (no row_end / skip / row list).
template <int LPE, int NCH, bool EXACT, int UNROLL>
__global__ void __launch_bounds__(256, 4) aggregate_flat(const AggParams p) {
    constexpr int EPW = pow2_floor(32 / LPE);
    constexpr uint32_t RG = LPE - 1;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    if (sub >= EPW) return;
    const int g0 = sub * LPE;  // first lane of this group
    const uint32_t gmask = (LPE >= 32) ? 0xffffffffu : (((1u << LPE) - 1u) << g0);
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t base = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint32_t ldb = p.ld_bytes;
    bool chan_on[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) chan_on[c] = EXACT || (lin + c * LPE) < p.c4;
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * EPW;
    for (uint64_t grp = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * EPW + sub;
         grp * RG < p.rows; grp += groups) {
        const uint32_t a = static_cast<uint32_t>(grp * RG);
        const uint32_t nr = (p.rows - a) < RG ? (p.rows - a) : RG;
        const uint64_t myoff = static_cast<uint32_t>(lin) <= nr ? p.row_ptr[a + lin] : 0;
        uint64_t e = __shfl_sync(gmask, myoff, g0);
        const uint64_t eend = __shfl_sync(gmask, myoff, g0 + static_cast<int>(nr));
        uint32_t k = 0;
        uint64_t next_off = __shfl_sync(gmask, myoff, g0 + 1);
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        while (e < eend) {
            const uint32_t cnt = static_cast<uint32_t>((eend - e) < LPE ? (eend - e) : LPE);
            const uint32_t mycol = static_cast<uint32_t>(lin) < cnt ? ld_stream_u32(p.col + e + lin, pol_stream) : 0u;
            for (uint32_t j = 0; j < cnt; j += UNROLL) {
                float4 v[UNROLL][NCH];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const uint32_t idx = j + u;
                    const uint32_t nb = __shfl_sync(gmask, mycol, g0 + static_cast<int>(idx < cnt ? idx : 0));
                    const char* rp = row_addr(base, nb, ldb);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        v[u][c] = (idx < cnt && chan_on[c]) ? ld_row4(rp + 16 * LPE * c, pol_keep)
                                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    if (j + u >= cnt) break;
                    const uint64_t ed = e + j + u;
                    while (ed >= next_off) {  // group-uniform: the walk passed row k
                        group_epilogue<LPE, NCH>(p, a + k, lin, chan_on, acc);
#pragma unroll
                        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                        ++k;
                        next_off = __shfl_sync(gmask, myoff, g0 + static_cast<int>(k + 1));
                    }
#pragma unroll
                    for (int c = 0; c < NCH; ++c) add4(acc[c], v[u][c]);
                }
            }
            e += cnt;
        }
        for (; k < nr; ++k) {
            group_epilogue<LPE, NCH>(p, a + k, lin, chan_on, acc);
#pragma unroll
            for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// Any width / alignment: one warp per row, lanes stride over columns.
__global__ void __launch_bounds__(256) aggregate_scalar(const AggParams p, uint32_t width) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < p.rows;
         it += warps_total) {
        const uint32_t row = p.row_list ? p.row_list[it] : it;
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

// ---- packed-24 rows ----------------------------------------------------------------
// A gathered matrix may be stored as fp32 rounded to 24 bits (sign, exponent, 15
// mantissa bits; relative error <= 2^-16, the precision of the split-bf16 GEMM
// operands that produce and consume it) in two planes: the high 16 bits (u16) and
// the next 8 bits (u8).  A 64-wide row is then 128 + 64 bytes (6 sectors) instead
// of 256 (8 sectors): the L2-bound gather moves 25% fewer bytes.  Decoding is three
// byte permutes per two values; accumulation stays fp32. pack24 / unpack24 are in
// gdx_common.cuh (the GEMM epilogue writes the format too).

// 8 values from one 16-byte high-plane vector and one 8-byte low-plane vector
__device__ __forceinline__ void decode8(const uint4 h, const uint2 l, float4& a, float4& b) {
    // t = [l1 0 l0 0] style spreads of the low bytes, then [h.hi h.lo l 0] per value
    const uint32_t t0 = __byte_perm(l.x, 0u, 0x1404), t1 = __byte_perm(l.x, 0u, 0x3424);
    const uint32_t t2 = __byte_perm(l.y, 0u, 0x1404), t3 = __byte_perm(l.y, 0u, 0x3424);
    a.x = __uint_as_float(__byte_perm(h.x, t0, 0x1054));
    a.y = __uint_as_float(__byte_perm(h.x, t0, 0x3276));
    a.z = __uint_as_float(__byte_perm(h.y, t1, 0x1054));
    a.w = __uint_as_float(__byte_perm(h.y, t1, 0x3276));
    b.x = __uint_as_float(__byte_perm(h.z, t2, 0x1054));
    b.y = __uint_as_float(__byte_perm(h.z, t2, 0x3276));
    b.z = __uint_as_float(__byte_perm(h.w, t3, 0x1054));
    b.w = __uint_as_float(__byte_perm(h.w, t3, 0x3276));
}

__device__ __forceinline__ uint2 ld_row8b(const void* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_row16b(const void* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// Epilogue of 8 columns [8 ch, 8 ch + 8) of one destination row (shared by the
// packed-24 kernels): partial, self term, scale, SAGE add, ReLU, fp32 / split /
// packed-24 stores.
__device__ __forceinline__ void epilogue8(const AggParams& p, uint32_t row, uint32_t ch, float4 r0, float4 r1) {
    const float scale = p.post_scale ? p.post_scale[row] : 1.f;
    float v[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const uint32_t c0 = 8 * ch;
    if (p.partial) {
        const float4 a = ld_plain4(p.partial + row * p.ld_partial + c0);
        const float4 b = ld_plain4(p.partial + row * p.ld_partial + c0 + 4);
        v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
        v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
    if (p.self_coef != 0.f) {
        const uint64_t o = (p.self_base + row) * p.ld_src + c0;
        const uint4 h = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.src) + o));
        const uint2 l = __ldg(reinterpret_cast<const uint2*>(p.src_lo8 + (p.self_base + row) * p.ld_lo8 + c0));
        float4 a, b;
        decode8(h, l, a, b);
        v[0] += p.self_coef * a.x; v[1] += p.self_coef * a.y; v[2] += p.self_coef * a.z; v[3] += p.self_coef * a.w;
        v[4] += p.self_coef * b.x; v[5] += p.self_coef * b.y; v[6] += p.self_coef * b.z; v[7] += p.self_coef * b.w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] *= scale;
    if (p.add) {
        const float4 a = ld_plain4(p.add + row * p.ld_add + c0);
        const float4 b = ld_plain4(p.add + row * p.ld_add + c0 + 4);
        v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
        v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
    if (p.relu) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
    }
    if (p.out) {
        *reinterpret_cast<float4*>(p.out + row * p.ld_out + c0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(p.out + row * p.ld_out + c0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (p.out_hi) {
        ushort4 h0, l0, h1, l1;
        split_bf16(v[0], h0.x, l0.x); split_bf16(v[1], h0.y, l0.y);
        split_bf16(v[2], h0.z, l0.z); split_bf16(v[3], h0.w, l0.w);
        split_bf16(v[4], h1.x, l1.x); split_bf16(v[5], h1.y, l1.y);
        split_bf16(v[6], h1.z, l1.z); split_bf16(v[7], h1.w, l1.w);
        *reinterpret_cast<ushort4*>(p.out_hi + row * p.ld_split + c0) = h0;
        *reinterpret_cast<ushort4*>(p.out_hi + row * p.ld_split + c0 + 4) = h1;
        *reinterpret_cast<ushort4*>(p.out_lo + row * p.ld_split + c0) = l0;
        *reinterpret_cast<ushort4*>(p.out_lo + row * p.ld_split + c0 + 4) = l1;
    }
    if (p.out24_hi) {
        uint16_t h[8];
        uint8_t l[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pack24(v[i], h[i], l[i]);
        *reinterpret_cast<uint4*>(p.out24_hi + row * p.ld_out24 + c0) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint2*>(p.out24_lo + row * p.ld_out24 + c0) = *reinterpret_cast<uint2*>(l);
    }
}

// Warp per destination row over packed-24 sources: LPE lanes x 8 values cover a row,
// EPW rows in flight per warp step, UNROLL steps unrolled.
template <int LPE, int UNROLL, int MINB, bool HOLE = false>
__global__ void __launch_bounds__(256, MINB) aggregate_p24(const AggParams p) {
    constexpr int EPW = pow2_floor(32 / LPE);
    constexpr int STEP = EPW * UNROLL;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    const bool lane_on = sub < EPW;
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t hbase = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint64_t lbase = reinterpret_cast<uint64_t>(p.src_lo8) + 8 * lin;
    const uint32_t ldh = static_cast<uint32_t>(p.ld_src * 2), ldl = static_cast<uint32_t>(p.ld_lo8);
    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < p.rows; it += warps_total) {
        const uint32_t row = p.row_list ? p.row_list[it] : it;
        const uint64_t beg = p.row_ptr[row];
        const uint64_t end = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
        // HOLE (the exchange's remote-source pass, skip range [skip_lo, skip_hi) given):
        // both sides of the hole are walked as ONE logical edge stream, so 32-edge chunks
        // run across it and a row pays one partial chunk instead of two.  Otherwise the
        // row (or each side of a skip range) is its own segment.
        const int nseg = (!HOLE && p.skip_lo) ? 2 : 1;
        for (int seg = 0; seg < nseg; ++seg) {
            uint64_t sbeg = beg, send = end, n0 = ~0ull, hole = 0;
            if (HOLE) {
                const uint64_t slo = p.skip_lo[row], shi = p.skip_hi[row];
                n0 = slo;
                hole = shi - slo;
                send = end - hole;
            } else if (p.skip_lo) {
                if (seg == 0) send = p.skip_lo[row];
                else sbeg = p.skip_hi[row];
            }
            // logical edge e -> physical e (+ hole past skip_lo)
            uint32_t my = (sbeg + lane < send)
                              ? ld_stream_u32(p.col + sbeg + lane + (HOLE && sbeg + lane >= n0 ? hole : 0), pol_stream)
                              : 0u;
            for (uint64_t e0 = sbeg; e0 < send; e0 += 32) {
                const uint32_t cnt = static_cast<uint32_t>((send - e0) < 32 ? (send - e0) : 32);
                const uint64_t e1 = e0 + 32;
                const uint32_t nxt = (e1 + lane < send)
                                         ? ld_stream_u32(p.col + e1 + lane + (HOLE && e1 + lane >= n0 ? hole : 0), pol_stream)
                                         : 0u;
                uint32_t j = 0;
                for (; j + STEP <= cnt; j += STEP) {
                    uint4 h[UNROLL];
                    uint2 l[UNROLL];
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        const uint32_t nb = __shfl_sync(0xffffffffu, my, (j + u * EPW + sub) & 31);
                        if (lane_on) {
                            h[u] = ld_row16b(row_addr(hbase, nb, ldh), pol_keep);
                            l[u] = ld_row8b(row_addr(lbase, nb, ldl), pol_keep);
                        } else {
                            h[u] = make_uint4(0, 0, 0, 0);
                            l[u] = make_uint2(0, 0);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        float4 x0, x1;
                        decode8(h[u], l[u], x0, x1);
                        add4(a0, x0);
                        add4(a1, x1);
                    }
                }
                for (; j < cnt; j += EPW) {
                    const uint32_t slot = j + sub;
                    const uint32_t nb = __shfl_sync(0xffffffffu, my, slot & 31);
                    if (lane_on && slot < cnt) {
                        float4 x0, x1;
                        decode8(ld_row16b(row_addr(hbase, nb, ldh), pol_keep), ld_row8b(row_addr(lbase, nb, ldl), pol_keep),
                                x0, x1);
                        add4(a0, x0);
                        add4(a1, x1);
                    }
                }
                my = nxt;
            }
        }
#pragma unroll
        for (int k = EPW / 2; k >= 1; k >>= 1) {
            a0.x += __shfl_down_sync(0xffffffffu, a0.x, k * LPE);
            a0.y += __shfl_down_sync(0xffffffffu, a0.y, k * LPE);
            a0.z += __shfl_down_sync(0xffffffffu, a0.z, k * LPE);
            a0.w += __shfl_down_sync(0xffffffffu, a0.w, k * LPE);
            a1.x += __shfl_down_sync(0xffffffffu, a1.x, k * LPE);
            a1.y += __shfl_down_sync(0xffffffffu, a1.y, k * LPE);
            a1.z += __shfl_down_sync(0xffffffffu, a1.z, k * LPE);
            a1.w += __shfl_down_sync(0xffffffffu, a1.w, k * LPE);
        }
        if (sub == 0 && 2 * lin < static_cast<int>(p.c4)) epilogue8(p, row, lin, a0, a1);
    }
}

// Lane group per destination row (low-degree rows) over packed-24 sources.
template <int LPE, int UNROLL, int MINB>
__global__ void __launch_bounds__(256, MINB) aggregate_rows_p24(const AggParams p) {
    constexpr int EPW = pow2_floor(32 / LPE);
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    if (sub >= EPW) return;
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t hbase = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    const uint64_t lbase = reinterpret_cast<uint64_t>(p.src_lo8) + 8 * lin;
    const uint32_t ldh = static_cast<uint32_t>(p.ld_src * 2), ldl = static_cast<uint32_t>(p.ld_lo8);
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * EPW;
    for (uint64_t r = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * EPW + sub; r < p.rows;
         r += groups) {
        const uint32_t row = p.row_list ? p.row_list[r] : static_cast<uint32_t>(r);
        const uint64_t beg = p.row_ptr[row];
        const uint64_t end = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
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
                uint4 h[UNROLL];
                uint2 l[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    h[u] = ld_row16b(row_addr(hbase, nb[u], ldh), pol_keep);
                    l[u] = ld_row8b(row_addr(lbase, nb[u], ldl), pol_keep);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    float4 x0, x1;
                    decode8(h[u], l[u], x0, x1);
                    add4(a0, x0);
                    add4(a1, x1);
                }
            }
            for (; e < send; ++e) {
                const uint32_t nb = ld_stream_u32(p.col + e, pol_stream);
                float4 x0, x1;
                decode8(ld_row16b(row_addr(hbase, nb, ldh), pol_keep), ld_row8b(row_addr(lbase, nb, ldl), pol_keep), x0,
                        x1);
                add4(a0, x0);
                add4(a1, x1);
            }
        }
        if (2 * lin < static_cast<int>(p.c4)) epilogue8(p, row, lin, a0, a1);
    }
}

__global__ void pack24_kernel(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols, uint16_t* hi,
                              uint8_t* lo, uint64_t ld_dst) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        pack24(src[r * ld_src + c], hi[r * ld_dst + c], lo[r * ld_dst + c]);
    }
}

__global__ void unpack24_kernel(const uint16_t* hi, const uint8_t* lo, uint64_t ld_src, uint32_t rows, uint32_t cols,
                                float* dst, uint64_t ld_dst) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        dst[r * ld_dst + c] = unpack24(hi[r * ld_src + c], lo[r * ld_src + c]);
    }
}

int launch_p24(const AggParams& p, int variant, cudaStream_t s) {
    const uint32_t c8 = p.c4 / 2;
    auto vec = [&](auto kern, int epw) {
        uint64_t blocks = (static_cast<uint64_t>(p.rows) + 7) / 8;
        if (variant == GDX_AGG_ROWS) blocks = (static_cast<uint64_t>(p.rows) + 8 * epw - 1) / (8 * epw);
        if (blocks > 65535ull * 64) blocks = 65535ull * 64;
        kern<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p);
    };
    const bool rows = variant == GDX_AGG_ROWS;
    // resident blocks per SM: GDX_P24_MINB tuning knob, default 4 (60 registers, no spills;
    // measured: Reddit 64-wide 1.22 ms at 4, 1.69 at 6, 2.61 at 8 -- tools/agg24_bench.py;
    // 5 (48-register cap, 40 warps/SM) spills at UNROLL 4: epoch 8.8 -> 9.6 ms, 10.0 at UNROLL 2)
    static const int minb = [] {
        const char* e = std::getenv("GDX_P24_MINB");
        return e ? std::atoi(e) : 4;
    }();
#define GDX_P24_CASE(C8, LPE, UN, EPW)                                                          \
    case C8:                                                                                    \
        if (minb >= 8) rows ? vec(aggregate_rows_p24<LPE, UN, 8>, EPW) : vec(aggregate_p24<LPE, UN, 8>, EPW); \
        else if (minb >= 6) rows ? vec(aggregate_rows_p24<LPE, UN, 6>, EPW) : vec(aggregate_p24<LPE, UN, 6>, EPW); \
        else rows ? vec(aggregate_rows_p24<LPE, UN, 4>, EPW) : vec(aggregate_p24<LPE, UN, 4>, EPW); \
        return 0;
    // tuning: GDX_P24_UN=2 for the 64-wide warp-per-row kernel (lower unroll, more
    // resident warps at MINB 6/8)
    static const int un2 = [] {
        const char* e = std::getenv("GDX_P24_UN");
        return e && std::atoi(e) == 2;
    }();
    // GDX_AGG_P24_WIDE: 48-wide rows on a >= 64-column pitch gathered as whole 64-wide
    // rows by the 8-lane kernels (16 lanes per 4 rows instead of 6-lane groups that leave
    // a quarter of the warp idle); columns >= width are summed but never stored.
    // Measured (Reddit, tools/agg24_bench.py): 6-lane row groups 1.38 ms, 6-lane warp per
    // row 1.66 ms.
    // the exchange's remote-source pass (skip range): one edge stream across the hole
    // (N=2: 4.95 -> 4.88 ms, N=4: 2.66 -> 2.63 ms per Reddit epoch, tools/r02/hole_ab.sh)
    const bool hole = p.skip_lo && minb < 6 && !un2 && !rows;
    if (variant == GDX_AGG_P24_WIDE && c8 == 6) {
        if (minb >= 6) vec(aggregate_p24<8, 4, 6>, 4);
        else if (hole) vec(aggregate_p24<8, 4, 4, true>, 4);
        else vec(aggregate_p24<8, 4, 4>, 4);
        return 0;
    }
    if (c8 == 8 && hole) {
        vec(aggregate_p24<8, 4, 4, true>, 4);
        return 0;
    }
    if (c8 == 8 && un2 && !rows) {
        if (minb >= 8) vec(aggregate_p24<8, 2, 8>, 4);
        else if (minb >= 6) vec(aggregate_p24<8, 2, 6>, 4);
        else vec(aggregate_p24<8, 2, 4>, 4);
        return 0;
    }
    switch (c8) {
        GDX_P24_CASE(1, 1, 4, 32)
        GDX_P24_CASE(2, 2, 4, 16)
        GDX_P24_CASE(4, 4, 4, 8)
        GDX_P24_CASE(6, 6, 4, 4)
        GDX_P24_CASE(8, 8, 4, 4)
        GDX_P24_CASE(12, 12, 4, 2)
        GDX_P24_CASE(16, 16, 4, 2)
        GDX_P24_CASE(32, 32, 2, 1)
        default: return -1;
    }
#undef GDX_P24_CASE
}

// ---- heavy rows (degree-binned load balancing) ----------------------------------
// On skewed graphs a hub row (10^4..10^6 edges) would keep one warp busy long after
// the rest of the pass finished.  Rows above a degree threshold are cut into chunks of
// a fixed number of edges; one warp per chunk gathers it (the aggregate_vec4 inner
// loop, same MLP) into an fp32 partial row, then one warp per heavy row sums its
// chunks in chunk order (deterministic) and applies the epilogue.  Light rows run the
// normal kernels through a row list.

// Epilogue of one float4 column chunk (the fp32 kernels' epilogue, shared form).
__device__ __forceinline__ void epi4(const AggParams& p, uint32_t row, uint32_t ch, float4 r) {
    const float scale = p.post_scale ? p.post_scale[row] : 1.f;
    if (p.partial) {
        const float4 q = ld_plain4(p.partial + row * p.ld_partial + 4 * ch);
        r.x += q.x; r.y += q.y; r.z += q.z; r.w += q.w;
    }
    if (p.self_coef != 0.f) {
        const float4 q = ld_plain4(p.src + (p.self_base + row) * p.ld_src + 4 * ch);
        r.x += p.self_coef * q.x; r.y += p.self_coef * q.y; r.z += p.self_coef * q.z; r.w += p.self_coef * q.w;
    }
    r.x *= scale; r.y *= scale; r.z *= scale; r.w *= scale;
    if (p.add) {
        const float4 q = ld_plain4(p.add + row * p.ld_add + 4 * ch);
        r.x += q.x; r.y += q.y; r.z += q.z; r.w += q.w;
    }
    if (p.relu) {
        r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f); r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
    }
    if (p.out) *reinterpret_cast<float4*>(p.out + row * p.ld_out + 4 * ch) = r;
    if (p.out_hi) {
        ushort4 h, l;
        split_bf16(r.x, h.x, l.x); split_bf16(r.y, h.y, l.y); split_bf16(r.z, h.z, l.z); split_bf16(r.w, h.w, l.w);
        *reinterpret_cast<ushort4*>(p.out_hi + row * p.ld_split + 4 * ch) = h;
        *reinterpret_cast<ushort4*>(p.out_lo + row * p.ld_split + 4 * ch) = l;
    }
}

// One warp per chunk: edges [chunk_beg, chunk_beg + chunk_edges) of row heavy[chunk_row],
// clipped to the row's effective range (row_ptr / row_end) minus the skip range.
template <int LPE, int NCH>
__global__ void __launch_bounds__(256) heavy_chunks(const AggParams p, const uint32_t* heavy, const uint32_t* chunk_row,
                                                   const uint64_t* chunk_beg, uint32_t nchunks, uint32_t chunk_edges,
                                                   float* part, uint64_t ld_part) {
    constexpr int EPW = pow2_floor(32 / LPE);
    constexpr int UNROLL = 4;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPE;
    const int lin = lane - sub * LPE;
    const bool lane_on = sub < EPW;
    uint64_t pol_keep, pol_stream;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const uint64_t base = reinterpret_cast<uint64_t>(p.src) + 16 * lin;
    bool chan_on[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) chan_on[c] = (lin + c * LPE) < p.c4;
    const uint32_t warps_total = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ci < nchunks; ci += warps_total) {
        const uint32_t row = heavy[chunk_row[ci]];
        const uint64_t rb = p.row_ptr[row];
        const uint64_t re = p.row_end ? p.row_end[row] : p.row_ptr[row + 1];
        const uint64_t cb = chunk_beg[ci], ce = cb + chunk_edges;
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int nseg = p.skip_lo ? 2 : 1;
        for (int seg = 0; seg < nseg; ++seg) {
            uint64_t a = rb, b = re;
            if (p.skip_lo) {
                if (seg == 0) b = p.skip_lo[row];
                else a = p.skip_hi[row];
            }
            a = a > cb ? a : cb;
            b = b < ce ? b : ce;
            for (uint64_t e0 = a; e0 < b; e0 += 32) {
                const uint32_t cnt = static_cast<uint32_t>((b - e0) < 32 ? (b - e0) : 32);
                const uint32_t my = lane < cnt ? ld_stream_u32(p.col + e0 + lane, pol_stream) : 0u;
                for (uint32_t j = 0; j < cnt; j += EPW * UNROLL) {
                    float4 v[UNROLL][NCH];
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u) {
                        const uint32_t slot = j + u * EPW + sub;
                        const uint32_t nb = __shfl_sync(0xffffffffu, my, slot & 31);
                        const char* rp = row_addr(base, nb, p.ld_bytes);
#pragma unroll
                        for (int c = 0; c < NCH; ++c)
                            v[u][c] = (lane_on && chan_on[c] && slot < cnt) ? ld_row4(rp + 16 * LPE * c, pol_keep)
                                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                        for (int c = 0; c < NCH; ++c) add4(acc[c], v[u][c]);
                }
            }
        }
#pragma unroll
        for (int k = EPW / 2; k >= 1; k >>= 1)
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                acc[c].x += __shfl_down_sync(0xffffffffu, acc[c].x, k * LPE);
                acc[c].y += __shfl_down_sync(0xffffffffu, acc[c].y, k * LPE);
                acc[c].z += __shfl_down_sync(0xffffffffu, acc[c].z, k * LPE);
                acc[c].w += __shfl_down_sync(0xffffffffu, acc[c].w, k * LPE);
            }
        if (sub == 0) {
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                if (chan_on[c]) *reinterpret_cast<float4*>(part + ci * ld_part + 4 * (lin + c * LPE)) = acc[c];
        }
    }
}

// One block per heavy row: warp w sums the row's chunks w, w+8, w+16, ... in order, the
// eight warp sums are added in warp order through shared memory (a fixed order, so the
// result is deterministic), then the epilogue.  (A single warp walking ~500 chunks per hub
// row was latency-bound: 0.23 ms for 16 hubs.)
__global__ void __launch_bounds__(256) heavy_combine(const AggParams p, const uint32_t* heavy, uint32_t nheavy,
                                                     const uint64_t* chunk_off, const float* part, uint64_t ld_part) {
    __shared__ float4 red[8][32];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    for (uint32_t h = blockIdx.x; h < nheavy; h += gridDim.x) {
        const uint32_t row = heavy[h];
        const uint64_t c0 = chunk_off[h], c1 = chunk_off[h + 1];
        for (uint32_t cb = 0; cb < p.c4; cb += 32) {
            const uint32_t ch = cb + lane;
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ch < p.c4)
                for (uint64_t c = c0 + warp; c < c1; c += 8) add4(r, ld_plain4(part + c * ld_part + 4 * ch));
            red[warp][lane] = r;
            __syncthreads();
            if (warp == 0 && ch < p.c4) {
                float4 t = red[0][lane];
#pragma unroll
                for (int w = 1; w < 8; ++w) add4(t, red[w][lane]);
                epi4(p, row, ch, t);
            }
            __syncthreads();
        }
    }
}

template <int LPE, int NCH>
void launch_heavy(const AggParams& p, const gdx_row_bins* b, uint32_t nchunks, cudaStream_t s) {
    uint64_t blocks = (static_cast<uint64_t>(nchunks) + 7) / 8;
    if (blocks > 65535ull * 64) blocks = 65535ull * 64;
    heavy_chunks<LPE, NCH><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, b->heavy_rows, b->chunk_row, b->chunk_beg,
                                                                         nchunks, b->chunk_edges, b->partial,
                                                                         b->ld_partial);
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
// GDX_AGG_ROWS2: lane groups of half the width, two 16-byte chunks per lane, so twice
// the destination rows (independent row_ptr -> col -> row chains) per warp.
int launch_rows_wide(const AggParams& p, cudaStream_t s) {
    switch (p.c4) {
        case 16: launch_rows<8, 2, true>(p, s); return 0;
        case 12: launch_rows<6, 2, true>(p, s); return 0;
        case 32: launch_rows<16, 2, true>(p, s); return 0;
        case 8: launch_rows<4, 2, true>(p, s); return 0;
        default: return launch_rows_any(p, s);
    }
}

template <int LPE, int NCH, bool EXACT, int UNROLL = 4>
void launch_flat(const AggParams& p, cudaStream_t s) {
    constexpr int EPW = pow2_floor(32 / LPE);
    const uint64_t per_block = 8ull * EPW * (LPE - 1);
    uint64_t blocks = (static_cast<uint64_t>(p.rows) + per_block - 1) / per_block;
    if (blocks > 65535ull * 64) blocks = 65535ull * 64;
    aggregate_flat<LPE, NCH, EXACT, UNROLL><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p);
}

// GDX_AGG_FLAT: edge-flat low-degree kernel where it applies (plain CSR rows, exact
// power-of-two lane groups), the row-group kernel otherwise.
int launch_flat_any(const AggParams& p, cudaStream_t s) {
    if (p.row_end || p.skip_lo || p.row_list) return launch_rows_any(p, s);
    switch (p.c4) {
        case 16: launch_flat<16, 1, true>(p, s); return 0;
        case 8: launch_flat<8, 1, true>(p, s); return 0;
        case 32: launch_flat<32, 1, true>(p, s); return 0;
        case 64: launch_flat<32, 2, true>(p, s); return 0;
        case 12: launch_flat<16, 1, false>(p, s); return 0;
        default: return launch_rows_any(p, s);
    }
}

int launch_variant(const AggParams& p, int variant, cudaStream_t s) {
    if (variant == GDX_AGG_ROWS) return launch_rows_any(p, s);
    if (variant == 3) return launch_flat_any(p, s);
    if (variant == 5 && !p.row_end && !p.skip_lo && !p.row_list && p.c4 == 16) {  // tuning: 8 gathers in flight
        launch_flat<16, 1, true, 8>(p, s);
        return 0;
    }
    if (variant == 6 && !p.row_end && !p.skip_lo && !p.row_list && p.c4 == 16) {  // tuning: 8-lane groups x 2 chunks
        launch_flat<8, 2, true, 4>(p, s);
        return 0;
    }
    if (variant == 2) return launch_rows_wide(p, s);
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
                a->add, a->ld_add, a->relu, a->out, a->ld_out, a->out_hi, a->out_lo, a->ld_split,
                nullptr, a->src_lo8, a->out24_hi, a->out24_lo, a->ld_out24,
                a->ld_src_lo8 ? a->ld_src_lo8 : a->ld_src};
    if (a->src_lo8 || a->out24_hi) {
        // packed-24 rows: widths in whole 8-value groups (8..256, 48 included), 16-byte rows
        GDX_REQUIRE(!a->out24_hi == !a->out24_lo, GDX_INPUT, "gdx_aggregate: out24_hi/out24_lo must pair");
        GDX_REQUIRE(a->width % 8 == 0 && a->ld_src % 8 == 0 && aligned16(a->src) &&
                        (!a->src_lo8 || (reinterpret_cast<uintptr_t>(a->src_lo8) & 7) == 0),
                    GDX_INPUT, "gdx_aggregate: packed-24 rows need width and pitch multiples of 8");
        GDX_REQUIRE(a->src_lo8, GDX_INPUT, "gdx_aggregate: a packed-24 output needs a packed-24 source");
        GDX_REQUIRE(a->ld_src_lo8 % 8 == 0, GDX_INPUT, "gdx_aggregate: ld_src_lo8 must be a multiple of 8");
        GDX_REQUIRE(!a->out24_hi || (a->ld_out24 % 8 == 0 && aligned16(a->out24_hi) &&
                                     (reinterpret_cast<uintptr_t>(a->out24_lo) & 7) == 0),
                    GDX_INPUT, "gdx_aggregate: packed-24 output pitch must be a multiple of 8");
        GDX_REQUIRE((!a->add || (a->ld_add % 4 == 0 && aligned16(a->add))) &&
                        (!a->partial || (a->ld_partial % 4 == 0 && aligned16(a->partial))) &&
                        (!a->out || (a->ld_out % 4 == 0 && aligned16(a->out))),
                    GDX_INPUT, "gdx_aggregate: packed-24 epilogue operands must be 16-byte rows");
        GDX_REQUIRE(variant != GDX_AGG_P24_WIDE ||
                        (a->src_lo8 && a->width == 48 && a->ld_src >= 64 && p.ld_lo8 >= 64),
                    GDX_INPUT, "gdx_aggregate: GDX_AGG_P24_WIDE needs 48-wide packed-24 rows on a 64-column pitch");
        GDX_REQUIRE(launch_p24(p, variant, as_cuda(stream)) == 0, GDX_INPUT,
                    "gdx_aggregate: packed-24 width must be 8, 16, 32, 48, 64, 96, 128 or 256");
        note_launch();
        return check_launch("gdx_aggregate");
    }
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

extern "C" int gdx_pack24(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols, uint16_t* hi,
                          uint8_t* lo, uint64_t ld_dst, gdx_stream stream) {
    GDX_REQUIRE(src && hi && lo, GDX_INPUT, "gdx_pack24: null pointer");
    if (!rows || !cols) return GDX_OK;
    uint64_t blocks = (static_cast<uint64_t>(rows) * cols + 255) / 256;
    if (blocks > static_cast<uint64_t>(gdx::device_sms()) * 16) blocks = static_cast<uint64_t>(gdx::device_sms()) * 16;
    gdx::pack24_kernel<<<static_cast<unsigned>(blocks), 256, 0, gdx::as_cuda(stream)>>>(src, ld_src, rows, cols, hi,
                                                                                        lo, ld_dst);
    gdx::note_launch();
    return gdx::check_launch("gdx_pack24");
}

extern "C" int gdx_unpack24(const uint16_t* hi, const uint8_t* lo, uint64_t ld_src, uint32_t rows, uint32_t cols,
                            float* dst, uint64_t ld_dst, gdx_stream stream) {
    GDX_REQUIRE(hi && lo && dst, GDX_INPUT, "gdx_unpack24: null pointer");
    if (!rows || !cols) return GDX_OK;
    uint64_t blocks = (static_cast<uint64_t>(rows) * cols + 255) / 256;
    if (blocks > static_cast<uint64_t>(gdx::device_sms()) * 16) blocks = static_cast<uint64_t>(gdx::device_sms()) * 16;
    gdx::unpack24_kernel<<<static_cast<unsigned>(blocks), 256, 0, gdx::as_cuda(stream)>>>(hi, lo, ld_src, rows, cols,
                                                                                          dst, ld_dst);
    gdx::note_launch();
    return gdx::check_launch("gdx_unpack24");
}

// ---- degree bins ------------------------------------------------------------------
extern "C" int gdx_row_bins_build(const uint64_t* row_ptr_host, uint32_t rows, uint32_t heavy_degree,
                                  uint32_t chunk_edges, uint32_t max_width, gdx_row_bins** out) {
    GDX_REQUIRE(row_ptr_host && out, GDX_INPUT, "gdx_row_bins_build: null pointer");
    GDX_REQUIRE(heavy_degree >= 1 && chunk_edges >= 32 && max_width >= 1, GDX_INPUT,
                "gdx_row_bins_build: heavy_degree >= 1, chunk_edges >= 32, max_width >= 1");
    *out = nullptr;
    std::vector<uint32_t> light, heavy, crow;
    std::vector<uint64_t> cbeg, coff{0};
    for (uint32_t v = 0; v < rows; ++v) {
        const uint64_t d = row_ptr_host[v + 1] - row_ptr_host[v];
        if (d <= heavy_degree) {
            light.push_back(v);
            continue;
        }
        for (uint64_t e = row_ptr_host[v]; e < row_ptr_host[v + 1]; e += chunk_edges) {
            crow.push_back(static_cast<uint32_t>(heavy.size()));
            cbeg.push_back(e);
        }
        heavy.push_back(v);
        coff.push_back(cbeg.size());
    }
    auto* b = new gdx_row_bins{};
    b->rows = rows;
    b->n_light = static_cast<uint32_t>(light.size());
    b->n_heavy = static_cast<uint32_t>(heavy.size());
    b->n_chunks = static_cast<uint32_t>(cbeg.size());
    b->chunk_edges = chunk_edges;
    b->ld_partial = (static_cast<uint64_t>(max_width) + 3) / 4 * 4;
    auto up = [](auto** dst, const auto& v) -> cudaError_t {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(v.size(), 1) * sizeof(T));
        if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
        return e;
    };
    cudaError_t e = up(&b->light_rows, light);
    if (e == cudaSuccess) e = up(&b->heavy_rows, heavy);
    if (e == cudaSuccess) e = up(&b->chunk_row, crow);
    if (e == cudaSuccess) e = up(&b->chunk_beg, cbeg);
    if (e == cudaSuccess) e = up(&b->chunk_off, coff);
    if (e == cudaSuccess)
        e = cudaMalloc(reinterpret_cast<void**>(&b->partial), std::max<uint64_t>(b->n_chunks, 1) * b->ld_partial * 4);
    b->light_host = new uint32_t[std::max<size_t>(light.size(), 1)];
    b->heavy_host = new uint32_t[std::max<size_t>(heavy.size(), 1)];
    b->chunk_off_host = new uint64_t[coff.size()];
    std::copy(light.begin(), light.end(), b->light_host);
    std::copy(heavy.begin(), heavy.end(), b->heavy_host);
    std::copy(coff.begin(), coff.end(), b->chunk_off_host);
    if (e != cudaSuccess) {
        gdx_row_bins_free(b);
        return gdx::fail(GDX_INTERNAL, std::string("gdx_row_bins_build: ") + cudaGetErrorString(e));
    }
    *out = b;
    return GDX_OK;
}

extern "C" int gdx_row_bins_free(gdx_row_bins* b) {
    if (!b) return GDX_OK;
    cudaFree(b->light_rows);
    cudaFree(b->heavy_rows);
    cudaFree(b->chunk_row);
    cudaFree(b->chunk_beg);
    cudaFree(b->chunk_off);
    cudaFree(b->partial);
    delete[] b->light_host;
    delete[] b->heavy_host;
    delete[] b->chunk_off_host;
    delete b;
    return GDX_OK;
}

extern "C" int gdx_aggregate_balanced(const gdx_aggregate_args* a, int variant, const gdx_row_bins* b,
                                      gdx_stream stream) {
    using namespace gdx;
    if (!b || b->n_heavy == 0) return aggregate_impl(a, variant, stream);
    GDX_REQUIRE(a != nullptr, GDX_INPUT, "gdx_aggregate_balanced: null args");
    GDX_REQUIRE(a->rows <= b->rows, GDX_INPUT, "gdx_aggregate_balanced: more rows than the bins");
    GDX_REQUIRE(!a->src_lo8 && !a->out24_hi, GDX_INPUT, "gdx_aggregate_balanced: fp32 rows only");
    GDX_REQUIRE(a->width % 4 == 0 && a->ld_src % 4 == 0 && (reinterpret_cast<uintptr_t>(a->src) & 15) == 0 &&
                    a->width <= b->ld_partial,
                GDX_INPUT, "gdx_aggregate_balanced: 16-byte rows, width <= the bins' max width");
    if (a->rows == 0) return GDX_OK;
    // rows < a->rows only (a hop prefix): lists are ascending, so prefixes of them
    const uint32_t nl = static_cast<uint32_t>(std::lower_bound(b->light_host, b->light_host + b->n_light, a->rows) -
                                              b->light_host);
    const uint32_t nh = static_cast<uint32_t>(std::lower_bound(b->heavy_host, b->heavy_host + b->n_heavy, a->rows) -
                                              b->heavy_host);
    const uint32_t nc = static_cast<uint32_t>(b->chunk_off_host[nh]);
    cudaStream_t s = as_cuda(stream);
    if (nl) {
        gdx_aggregate_args la = *a;
        la.rows = nl;
        // the light pass reuses aggregate_impl with the row list
        AggParams p{la.row_ptr, la.row_end, la.skip_lo, la.skip_hi, la.partial, la.ld_partial, la.col, nl,
                    la.width / 4, la.src, la.ld_src, static_cast<uint32_t>(la.ld_src * 4), la.self_coef, la.self_base,
                    la.post_scale, la.add, la.ld_add, la.relu, la.out, la.ld_out, la.out_hi, la.out_lo, la.ld_split,
                    b->light_rows, nullptr, nullptr, nullptr, 0};
        if (variant) launch_variant(p, variant, s);
        else pick_and_launch(p, s);
        note_launch();
        if (int rc = check_launch("gdx_aggregate_balanced")) return rc;
    }
    if (nh) {
        AggParams p{a->row_ptr, a->row_end, a->skip_lo, a->skip_hi, a->partial, a->ld_partial, a->col, nh,
                    a->width / 4, a->src, a->ld_src, static_cast<uint32_t>(a->ld_src * 4), a->self_coef, a->self_base,
                    a->post_scale, a->add, a->ld_add, a->relu, a->out, a->ld_out, a->out_hi, a->out_lo, a->ld_split,
                    nullptr, nullptr, nullptr, nullptr, 0};
        const uint32_t c4 = p.c4;
        if (c4 <= 8) launch_heavy<8, 1>(p, b, nc, s);
        else if (c4 <= 16) launch_heavy<16, 1>(p, b, nc, s);
        else if (c4 <= 32) launch_heavy<32, 1>(p, b, nc, s);
        else if (c4 <= 64) launch_heavy<32, 2>(p, b, nc, s);
        else launch_heavy<32, 8>(p, b, nc, s);
        note_launch();
        if (int rc = check_launch("gdx_aggregate_balanced")) return rc;
        const uint64_t blocks = nh < 65535u ? nh : 65535u;
        heavy_combine<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, b->heavy_rows, nh, b->chunk_off, b->partial,
                                                                    b->ld_partial);
        note_launch();
        return check_launch("gdx_aggregate_balanced");
    }
    return GDX_OK;
}
