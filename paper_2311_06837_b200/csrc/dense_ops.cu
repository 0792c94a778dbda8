// dense_ops.cu -- initialisation (K7), layout and elementwise kernels of the
// training extension (K8): split-bf16 conversion/transposes, ReLU/scale
// backward prep, softmax cross-entropy, degree scales, split-K reduce + SGD.
#include "gdx_common.cuh"

namespace gdx {
namespace {

// make_features / make_layer_weights (reference_gnn.cpp:11-32): draw index
// first + r*cols + c of stream (seed,k1,k2), uniform(lo,hi) in double, then fp32.
__global__ void init_uniform_kernel(uint64_t s0, uint64_t first, uint32_t rows, uint32_t cols,
                                    double lo, double hi, float* out, uint64_t ld) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        const double u = to_unit(draw_at(s0, first + i));
        out[r * ld + c] = static_cast<float>(lo + (hi - lo) * u);
    }
}

__global__ void init_uniform_f64_kernel(uint64_t s0, uint64_t first, uint32_t rows, uint32_t cols,
                                        double lo, double hi, double* out, uint64_t ld) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        out[r * ld + c] = lo + (hi - lo) * to_unit(draw_at(s0, first + i));
    }
}

__global__ void init_labels_kernel(uint64_t seed, uint64_t base, uint32_t rows, uint32_t classes,
                                   int32_t* out) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rows; v += gridDim.x * blockDim.x) {
        const uint64_t s = keyed_state(seed, base + v, 0x6c61626cULL);  // "labl"
        out[v] = static_cast<int32_t>(below(draw_at(s, 0), classes));
    }
}

__global__ void split_kernel(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols,
                             uint16_t* hi, uint16_t* lo, uint64_t ld_dst) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        split_bf16(src[r * ld_src + c], hi[r * ld_dst + c], lo[r * ld_dst + c]);
    }
}

// 32x32 tiles through shared memory so both the read and the write are coalesced.
__global__ void split_transpose_kernel(const float* src, uint64_t ld_src, uint32_t rows,
                                       uint32_t cols, uint16_t* hi, uint16_t* lo, uint64_t ld_dst) {
    __shared__ float tile[32][33];
    const uint32_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t r = r0 + j, c = c0 + threadIdx.x;
        tile[j][threadIdx.x] = (r < rows && c < cols) ? src[static_cast<uint64_t>(r) * ld_src + c] : 0.f;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t c = c0 + j, r = r0 + threadIdx.x;  // dst[c][r]
        if (c < cols && r < rows)
            split_bf16(tile[threadIdx.x][j], hi[static_cast<uint64_t>(c) * ld_dst + r],
                       lo[static_cast<uint64_t>(c) * ld_dst + r]);
    }
}

__global__ void transpose_split_kernel(const uint16_t* shi, const uint16_t* slo, uint64_t ld_src,
                                       uint32_t rows, uint32_t cols, uint16_t* dhi, uint16_t* dlo,
                                       uint64_t ld_dst) {
    __shared__ uint16_t th[32][34];
    __shared__ uint16_t tl[32][34];
    const uint32_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t r = r0 + j, c = c0 + threadIdx.x;
        const bool ok = r < rows && c < cols;
        th[j][threadIdx.x] = ok ? shi[static_cast<uint64_t>(r) * ld_src + c] : 0;
        tl[j][threadIdx.x] = ok ? slo[static_cast<uint64_t>(r) * ld_src + c] : 0;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t c = c0 + j, r = r0 + threadIdx.x;
        if (c < cols && r < rows) {
            dhi[static_cast<uint64_t>(c) * ld_dst + r] = th[threadIdx.x][j];
            dlo[static_cast<uint64_t>(c) * ld_dst + r] = tl[threadIdx.x][j];
        }
    }
}

__global__ void grad_prepare_kernel(const float* dH, uint64_t ld_dh, const float* H, uint64_t ld_h,
                                    uint32_t rows, uint32_t width, const float* dst_scale,
                                    float* g_out, uint64_t ld_gout, float* gs, uint64_t ld_gs,
                                    uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g) {
    const uint64_t total = static_cast<uint64_t>(rows) * width;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / width, c = i % width;
        float g = dH[r * ld_dh + c];
        if (H && !(H[r * ld_h + c] > 0.f)) g = 0.f;
        if (g_out) g_out[r * ld_gout + c] = g;
        if (gs) gs[r * ld_gs + c] = dst_scale ? g * dst_scale[r] : g;
        if (g_hi) split_bf16(g, g_hi[r * ld_g + c], g_lo[r * ld_g + c]);
    }
}

// Vector form: c4 = width/4 threads per row, float4 loads/stores, ushort4 split stores.
__global__ void grad_prepare_vec4(const float* __restrict__ dH, uint64_t ld_dh, const float* __restrict__ H,
                                  uint64_t ld_h, uint32_t rows, uint32_t c4, uint32_t rows_per_block,
                                  const float* __restrict__ dst_scale, float* g_out, uint64_t ld_gout,
                                  float* gs, uint64_t ld_gs, uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g) {
    const uint32_t sub = threadIdx.x / c4, c = threadIdx.x - sub * c4;
    if (sub >= rows_per_block) return;
    for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * rows_per_block + sub; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * rows_per_block) {
        float4 g = *reinterpret_cast<const float4*>(dH + r * ld_dh + 4 * c);
        if (H) {
            const float4 h = __ldg(reinterpret_cast<const float4*>(H + r * ld_h + 4 * c));
            if (!(h.x > 0.f)) g.x = 0.f;
            if (!(h.y > 0.f)) g.y = 0.f;
            if (!(h.z > 0.f)) g.z = 0.f;
            if (!(h.w > 0.f)) g.w = 0.f;
        }
        if (g_out) *reinterpret_cast<float4*>(g_out + r * ld_gout + 4 * c) = g;
        if (gs) {
            const float sc = dst_scale ? dst_scale[r] : 1.f;
            *reinterpret_cast<float4*>(gs + r * ld_gs + 4 * c) = make_float4(g.x * sc, g.y * sc, g.z * sc, g.w * sc);
        }
        if (g_hi) {
            ushort4 hh, ll;
            split_bf16(g.x, hh.x, ll.x);
            split_bf16(g.y, hh.y, ll.y);
            split_bf16(g.z, hh.z, ll.z);
            split_bf16(g.w, hh.w, ll.w);
            *reinterpret_cast<ushort4*>(g_hi + r * ld_g + 4 * c) = hh;
            *reinterpret_cast<ushort4*>(g_lo + r * ld_g + 4 * c) = ll;
        }
    }
}

// One warp per row.  Optional fused outputs of the last layer's backward prep:
// split-bf16 copy of g = dlogits and gs = g * row_scale.
struct PeerDeltas {
    uint32_t n;
    int64_t d[7];
};

__global__ void softmax_xent_kernel(const float* logits, uint64_t ld, uint32_t rows,
                                    uint32_t classes, const int32_t* labels, float inv_count,
                                    float* dlogits, uint64_t ld_d, const float* row_scale, float* gs,
                                    uint64_t ld_gs, uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g,
                                    double* loss_sum, PeerDeltas peers) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    double local = 0.0;
    for (uint32_t r = warp; r < rows; r += nwarps) {
        const float* z = logits + static_cast<uint64_t>(r) * ld;
        float mx = -INFINITY;
        for (uint32_t c = lane; c < classes; c += 32) mx = fmaxf(mx, z[c]);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.f;
        for (uint32_t c = lane; c < classes; c += 32) sum += expf(z[c] - mx);
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const float lse = mx + logf(sum);
        const int32_t y = labels[r];
        const float rs = row_scale ? row_scale[r] : 1.f;
        for (uint32_t c = lane; c < classes; c += 32) {
            const float p = expf(z[c] - lse);
            const float g = (p - (static_cast<int32_t>(c) == y ? 1.f : 0.f)) * inv_count;
            if (dlogits) dlogits[static_cast<uint64_t>(r) * ld_d + c] = g;
            if (gs) {
                float* p = gs + static_cast<uint64_t>(r) * ld_gs + c;
                *p = g * rs;
                for (uint32_t q = 0; q < peers.n; ++q)
                    *reinterpret_cast<float*>(reinterpret_cast<char*>(p) + peers.d[q]) = g * rs;
            }
            if (g_hi) split_bf16(g, g_hi[static_cast<uint64_t>(r) * ld_g + c], g_lo[static_cast<uint64_t>(r) * ld_g + c]);
        }
        if (lane == 0) local += static_cast<double>(lse - z[y]);
    }
    if (lane == 0 && local != 0.0) atomicAdd(loss_sum, local);
}

__global__ void degree_scale_kernel(const uint64_t* row_ptr, uint32_t rows, int kind, float* out) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rows; v += gridDim.x * blockDim.x) {
        const double d = static_cast<double>(row_ptr[v + 1] - row_ptr[v]);
        out[v] = kind == 0 ? (d > 0 ? static_cast<float>(1.0 / d) : 0.f)
                           : static_cast<float>(1.0 / sqrt(d + 1.0));
    }
}

__global__ void splitk_reduce_kernel(const float* ws, uint32_t split_k, uint64_t stride,
                                     uint32_t rows, uint32_t cols, uint64_t ld, float* out,
                                     float* w, float lr, uint16_t* w_hi, uint16_t* w_lo) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols, o = r * ld + c;
        float acc = 0.f;
        for (uint32_t z = 0; z < split_k; ++z) acc += ws[z * stride + o];
        if (out) out[o] = acc;
        if (w) {
            const float nw = w[o] - lr * acc;
            w[o] = nw;
            if (w_hi) split_bf16(nw, w_hi[o], w_lo[o]);
        }
    }
}

// Bandwidth probe (roofline denominators): mode 0 streams the buffer with 16 B
// loads (coalesced), mode 1 gathers random 256 B rows (the fp32 aggregation's access
// pattern without the CSR), mode 2 random 192 B packed-24 rows.  The buffer is L2-resident when it fits.
__global__ void __launch_bounds__(256) probe_kernel(const float4* __restrict__ buf, uint64_t n4,
                                                    uint32_t reps, int mode, float* sink) {
    constexpr int U = 8;  // independent 16 B loads in flight per thread
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    if (mode == 0) {
        for (uint32_t r = 0; r < reps; ++r)
            for (uint64_t i = tid; i + (U - 1) * nthreads < n4; i += U * nthreads) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = __ldcg(buf + i + u * nthreads);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
                }
            }
    } else if (mode == 2) {
        // packed-24 row gathers: random 192-byte rows (a 64-wide packed-24 row), 8 lanes
        // per row, each lane a 16 B load of the u16 plane + an 8 B load of the u8 plane --
        // the access pattern of aggregate_p24 without the CSR.  24 B per thread per load pair;
        // steps rounded up so a thread moves >= reps * bytes / nthreads (the caller counts
        // steps * U * nthreads * 24 bytes).
        // row ids: a 32-bit LCG per 8-lane group mapped onto [0, rows) by a multiply-high
        // (no 64-bit modulo: the probe must stay load-bound, not integer-bound)
        const uint32_t rows = static_cast<uint32_t>(n4 * 16 / 192);
        const int lane8 = threadIdx.x & 7;
        const char* base = reinterpret_cast<const char*>(buf);
        uint32_t h = static_cast<uint32_t>(tid >> 3) * 2654435761u + 12345u;
        const uint64_t per = static_cast<uint64_t>(U) * nthreads * 24;
        const uint64_t steps = (reps * n4 * 16 + per - 1) / per;
        for (uint64_t k = 0; k < steps; ++k) {
            uint4 v[U];
            uint2 w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                h = h * 1664525u + 1013904223u;
                const char* r = base + static_cast<uint64_t>(__umulhi(h, rows)) * 192;
                v[u] = __ldcg(reinterpret_cast<const uint4*>(r + 16 * lane8));
                w[u] = __ldcg(reinterpret_cast<const uint2*>(r + 128 + 8 * lane8));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc.x += __uint_as_float(v[u].x ^ w[u].x);
                acc.y += __uint_as_float(v[u].y ^ w[u].y);
                acc.z += __uint_as_float(v[u].z);
                acc.w += __uint_as_float(v[u].w);
            }
        }
    } else {
        const uint64_t rows = n4 / 16;  // 256-byte rows, 16 lanes per row
        const int lane16 = threadIdx.x & 15;
        uint64_t h = (tid >> 4) * 0x9e3779b97f4a7c15ULL + 1;
        const uint64_t steps = reps * (n4 / nthreads) / U;
        for (uint64_t k = 0; k < steps; ++k) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                h = h * 6364136223846793005ULL + 1442695040888963407ULL;
                v[u] = __ldcg(buf + ((h >> 33) % rows) * 16 + lane16);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
            }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.678f) sink[0] = acc.x;
}

unsigned grid_for(uint64_t total, unsigned block = 256) {
    uint64_t b = (total + block - 1) / block;
    const uint64_t cap = static_cast<uint64_t>(device_sms()) * 16;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b ? b : 1);
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" int gdx_init_uniform(uint64_t seed, uint64_t k1, uint64_t k2, uint64_t first_draw,
                                uint32_t rows, uint32_t cols, double lo, double hi, float* out,
                                uint64_t ld, gdx_stream stream) {
    GDX_REQUIRE(out || rows * static_cast<uint64_t>(cols) == 0, GDX_INPUT, "gdx_init_uniform: null out");
    GDX_REQUIRE(ld >= cols, GDX_INPUT, "gdx_init_uniform: ld < cols");
    if (!rows || !cols) return GDX_OK;
    init_uniform_kernel<<<grid_for(static_cast<uint64_t>(rows) * cols), 256, 0, as_cuda(stream)>>>(
        keyed_state(seed, k1, k2), first_draw, rows, cols, lo, hi, out, ld);
    note_launch();
    return check_launch("gdx_init_uniform");
}

extern "C" int gdx_init_uniform_f64(uint64_t seed, uint64_t k1, uint64_t k2, uint64_t first_draw,
                                    uint32_t rows, uint32_t cols, double lo, double hi, double* out,
                                    uint64_t ld, gdx_stream stream) {
    GDX_REQUIRE(out || rows * static_cast<uint64_t>(cols) == 0, GDX_INPUT, "gdx_init_uniform_f64: null out");
    GDX_REQUIRE(ld >= cols, GDX_INPUT, "gdx_init_uniform_f64: ld < cols");
    if (!rows || !cols) return GDX_OK;
    init_uniform_f64_kernel<<<grid_for(static_cast<uint64_t>(rows) * cols), 256, 0, as_cuda(stream)>>>(
        keyed_state(seed, k1, k2), first_draw, rows, cols, lo, hi, out, ld);
    note_launch();
    return check_launch("gdx_init_uniform_f64");
}

extern "C" int gdx_init_labels(uint64_t seed, uint64_t base, uint32_t rows, uint32_t classes,
                               int32_t* out, gdx_stream stream) {
    GDX_REQUIRE(classes > 0, GDX_INPUT, "gdx_init_labels: classes must be >= 1");
    if (!rows) return GDX_OK;
    init_labels_kernel<<<grid_for(rows), 256, 0, as_cuda(stream)>>>(seed, base, rows, classes, out);
    note_launch();
    return check_launch("gdx_init_labels");
}

extern "C" int gdx_split_bf16(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols,
                              uint16_t* hi, uint16_t* lo, uint64_t ld_dst, int transpose,
                              gdx_stream stream) {
    GDX_REQUIRE(src && hi && lo, GDX_INPUT, "gdx_split_bf16: null pointer");
    GDX_REQUIRE(ld_src >= cols && ld_dst >= (transpose ? rows : cols), GDX_INPUT,
                "gdx_split_bf16: leading dimension too small");
    if (!rows || !cols) return GDX_OK;
    if (transpose) {
        dim3 blk(32, 8), grid((cols + 31) / 32, (rows + 31) / 32);
        split_transpose_kernel<<<grid, blk, 0, as_cuda(stream)>>>(src, ld_src, rows, cols, hi, lo, ld_dst);
    } else {
        split_kernel<<<grid_for(static_cast<uint64_t>(rows) * cols), 256, 0, as_cuda(stream)>>>(
            src, ld_src, rows, cols, hi, lo, ld_dst);
    }
    note_launch();
    return check_launch("gdx_split_bf16");
}

extern "C" int gdx_transpose_split(const uint16_t* src_hi, const uint16_t* src_lo, uint64_t ld_src,
                                   uint32_t rows, uint32_t cols, uint16_t* dst_hi, uint16_t* dst_lo,
                                   uint64_t ld_dst, gdx_stream stream) {
    GDX_REQUIRE(src_hi && src_lo && dst_hi && dst_lo, GDX_INPUT, "gdx_transpose_split: null pointer");
    GDX_REQUIRE(ld_src >= cols && ld_dst >= rows, GDX_INPUT, "gdx_transpose_split: leading dimension too small");
    if (!rows || !cols) return GDX_OK;
    dim3 blk(32, 8), grid((cols + 31) / 32, (rows + 31) / 32);
    transpose_split_kernel<<<grid, blk, 0, as_cuda(stream)>>>(src_hi, src_lo, ld_src, rows, cols,
                                                               dst_hi, dst_lo, ld_dst);
    note_launch();
    return check_launch("gdx_transpose_split");
}

extern "C" int gdx_grad_prepare(const float* dH, uint64_t ld_dh, const float* H, uint64_t ld_h,
                                uint32_t rows, uint32_t width, const float* dst_scale, float* g_out,
                                uint64_t ld_gout, float* gs, uint64_t ld_gs, uint16_t* g_hi,
                                uint16_t* g_lo, uint64_t ld_g, gdx_stream stream) {
    GDX_REQUIRE(dH, GDX_INPUT, "gdx_grad_prepare: null dH");
    GDX_REQUIRE(!g_hi == !g_lo, GDX_INPUT, "gdx_grad_prepare: g_hi/g_lo must pair");
    if (!rows || !width) return GDX_OK;
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    auto a8 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 7) == 0; };
    const bool vec = width % 4 == 0 && width <= 1024 && ld_dh % 4 == 0 && a16(dH) &&
                     (!H || (ld_h % 4 == 0 && a16(H))) && (!g_out || (ld_gout % 4 == 0 && a16(g_out))) &&
                     (!gs || (ld_gs % 4 == 0 && a16(gs))) && (!g_hi || (ld_g % 4 == 0 && a8(g_hi) && a8(g_lo)));
    if (vec) {
        const uint32_t c4 = width / 4, rpb = 256 / c4;
        const uint64_t blocks = (static_cast<uint64_t>(rows) + rpb - 1) / rpb;
        grad_prepare_vec4<<<static_cast<unsigned>(blocks < 65535ull * 32 ? blocks : 65535ull * 32), 256, 0,
                            as_cuda(stream)>>>(dH, ld_dh, H, ld_h, rows, c4, rpb, dst_scale, g_out, ld_gout,
                                               gs, ld_gs, g_hi, g_lo, ld_g);
    } else {
        grad_prepare_kernel<<<grid_for(static_cast<uint64_t>(rows) * width), 256, 0, as_cuda(stream)>>>(
            dH, ld_dh, H, ld_h, rows, width, dst_scale, g_out, ld_gout, gs, ld_gs, g_hi, g_lo, ld_g);
    }
    note_launch();
    return check_launch("gdx_grad_prepare");
}

// Vector form for classes <= 4*GL: GL lanes per row (32/GL rows per warp), 4 logits
// per lane held in registers, group-local shuffles; float4 / ushort4 stores.  Padding
// columns (classes .. 4*GL) get g = 0.
template <int GL>
__global__ void __launch_bounds__(256) softmax_xent_vec(const float* __restrict__ logits, uint64_t ld,
                                                        uint32_t rows, uint32_t classes,
                                                        const int32_t* __restrict__ labels, float inv_count,
                                                        const float* __restrict__ row_scale, float* gs,
                                                        uint64_t ld_gs, uint16_t* g_hi, uint16_t* g_lo,
                                                        uint64_t ld_g, uint32_t out_cols, double* loss_sum,
                                                        uint16_t* gs24_hi, uint8_t* gs24_lo, uint64_t ld24_hi,
                                                        uint64_t ld24_lo) {
    constexpr int RPW = 32 / GL;
    const int lane = threadIdx.x & 31;
    const int sub = lane / GL, gl = lane - sub * GL;
    const uint32_t c0 = 4 * gl;
    const unsigned gmask = (GL == 32) ? 0xffffffffu : (((1u << GL) - 1u) << (sub * GL));
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * RPW;
    double local = 0.0;
    for (uint64_t r = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RPW + sub; r < rows;
         r += groups) {
        float z[4];
        const float* zr = logits + r * ld;
        if (c0 + 4 <= classes) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(zr + c0));
            z[0] = q.x; z[1] = q.y; z[2] = q.z; z[3] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) z[j] = (c0 + j < classes) ? zr[c0 + j] : -INFINITY;
        }
        float mx = fmaxf(fmaxf(z[0], z[1]), fmaxf(z[2], z[3]));
#pragma unroll
        for (int o = GL / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o));
        float e[4], sum = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            e[j] = (c0 + j < classes) ? expf(z[j] - mx) : 0.f;
            sum += e[j];
        }
#pragma unroll
        for (int o = GL / 2; o; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o);
        const float inv = 1.f / sum;
        const int32_t y = labels[r];
        const float rs = row_scale ? row_scale[r] : 1.f;
        float g[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            g[j] = (c0 + j < classes) ? (e[j] * inv - (static_cast<int32_t>(c0 + j) == y ? 1.f : 0.f)) * inv_count
                                      : 0.f;
        if (c0 < out_cols) {
            if (gs)
                *reinterpret_cast<float4*>(gs + r * ld_gs + c0) = make_float4(g[0] * rs, g[1] * rs, g[2] * rs, g[3] * rs);
            if (gs24_hi) {  // gs as packed-24 rows (interleaved planes, trainer.cu Mat::p24)
                ushort4 hh;
                uchar4 ll;
                pack24(g[0] * rs, hh.x, ll.x);
                pack24(g[1] * rs, hh.y, ll.y);
                pack24(g[2] * rs, hh.z, ll.z);
                pack24(g[3] * rs, hh.w, ll.w);
                *reinterpret_cast<ushort4*>(gs24_hi + r * ld24_hi + c0) = hh;
                *reinterpret_cast<uchar4*>(gs24_lo + r * ld24_lo + c0) = ll;
            }
            if (g_hi) {
                ushort4 hh, ll;
                split_bf16(g[0], hh.x, ll.x);
                split_bf16(g[1], hh.y, ll.y);
                split_bf16(g[2], hh.z, ll.z);
                split_bf16(g[3], hh.w, ll.w);
                *reinterpret_cast<ushort4*>(g_hi + r * ld_g + c0) = hh;
                *reinterpret_cast<ushort4*>(g_lo + r * ld_g + c0) = ll;
            }
        }
        // loss: lse - z[y], by the lane holding column y
        if (static_cast<uint32_t>(y) >= c0 && static_cast<uint32_t>(y) < c0 + 4)
            local += static_cast<double>(mx + logf(sum) - z[y - c0]);
    }
    // one atomic per warp (per-row atomics on one address serialise)
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if (lane == 0 && local != 0.0) atomicAdd(loss_sum, local);
}

// launches the vector form when the shapes allow; returns false otherwise
bool softmax_vec_launch(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes, const int32_t* labels,
                        float inv_count, float* dlogits, const float* row_scale, float* gs, uint64_t ld_gs,
                        uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g, double* loss_sum, uint32_t npeers,
                        cudaStream_t st, uint16_t* gs24_hi = nullptr, uint8_t* gs24_lo = nullptr,
                        uint64_t ld24_hi = 0, uint64_t ld24_lo = 0) {
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    auto a8 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 7) == 0; };
    if (dlogits || npeers || classes > 128 || ld % 4 || !a16(logits)) return false;
    const uint32_t cols = (classes + 3) / 4 * 4;  // whole float4 groups written
    if (gs && (ld_gs % 4 || !a16(gs) || ld_gs < cols)) return false;
    if (g_hi && (ld_g % 4 || !a8(g_hi) || !a8(g_lo) || ld_g < cols)) return false;
    if (gs24_hi && (ld24_hi % 4 || ld24_lo % 4 || !a8(gs24_hi) || (reinterpret_cast<uintptr_t>(gs24_lo) & 3) ||
                    ld24_hi < cols || ld24_lo < cols))
        return false;
    const uint64_t rpb = classes <= 64 ? 16 : 8;  // rows per 256-thread block and step
    // grid-stride with a bounded grid: the loss is one fp64 atomic per warp, and
    // ~10^6 atomics on one address would serialise
    uint64_t blocks = (static_cast<uint64_t>(rows) + rpb - 1) / rpb;
    if (blocks > static_cast<uint64_t>(device_sms()) * 8) blocks = static_cast<uint64_t>(device_sms()) * 8;
    if (classes <= 64)
        softmax_xent_vec<16><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
            logits, ld, rows, classes, labels, inv_count, row_scale, gs, ld_gs, g_hi, g_lo, ld_g, cols, loss_sum,
            gs24_hi, gs24_lo, ld24_hi, ld24_lo);
    else
        softmax_xent_vec<32><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
            logits, ld, rows, classes, labels, inv_count, row_scale, gs, ld_gs, g_hi, g_lo, ld_g, cols, loss_sum,
            gs24_hi, gs24_lo, ld24_hi, ld24_lo);
    return true;
}

extern "C" int gdx_softmax_xent(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                                const int32_t* labels, float inv_count, float* dlogits,
                                uint64_t ld_d, double* loss_sum, gdx_stream stream) {
    GDX_REQUIRE(logits && labels && dlogits && loss_sum, GDX_INPUT, "gdx_softmax_xent: null pointer");
    GDX_REQUIRE(classes >= 1, GDX_INPUT, "gdx_softmax_xent: classes must be >= 1");
    if (!rows) return GDX_OK;
    const uint64_t threads = static_cast<uint64_t>(rows) * 32;
    softmax_xent_kernel<<<grid_for(threads), 256, 0, as_cuda(stream)>>>(
        logits, ld, rows, classes, labels, inv_count, dlogits, ld_d, nullptr, nullptr, 0, nullptr,
        nullptr, 0, loss_sum, PeerDeltas{});
    note_launch();
    return check_launch("gdx_softmax_xent");
}

extern "C" int gdx_softmax_xent_fused(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                                      const int32_t* labels, float inv_count, float* dlogits,
                                      uint64_t ld_d, const float* row_scale, float* gs, uint64_t ld_gs,
                                      uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g, double* loss_sum,
                                      gdx_stream stream) {
    GDX_REQUIRE(logits && labels && loss_sum, GDX_INPUT, "gdx_softmax_xent_fused: null pointer");
    GDX_REQUIRE(!g_hi == !g_lo, GDX_INPUT, "gdx_softmax_xent_fused: g_hi/g_lo must pair");
    GDX_REQUIRE(classes >= 1, GDX_INPUT, "gdx_softmax_xent_fused: classes must be >= 1");
    if (!rows) return GDX_OK;
    if (!softmax_vec_launch(logits, ld, rows, classes, labels, inv_count, dlogits, row_scale, gs, ld_gs, g_hi,
                            g_lo, ld_g, loss_sum, 0, as_cuda(stream))) {
        const uint64_t threads = static_cast<uint64_t>(rows) * 32;
        softmax_xent_kernel<<<grid_for(threads), 256, 0, as_cuda(stream)>>>(
            logits, ld, rows, classes, labels, inv_count, dlogits, ld_d, row_scale, gs, ld_gs, g_hi, g_lo,
            ld_g, loss_sum, PeerDeltas{});
    }
    note_launch();
    return check_launch("gdx_softmax_xent_fused");
}

extern "C" int gdx_softmax_xent_fused_p24(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                                          const int32_t* labels, float inv_count, const float* row_scale,
                                          uint16_t* gs_hi24, uint64_t ld_hi24, uint8_t* gs_lo8, uint64_t ld_lo8,
                                          uint16_t* g_hi,
                                          uint16_t* g_lo, uint64_t ld_g, double* loss_sum, gdx_stream stream) {
    GDX_REQUIRE(logits && labels && loss_sum && gs_hi24 && gs_lo8, GDX_INPUT,
                "gdx_softmax_xent_fused_p24: null pointer");
    GDX_REQUIRE(!g_hi == !g_lo, GDX_INPUT, "gdx_softmax_xent_fused_p24: g_hi/g_lo must pair");
    GDX_REQUIRE(classes >= 1, GDX_INPUT, "gdx_softmax_xent_fused_p24: classes must be >= 1");
    if (!rows) return GDX_OK;
    GDX_REQUIRE(softmax_vec_launch(logits, ld, rows, classes, labels, inv_count, nullptr, row_scale, nullptr, 0, g_hi,
                                   g_lo, ld_g, loss_sum, 0, as_cuda(stream), gs_hi24, gs_lo8, ld_hi24, ld_lo8),
                GDX_INPUT,
                "gdx_softmax_xent_fused_p24: needs classes <= 128, 16-byte logits rows and packed-24 pitches "
                "(multiples of 4, >= classes rounded to 4)");
    note_launch();
    return check_launch("gdx_softmax_xent_fused_p24");
}

extern "C" int gdx_softmax_xent_fused_peers(const float* logits, uint64_t ld, uint32_t rows,
                                            uint32_t classes, const int32_t* labels, float inv_count,
                                            const float* row_scale, float* gs, uint64_t ld_gs,
                                            uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g,
                                            double* loss_sum, uint32_t npeers,
                                            const int64_t* gs_peer_delta, gdx_stream stream) {
    GDX_REQUIRE(logits && labels && loss_sum && gs, GDX_INPUT, "gdx_softmax_xent_fused_peers: null pointer");
    GDX_REQUIRE(npeers <= 7 && (npeers == 0 || gs_peer_delta), GDX_INPUT,
                "gdx_softmax_xent_fused_peers: at most 7 peers");
    GDX_REQUIRE(!g_hi == !g_lo, GDX_INPUT, "gdx_softmax_xent_fused_peers: g_hi/g_lo must pair");
    if (!rows) return GDX_OK;
    PeerDeltas pd{npeers, {}};
    for (uint32_t r = 0; r < npeers; ++r) pd.d[r] = gs_peer_delta[r];
    const uint64_t threads = static_cast<uint64_t>(rows) * 32;
    softmax_xent_kernel<<<grid_for(threads), 256, 0, as_cuda(stream)>>>(
        logits, ld, rows, classes, labels, inv_count, nullptr, 0, row_scale, gs, ld_gs, g_hi, g_lo, ld_g,
        loss_sum, pd);
    note_launch();
    return check_launch("gdx_softmax_xent_fused_peers");
}

extern "C" int gdx_degree_scale(const uint64_t* row_ptr, uint32_t rows, int kind, float* out,
                                gdx_stream stream) {
    GDX_REQUIRE(row_ptr && out, GDX_INPUT, "gdx_degree_scale: null pointer");
    if (!rows) return GDX_OK;
    degree_scale_kernel<<<grid_for(rows), 256, 0, as_cuda(stream)>>>(row_ptr, rows, kind, out);
    note_launch();
    return check_launch("gdx_degree_scale");
}

extern "C" int gdx_splitk_reduce(const float* ws, uint32_t split_k, uint64_t stride, uint32_t rows,
                                 uint32_t cols, uint64_t ld, float* out, float* w, float lr,
                                 uint16_t* w_hi, uint16_t* w_lo, gdx_stream stream) {
    GDX_REQUIRE(ws && split_k >= 1, GDX_INPUT, "gdx_splitk_reduce: bad workspace");
    GDX_REQUIRE(!w_hi == !w_lo, GDX_INPUT, "gdx_splitk_reduce: w_hi/w_lo must pair");
    if (!rows || !cols) return GDX_OK;
    splitk_reduce_kernel<<<grid_for(static_cast<uint64_t>(rows) * cols), 256, 0, as_cuda(stream)>>>(
        ws, split_k, stride, rows, cols, ld, out, w, lr, w_hi, w_lo);
    note_launch();
    return check_launch("gdx_splitk_reduce");
}

extern "C" int gdx_probe_bandwidth(const float* buf, uint64_t bytes, uint32_t reps, int mode,
                                   float* sink, gdx_stream stream) {
    GDX_REQUIRE(buf && sink && bytes >= 4096 && (bytes % 4096) == 0, GDX_INPUT,
                "gdx_probe_bandwidth: need a 4 KiB-multiple buffer");
    probe_kernel<<<device_sms() * 8, 256, 0, as_cuda(stream)>>>(reinterpret_cast<const float4*>(buf), bytes / 16,
                                                           reps, mode, sink);
    note_launch();
    return check_launch("gdx_probe_bandwidth");
}

// L2 persistence for the gathered matrix of the next aggregation: an access-policy
// window on the stream (kernel nodes captured into a CUDA graph inherit it).
// bytes == 0 clears the window.  The persisting carve-out is set once, on first use.
extern "C" int gdx_set_l2_window(const void* base, uint64_t bytes, float hit_ratio, gdx_stream stream) {
    static bool carved = false;
    cudaStream_t s = as_cuda(stream);
    if (bytes && !carved) {
        int dev = 0, maxp = 0;
        GDX_CUDA(cudaGetDevice(&dev));
        GDX_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
        if (maxp > 0) GDX_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(maxp)));
        carved = true;
    }
    cudaStreamAttrValue v{};
    if (bytes) {
        int dev = 0, maxw = 0;
        GDX_CUDA(cudaGetDevice(&dev));
        GDX_CUDA(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
        v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
        v.accessPolicyWindow.num_bytes = bytes < static_cast<uint64_t>(maxw) ? bytes : static_cast<uint64_t>(maxw);
        v.accessPolicyWindow.hitRatio = hit_ratio;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
        v.accessPolicyWindow.num_bytes = 0;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
        v.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    }
    GDX_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
    return GDX_OK;
}
