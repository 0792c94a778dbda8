// cobatch_plan.cu -- the cooperative-batch planner's evaluation step on the device
// for a whole target grouping at once (batch_plan.cpp:28-112 for every group of
// one R of plan_cobatch's scan, :146-180).
//
// The reference builds each batch on the host with O(V) char arrays: the sampled
// closure of the group's targets inside the server universe (batch_closure,
// :28-70), then a back-peel of its MFG layer counts (peel_mfg, :75-101), and it
// rebuilds every batch for every R it tries.  Here all groups of a chunk run
// together: every frontier entry is a (group, vertex) pair, each group has its
// own mark row (mark[group][v]: UNSEEN, or the hop that claimed v, with bit 31
// set once the peel reached v), and every hop / peel step is ONE launch over all
// pairs.  Launch grids are fixed and the kernels read their frontier sizes from
// device memory, so a whole evaluation is enqueued without a host round trip;
// the host synchronises once at the end to read the counts.
//
// Exactness: as in sampling.cu, the candidates a frontier vertex exposes depend
// only on (seed, v) and the group's static candidate mask (universe minus the
// group's own targets), never on claim order, so the claimed sets -- and hence
// the closure and every peel count -- equal the sequential reference's.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <vector>

#include "gdx_common.cuh"

namespace gdx {
namespace {

constexpr uint32_t kPeeled = 0x80000000u;

__device__ __forceinline__ bool cb_candidate(uint32_t u, uint32_t group, const uint8_t* universe,
                                             const uint32_t* group_of) {
    return universe[u] && group_of[u] != group;
}

// Warp-aggregated append of (group, vertex) pairs.
__device__ __forceinline__ void cb_append(bool pred, unsigned long long value, unsigned long long* list,
                                          unsigned long long* counter) {
    const uint32_t mask = __activemask();
    const uint32_t ballot = __ballot_sync(mask, pred);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<unsigned long long>(__popc(ballot)));
    base = __shfl_sync(mask, base, leader);
    if (pred) list[base + __popc(ballot & ((1u << lane) - 1))] = value;
}

__device__ __forceinline__ unsigned long long pair_of(uint32_t gl, uint32_t v) {
    return (static_cast<unsigned long long>(gl) << 32) | v;
}

__global__ void cb_fill(uint32_t* p, uint64_t n, uint32_t value) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = value;
}

// group_of[targets[i]] = group of position i (group_off: device copy of the slices)
__global__ void cb_group_of(const uint32_t* targets, uint64_t nt, const uint64_t* group_off,
                            uint32_t groups, uint32_t* group_of) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nt;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t lo = 0, hi = groups;  // largest g with group_off[g] <= i
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (group_off[mid] <= i) lo = mid;
            else hi = mid;
        }
        group_of[targets[i]] = lo;
    }
}

// Targets of the chunk: mark 0 (hop 0), and the hop-1 frontier = targets with at
// least one candidate neighbour (batch_plan.cpp:37-45).
__global__ void cb_seed(const uint64_t* row_ptr, const uint32_t* col, const uint32_t* targets, uint64_t nt,
                        const uint32_t* group_of, uint32_t g0, const uint8_t* universe, uint64_t n,
                        uint32_t* mark, unsigned long long* frontier, unsigned long long* count) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < nt; i += nw) {
        const uint32_t v = targets[i];
        const uint32_t grp = group_of[v];
        if (lane == 0) mark[static_cast<uint64_t>(grp - g0) * n + v] = 0;
        bool found = false;
        for (uint64_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) {
            if (cb_candidate(col[e], grp, universe, group_of)) found = true;
            if (__any_sync(__activemask(), found)) break;
        }
        found = __any_sync(0xffffffffu, found);
        if (lane == 0 && found) frontier[atomicAdd(count, 1ull)] = pair_of(grp - g0, v);
    }
}

// One hop for every (group, frontier vertex) pair: expose min(fanout, c) of the
// keyed shuffle of the group's candidates (slot replay as in sampling.cu's
// expand_hop), claim unseen ones for the group.
__global__ void __launch_bounds__(256) cb_expand(const uint64_t* row_ptr, const uint32_t* col,
                                                 const uint8_t* universe, const uint32_t* group_of,
                                                 uint32_t g0, uint64_t n,
                                                 const unsigned long long* frontier,
                                                 const unsigned long long* count_in, uint32_t fanout,
                                                 uint64_t seed, uint32_t hop, uint32_t* mark,
                                                 unsigned long long* next, unsigned long long* next_count,
                                                 unsigned long long* sizes) {
    const int lane = threadIdx.x & 31;
    const uint64_t nf = *count_in;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < nf; i += nw) {
        const unsigned long long pr = frontier[i];
        const uint32_t gl = static_cast<uint32_t>(pr >> 32), v = static_cast<uint32_t>(pr);
        const uint32_t grp = g0 + gl;
        uint32_t* gm = mark + static_cast<uint64_t>(gl) * n;
        const uint64_t beg = row_ptr[v], end = row_ptr[v + 1];
        uint32_t c = 0;
        for (uint64_t e0 = beg; e0 < end; e0 += 32) {
            const bool ok = e0 + lane < end && cb_candidate(col[e0 + lane], grp, universe, group_of);
            c += __popc(__ballot_sync(0xffffffffu, ok));
        }
        uint32_t claimed = 0;
        if (fanout == GDX_UNLIMITED_FANOUT || c <= fanout) {
            for (uint64_t e0 = beg; e0 < end; e0 += 32) {
                bool take = false;
                uint32_t u = 0;
                if (e0 + lane < end) {
                    u = col[e0 + lane];
                    if (cb_candidate(u, grp, universe, group_of))
                        take = atomicCAS(&gm[u], GDX_UNSEEN, hop) == GDX_UNSEEN;
                }
                claimed += __popc(__ballot_sync(0xffffffffu, take));
                cb_append(take, pair_of(gl, u), next, next_count);
            }
        } else {
            const uint64_t s0 = keyed_state(seed, v, 0x73616d70ULL);  // "samp", batch_plan.cpp:56
            for (uint32_t t0 = 0; t0 < fanout; t0 += 32) {
                const uint32_t t = t0 + lane;
                uint32_t pos = t;
                if (t < fanout) {
                    for (uint32_t step = 2; step <= c; ++step) {
                        const uint32_t j = static_cast<uint32_t>(below(draw_at(s0, c - step), step));
                        if (pos == step - 1) pos = j;
                        else if (pos == j) pos = step - 1;
                    }
                }
                const bool active = t < fanout;
                uint32_t base = 0, picked = 0;
                bool got = false;
                for (uint64_t e0 = beg; e0 < end; e0 += 32) {
                    const bool ok = e0 + lane < end && cb_candidate(col[e0 + lane], grp, universe, group_of);
                    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                    const uint32_t cntc = __popc(bal);
                    if (active && !got && pos >= base && pos < base + cntc) {
                        picked = col[e0 + __fns(bal, 0, pos - base + 1)];
                        got = true;
                    }
                    base += cntc;
                    if (__all_sync(0xffffffffu, got || !active)) break;
                }
                bool take = false;
                if (active && got) take = atomicCAS(&gm[picked], GDX_UNSEEN, hop) == GDX_UNSEEN;
                claimed += __popc(__ballot_sync(0xffffffffu, take));
                cb_append(take, pair_of(gl, picked), next, next_count);
            }
        }
        if (lane == 0 && claimed) atomicAdd(&sizes[grp], static_cast<unsigned long long>(claimed));
    }
}

// Peel start: the targets are the layer-L set (batch_plan.cpp:83-88).
__global__ void cb_peel_init(const uint32_t* targets, uint64_t nt, const uint32_t* group_of, uint32_t g0,
                             uint64_t n, uint32_t* mark, unsigned long long* frontier,
                             unsigned long long* count) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nt;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t v = targets[i];
        const uint32_t gl = group_of[v] - g0;
        mark[static_cast<uint64_t>(gl) * n + v] |= kPeeled;
        frontier[i] = pair_of(gl, v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = nt;
}

// One back-peel step: in-batch neighbours not yet in the group's set (:89-98).
__global__ void cb_peel_step(const uint64_t* row_ptr, const uint32_t* col, uint64_t n, uint32_t g0,
                             const unsigned long long* frontier, const unsigned long long* count_in,
                             uint32_t* mark, unsigned long long* next, unsigned long long* next_count,
                             unsigned long long* added, uint32_t stride, uint32_t slot) {
    const int lane = threadIdx.x & 31;
    const uint64_t nf = *count_in;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < nf; i += nw) {
        const unsigned long long pr = frontier[i];
        const uint32_t gl = static_cast<uint32_t>(pr >> 32), v = static_cast<uint32_t>(pr);
        uint32_t* gm = mark + static_cast<uint64_t>(gl) * n;
        uint32_t took = 0;
        for (uint64_t e0 = row_ptr[v]; e0 < row_ptr[v + 1]; e0 += 32) {
            bool take = false;
            uint32_t u = 0;
            if (e0 + lane < row_ptr[v + 1]) {
                u = col[e0 + lane];
                const uint32_t m = gm[u];
                if (m != GDX_UNSEEN && !(m & kPeeled)) take = !(atomicOr(&gm[u], kPeeled) & kPeeled);
            }
            took += __popc(__ballot_sync(0xffffffffu, take));
            cb_append(take, pair_of(gl, u), next, next_count);
        }
        if (lane == 0 && took)
            atomicAdd(&added[static_cast<uint64_t>(g0 + gl) * stride + slot], static_cast<unsigned long long>(took));
    }
}

struct InBatch {
    const uint32_t* mark;
    __host__ __device__ bool operator()(uint32_t v) const { return mark[v] != GDX_UNSEEN; }
};

unsigned fixed_grid() { return static_cast<unsigned>(device_sms()) * 8; }

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" int gdx_cobatch_eval(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                                const uint8_t* universe, const uint32_t* targets, const uint64_t* group_off,
                                uint32_t groups, uint32_t max_hop, uint32_t fanout, uint64_t seed,
                                uint32_t layers, uint64_t workspace_bytes, uint64_t* sizes, uint64_t* mfg,
                                uint32_t* vertices, const uint64_t* vertex_off, gdx_stream stream) {
    GDX_REQUIRE(row_ptr && col && universe && group_off && sizes && mfg, GDX_INPUT,
                "gdx_cobatch_eval: null pointer");
    GDX_REQUIRE(groups >= 1, GDX_INPUT, "gdx_cobatch_eval: need at least one group");
    GDX_REQUIRE(!vertices || vertex_off, GDX_INPUT, "gdx_cobatch_eval: vertices need vertex_off");
    const uint64_t nt = group_off[groups];
    GDX_REQUIRE(nt == 0 || targets, GDX_INPUT, "gdx_cobatch_eval: null targets");
    for (uint32_t g = 0; g < groups; ++g)
        GDX_REQUIRE(group_off[g] <= group_off[g + 1], GDX_INPUT, "gdx_cobatch_eval: group_off not ascending");
    cudaStream_t s = as_cuda(stream);
    const uint32_t L1 = layers + 1;
    // chunk of groups evaluated together: mark rows (4 B) + two pair frontiers (16 B) per vertex
    const uint64_t per_group = 20ull * (n ? n : 1);
    uint64_t chunk = workspace_bytes > per_group ? workspace_bytes / per_group : 1;
    if (chunk > groups) chunk = groups;
    uint32_t* group_of = nullptr;
    uint32_t* mark = nullptr;
    unsigned long long* fa = nullptr;
    unsigned long long* fb = nullptr;
    unsigned long long* counters = nullptr;   // [0..1] frontier counts, then sizes[groups], added[groups*L1]
    uint64_t* doff = nullptr;
    const uint64_t ncount = 2 + groups + static_cast<uint64_t>(groups) * L1;
    GDX_CUDA(cudaMallocAsync(&group_of, sizeof(uint32_t) * (n ? n : 1), s));
    GDX_CUDA(cudaMallocAsync(&mark, sizeof(uint32_t) * chunk * (n ? n : 1), s));
    GDX_CUDA(cudaMallocAsync(&fa, sizeof(unsigned long long) * chunk * (n ? n : 1), s));
    GDX_CUDA(cudaMallocAsync(&fb, sizeof(unsigned long long) * chunk * (n ? n : 1), s));
    GDX_CUDA(cudaMallocAsync(&counters, sizeof(unsigned long long) * ncount, s));
    GDX_CUDA(cudaMallocAsync(&doff, sizeof(uint64_t) * (groups + 1), s));
    unsigned long long* cnt = counters;
    unsigned long long* dsizes = counters + 2;
    unsigned long long* added = counters + 2 + groups;
    int rc = GDX_OK;
    auto launched = [&](const char* what) {
        note_launch();
        if (rc == GDX_OK) rc = check_launch(what);
    };
    const unsigned grid = fixed_grid();
    cudaError_t e = cudaMemcpyAsync(doff, group_off, sizeof(uint64_t) * (groups + 1), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * ncount, s);
    if (e != cudaSuccess) rc = fail(GDX_INTERNAL, std::string("gdx_cobatch_eval: ") + cudaGetErrorString(e));
    if (rc == GDX_OK && n) {
        cb_fill<<<grid, 256, 0, s>>>(group_of, n, GDX_UNSEEN);
        launched("gdx_cobatch_eval");
        if (nt) {
            cb_group_of<<<grid, 256, 0, s>>>(targets, nt, doff, groups, group_of);
            launched("gdx_cobatch_eval");
        }
    }
    size_t sel_bytes = 0;
    void* sel_tmp = nullptr;
    if (rc == GDX_OK && vertices && n) {
        thrust::counting_iterator<uint32_t> it(0);
        e = cub::DeviceSelect::If(nullptr, sel_bytes, it, vertices, cnt, static_cast<int64_t>(n),
                                  InBatch{mark}, s);
        if (e == cudaSuccess) e = cudaMallocAsync(&sel_tmp, sel_bytes ? sel_bytes : 16, s);
        if (e != cudaSuccess) rc = fail(GDX_INTERNAL, std::string("gdx_cobatch_eval select: ") + cudaGetErrorString(e));
    }
    for (uint64_t g0 = 0; rc == GDX_OK && n && g0 < groups; g0 += chunk) {
        const uint64_t gc = (g0 + chunk <= groups) ? chunk : groups - g0;
        const uint64_t t0 = group_off[g0], tn = group_off[g0 + gc] - t0;
        cb_fill<<<grid, 256, 0, s>>>(mark, gc * n, GDX_UNSEEN);
        launched("gdx_cobatch_eval");
        if (tn) {
            // closure: targets + max_hop sampled hops (batch_plan.cpp:46-67)
            cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s);
            cb_seed<<<grid, 256, 0, s>>>(row_ptr, col, targets + t0, tn, group_of, static_cast<uint32_t>(g0),
                                         universe, n, mark, fa, cnt);
            launched("gdx_cobatch_eval");
            unsigned long long* cur = fa;
            unsigned long long* nxt = fb;
            for (uint32_t h = 1; h <= max_hop && fanout != 0; ++h) {
                unsigned long long* cin = cnt + ((h - 1) & 1);
                unsigned long long* cout = cnt + (h & 1);
                cudaMemsetAsync(cout, 0, sizeof(unsigned long long), s);
                cb_expand<<<grid, 256, 0, s>>>(row_ptr, col, universe, group_of, static_cast<uint32_t>(g0), n,
                                               cur, cin, fanout, seed, h, mark, nxt, cout, dsizes);
                launched("gdx_cobatch_eval");
                unsigned long long* t = cur;
                cur = nxt;
                nxt = t;
            }
            // MFG peel from the targets over the batch's own vertices (:75-101)
            cb_peel_init<<<grid, 256, 0, s>>>(targets + t0, tn, group_of, static_cast<uint32_t>(g0), n, mark,
                                              fa, cnt);
            launched("gdx_cobatch_eval");
            cur = fa;
            nxt = fb;
            for (uint32_t back = 1; back <= layers; ++back) {
                unsigned long long* cin = cnt + ((back - 1) & 1);
                unsigned long long* cout = cnt + (back & 1);
                cudaMemsetAsync(cout, 0, sizeof(unsigned long long), s);
                cb_peel_step<<<grid, 256, 0, s>>>(row_ptr, col, n, static_cast<uint32_t>(g0), cur, cin, mark,
                                                  nxt, cout, added, L1, layers - back);
                launched("gdx_cobatch_eval");
                unsigned long long* t = cur;
                cur = nxt;
                nxt = t;
            }
        }
        if (vertices) {  // ascending vertex lists of the chunk's batches
            for (uint64_t gl = 0; gl < gc && rc == GDX_OK; ++gl) {
                thrust::counting_iterator<uint32_t> it(0);
                e = cub::DeviceSelect::If(sel_tmp, sel_bytes, it, vertices + vertex_off[g0 + gl], cnt,
                                          static_cast<int64_t>(n), InBatch{mark + gl * n}, s);
                if (e != cudaSuccess) rc = fail(GDX_INTERNAL, std::string("gdx_cobatch_eval select: ") +
                                                                  cudaGetErrorString(e));
                note_launch();
            }
        }
    }
    std::vector<unsigned long long> h(ncount, 0);
    if (rc == GDX_OK) {
        e = cudaMemcpyAsync(h.data(), counters, sizeof(unsigned long long) * ncount, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = fail(GDX_INTERNAL, std::string("gdx_cobatch_eval: ") + cudaGetErrorString(e));
    }
    if (sel_tmp) cudaFreeAsync(sel_tmp, s);
    cudaFreeAsync(doff, s);
    cudaFreeAsync(counters, s);
    cudaFreeAsync(fb, s);
    cudaFreeAsync(fa, s);
    cudaFreeAsync(mark, s);
    cudaFreeAsync(group_of, s);
    if (rc != GDX_OK) return rc;
    for (uint32_t g = 0; g < groups; ++g) {
        const uint64_t t = group_off[g + 1] - group_off[g];
        sizes[g] = t + h[2 + g];
        // counts[L] = targets, counts[L-back] = counts[L-back+1] + added in that step
        uint64_t total = t;
        mfg[static_cast<uint64_t>(g) * L1 + layers] = t;
        for (uint32_t back = 1; back <= layers; ++back) {
            total += h[2 + groups + static_cast<uint64_t>(g) * L1 + (layers - back)];
            mfg[static_cast<uint64_t>(g) * L1 + layers - back] = total;
        }
    }
    return GDX_OK;
}
