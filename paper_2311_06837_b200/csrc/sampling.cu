// sampling.cu -- K4/K5/K6: expansion-aware boundary sampling, closure BFS,
// induced-edge counting, MFG peeling, cooperative split and the local
// (hop-ordered) CSR of a dependency subgraph.  Integer work, bit-exact.
//
// Why a parallel version is exact: in extract_sampled (extract.cpp:135-182)
// and batch_closure (batch_plan.cpp:28-70) the edges a frontier vertex
// exposes depend only on (seed, v) and the static candidate mask, never on
// which vertices were taken earlier, so the set of vertices first taken at
// hop h is independent of the order frontier vertices are visited.  Each hop
// is one kernel: a warp per frontier vertex, claims by atomicCAS(UNSEEN -> h).
//
// The Fisher-Yates prefix (rng.hpp:55-61, extract.cpp:120-131) is replayed
// per OUTPUT slot: lane t follows slot t backwards through the swap sequence
// (swap i exchanges positions i-1 and j_i = below(draw_{c-i}, i)), which gives
// the original candidate index that ends in slot t without materialising the
// shuffled list.  Candidates are then selected by rank with warp ballots.
#include <cub/device/device_scan.cuh>

#include <vector>

#include "gdx_common.cuh"

namespace gdx {
namespace {

__device__ __forceinline__ bool is_candidate(uint32_t u, const uint8_t* excluded,
                                             const uint8_t* allowed) {
    return !excluded[u] && (!allowed || allowed[u]);
}

// Warp-aggregated append to a device list.
__device__ __forceinline__ void warp_append(bool pred, uint32_t value, uint32_t* list,
                                            uint32_t* counter) {
    const uint32_t mask = __activemask();
    const uint32_t ballot = __ballot_sync(mask, pred);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(ballot));
    base = __shfl_sync(mask, base, leader);
    if (pred) list[base + __popc(ballot & ((1u << lane) - 1))] = value;
}

// hop-1 frontier: excluded vertices with at least one candidate neighbour
__global__ void seed_frontier(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                              const uint8_t* excluded, const uint8_t* allowed, uint32_t* frontier,
                              uint32_t* count) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        bool found = false;
        if (excluded[v]) {
            for (uint64_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) {
                if (is_candidate(col[e], excluded, allowed)) found = true;
                if (__any_sync(__activemask(), found)) break;
            }
            found = __any_sync(0xffffffffu, found);
        }
        if (lane == 0 && found) frontier[atomicAdd(count, 1u)] = v;
    }
}

// One hop of sampled growth.  frontier[i] exposes min(fanout, c) candidates.
__global__ void __launch_bounds__(256) expand_hop(const uint64_t* row_ptr, const uint32_t* col,
                                                  const uint8_t* excluded, const uint8_t* allowed,
                                                  const uint32_t* frontier, const uint32_t* count_in,
                                                  uint32_t fanout, uint64_t seed, uint32_t hop,
                                                  uint32_t* mark, uint32_t* next,
                                                  uint32_t* next_count) {
    const int lane = threadIdx.x & 31;
    const uint32_t nf = *count_in;  // frontier size from device memory: no host round trip per hop
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nf; i += nw) {
        const uint32_t v = frontier[i];
        const uint64_t beg = row_ptr[v], end = row_ptr[v + 1];
        // c = number of candidates
        uint32_t c = 0;
        for (uint64_t e0 = beg; e0 < end; e0 += 32) {
            const bool ok = e0 + lane < end && is_candidate(col[e0 + lane], excluded, allowed);
            c += __popc(__ballot_sync(0xffffffffu, ok));
        }
        if (fanout == GDX_UNLIMITED_FANOUT || c <= fanout) {
            // every candidate is exposed (no shuffle drawn, extract.cpp:126)
            for (uint64_t e0 = beg; e0 < end; e0 += 32) {
                bool take = false;
                uint32_t u = 0;
                if (e0 + lane < end) {
                    u = col[e0 + lane];
                    if (is_candidate(u, excluded, allowed))
                        take = atomicCAS(&mark[u], GDX_UNSEEN, hop) == GDX_UNSEEN;
                }
                warp_append(take, u, next, next_count);
            }
            continue;
        }
        const uint64_t s0 = keyed_state(seed, v, 0x73616d70ULL);  // "samp"
        for (uint32_t t0 = 0; t0 < fanout; t0 += 32) {
            // replay the swap sequence backwards for slot t = t0 + lane
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
            // select the pos-th candidate (ascending neighbour order)
            uint32_t base = 0, picked = 0;
            bool got = false;
            for (uint64_t e0 = beg; e0 < end; e0 += 32) {
                const bool ok = e0 + lane < end && is_candidate(col[e0 + lane], excluded, allowed);
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                const uint32_t cntc = __popc(bal);
                if (active && !got && pos >= base && pos < base + cntc) {
                    const int which = __fns(bal, 0, pos - base + 1);
                    picked = col[e0 + which];
                    got = true;
                }
                base += cntc;
                if (__all_sync(0xffffffffu, got || !active)) break;
            }
            bool take = false;
            if (active && got) take = atomicCAS(&mark[picked], GDX_UNSEEN, hop) == GDX_UNSEEN;
            warp_append(take, picked, next, next_count);
        }
    }
}

__global__ void induced_count_kernel(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                                     const uint32_t* mark, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long local = 0;
    for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        if (mark[v] == GDX_UNSEEN) continue;
        for (uint64_t e0 = row_ptr[v]; e0 < row_ptr[v + 1]; e0 += 32) {
            const bool ok = e0 + lane < row_ptr[v + 1] && mark[col[e0 + lane]] != GDX_UNSEEN;
            local += __popc(__ballot_sync(0xffffffffu, ok));
        }
    }
    if (lane == 0 && local) atomicAdd(out, local);
}

__global__ void peel_init(const uint32_t* targets, uint64_t nt, uint32_t* in_set, uint32_t* frontier) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nt;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        in_set[targets[i]] = 1;
        frontier[i] = targets[i];
    }
}

__global__ void peel_step(const uint64_t* row_ptr, const uint32_t* col, const uint8_t* in_batch,
                          const uint32_t* frontier, const uint32_t* count_in, uint32_t* in_set, uint32_t* next,
                          uint32_t* next_count) {
    const int lane = threadIdx.x & 31;
    const uint32_t nf = *count_in;  // frontier size from device memory
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nf; i += nw) {
        const uint32_t v = frontier[i];
        for (uint64_t e0 = row_ptr[v]; e0 < row_ptr[v + 1]; e0 += 32) {
            bool take = false;
            uint32_t u = 0;
            if (e0 + lane < row_ptr[v + 1]) {
                u = col[e0 + lane];
                if (in_batch[u] && !in_set[u]) take = atomicExch(&in_set[u], 1u) == 0u;
            }
            warp_append(take, u, next, next_count);
        }
    }
}

// split_batch: flags, inner counts per GPU
__global__ void split_classify(const uint32_t* bv, uint64_t nb, const uint32_t* sp, const uint32_t* gp,
                               uint32_t server, uint32_t gpus, uint32_t* share_of, uint32_t* halo_flag,
                               unsigned long long* inner_counts) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nb;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t v = bv[i];
        if (sp[v] == server) {
            const uint32_t w = gp[v] - server * gpus;
            share_of[i] = w;
            halo_flag[i] = 0;
            atomicAdd(&inner_counts[w], 1ull);
        } else {
            halo_flag[i] = 1;
        }
    }
}

// halo rank j -> j-th slot in (level, gpu) order, slots (l, w) for l >= s_w
__global__ void split_assign(uint64_t nb, uint32_t gpus, const uint32_t* halo_flag,
                             const uint64_t* halo_rank, const unsigned long long* inner_counts,
                             uint32_t* share_of) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nb;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!halo_flag[i]) continue;
        const uint64_t j = halo_rank[i];
        uint64_t smin = ~0ull;
        for (uint32_t w = 0; w < gpus; ++w) smin = min(smin, static_cast<uint64_t>(inner_counts[w]));
        // cnt(l) = sum_w max(0, l - s_w): slots strictly below level l
        auto cnt = [&](uint64_t l) {
            uint64_t t = 0;
            for (uint32_t w = 0; w < gpus; ++w) {
                const uint64_t s = inner_counts[w];
                if (l > s) t += l - s;
            }
            return t;
        };
        uint64_t lo = smin, hi = smin + j + 1;  // cnt(lo) <= j < cnt(hi)
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (cnt(mid) <= j) lo = mid;
            else hi = mid;
        }
        uint64_t k = j - cnt(lo);
        for (uint32_t w = 0; w < gpus; ++w) {
            if (inner_counts[w] <= lo) {
                if (k == 0) {
                    share_of[i] = w;
                    break;
                }
                --k;
            }
        }
    }
}

__global__ void hop_flags(const uint32_t* hop, uint32_t n, uint32_t h, uint32_t* flag) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        flag[v] = hop[v] == h;
}

__global__ void hop_scatter(const uint32_t* hop, uint32_t n, uint32_t h, const uint32_t* rank,
                            uint32_t base, uint32_t* l2g, uint32_t* local_of) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (hop[v] == h) {
            const uint32_t l = base + rank[v];
            l2g[l] = v;
            local_of[v] = l;
        }
    }
}

__global__ void fill_u32(uint32_t* p, uint64_t n, uint32_t value) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = value;
}

// Rows of the local CSR: the global row filtered to subgraph members, order kept.
__global__ void local_csr_kernel(const uint64_t* row_ptr, const uint32_t* col, const uint32_t* l2g,
                                 uint32_t local_n, const uint32_t* local_of, uint64_t* counts,
                                 const uint64_t* lptr, uint32_t* lcol) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < local_n; i += nw) {
        const uint32_t g = l2g[i];
        const uint64_t beg = row_ptr[g], end = row_ptr[g + 1];
        uint64_t w = lptr ? lptr[i] : 0;
        for (uint64_t e0 = beg; e0 < end; e0 += 32) {
            uint32_t l = GDX_UNSEEN;
            if (e0 + lane < end) l = local_of[col[e0 + lane]];
            const bool ok = l != GDX_UNSEEN;
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (lptr && ok) lcol[w + __popc(bal & ((1u << lane) - 1))] = l;
            w += __popc(bal);
        }
        if (!lptr && lane == 0) counts[i] = w;
    }
}

// Cooperative-batch feature LOAD: rows idx[i] of a split-bf16 store (hi and lo
// planes, pitch ld_src) into the batch operand (pitch ld_out).  A warp per row,
// 16-byte vectors (8 elements) per lane; both planes in one pass.
__global__ void gather_split_rows_kernel(const uint16_t* __restrict__ src_hi,
                                         const uint16_t* __restrict__ src_lo, uint64_t ld_src,
                                         const uint32_t* __restrict__ idx, uint32_t rows,
                                         uint32_t vecs, uint16_t* __restrict__ out_hi,
                                         uint16_t* __restrict__ out_lo, uint64_t ld_out) {
    // a group of `vecs` lanes per row (32/vecs rows per warp when a row is <= 16 vectors)
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rpw = vecs >= 32 ? 1 : 32 / vecs;
    const uint32_t sub = vecs >= 32 ? 0 : lane / vecs;
    const uint32_t v0 = vecs >= 32 ? lane : lane - sub * vecs;
    if (sub >= rpw) return;
    const uint64_t groups = static_cast<uint64_t>((gridDim.x * blockDim.x) >> 5) * rpw;
    for (uint64_t r = static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * rpw + sub; r < rows;
         r += groups) {
        const uint64_t so = static_cast<uint64_t>(idx[r]) * ld_src, oo = r * ld_out;
        const uint4* sh = reinterpret_cast<const uint4*>(src_hi + so);
        const uint4* sl = reinterpret_cast<const uint4*>(src_lo + so);
        uint4* dh = reinterpret_cast<uint4*>(out_hi + oo);
        uint4* dl = reinterpret_cast<uint4*>(out_lo + oo);
        for (uint32_t v = v0; v < vecs; v += 32) {
            const uint4 a = __ldg(sh + v), b = __ldg(sl + v);
            dh[v] = a;
            dl[v] = b;
        }
    }
}

__global__ void gather_rows_kernel(const float* src, uint64_t ld_src, const uint32_t* idx,
                                   uint32_t rows, uint32_t cols, float* out, uint64_t ld_out) {
    const uint64_t total = static_cast<uint64_t>(rows) * cols;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        out[r * ld_out + c] = src[static_cast<uint64_t>(idx[r]) * ld_src + c];
    }
}

__global__ void widen_u32(const uint32_t* in, uint64_t n, uint64_t* out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

__global__ void tail_total(const uint64_t* counts, uint64_t* out, uint64_t n) {
    out[n] = out[n - 1] + counts[n - 1];
}

unsigned grid_for(uint64_t threads, unsigned block = 256) {
    uint64_t b = (threads + block - 1) / block;
    const uint64_t cap = static_cast<uint64_t>(device_sms()) * 32;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b ? b : 1);
}

template <class T>
int scan_exclusive(const T* in, T* out, uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    GDX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int64_t>(n), s));
    void* tmp = nullptr;
    GDX_CUDA(cudaMallocAsync(&tmp, bytes ? bytes : 16, s));
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, static_cast<int64_t>(n), s);
    cudaFreeAsync(tmp, s);
    GDX_CUDA(e);
    note_launch();
    return GDX_OK;
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" int gdx_sampled_growth(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                                  const uint8_t* excluded, const uint8_t* allowed,
                                  uint32_t max_hop, uint32_t fanout, uint64_t seed, uint32_t* mark,
                                  uint32_t* work, gdx_stream stream) {
    GDX_REQUIRE(row_ptr && col && excluded && mark && work, GDX_INPUT,
                "gdx_sampled_growth: null pointer");
    cudaStream_t s = as_cuda(stream);
    uint32_t* fa = work;
    uint32_t* fb = work + n;
    uint32_t* cnt = work + 2 * static_cast<uint64_t>(n);  // [0] current, [1] next
    GDX_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(uint32_t), s));
    if (max_hop == 0 || fanout == 0 || n == 0) return GDX_OK;  // extract.cpp:158 loop never runs
    seed_frontier<<<grid_for(static_cast<uint64_t>(n) * 32), 256, 0, s>>>(row_ptr, col, n, excluded,
                                                                          allowed, fa, cnt);
    note_launch();
    GDX_CUDA(cudaGetLastError());
    // Hops are enqueued in batches with no host round trip: each expand kernel reads its
    // frontier size from device memory (cnt alternates in / out) over a fixed grid.  The
    // host looks once per batch of kHopBatch hops whether the frontier emptied (a BFS to
    // depth max_hop would otherwise enqueue max_hop launches).
    constexpr uint32_t kHopBatch = 16;
    const unsigned grid = static_cast<unsigned>(device_sms()) * 8;
    for (uint32_t h = 1; h <= max_hop;) {
        const uint32_t stop = (max_hop - h + 1 > kHopBatch) ? h + kHopBatch : max_hop + 1;
        for (; h < stop; ++h) {
            uint32_t* cin = cnt + ((h - 1) & 1);
            uint32_t* cout = cnt + (h & 1);
            GDX_CUDA(cudaMemsetAsync(cout, 0, sizeof(uint32_t), s));
            expand_hop<<<grid, 256, 0, s>>>(row_ptr, col, excluded, allowed, fa, cin, fanout, seed, h, mark, fb,
                                            cout);
            note_launch();
            GDX_CUDA(cudaGetLastError());
            uint32_t* t = fa;
            fa = fb;
            fb = t;
        }
        if (h > max_hop) break;
        uint32_t nf = 0;
        GDX_CUDA(cudaMemcpyAsync(&nf, cnt + ((h - 1) & 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        if (nf == 0) break;
    }
    return GDX_OK;
}

extern "C" int gdx_induced_count(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                                 const uint32_t* mark, unsigned long long* work, uint64_t* result,
                                 gdx_stream stream) {
    GDX_REQUIRE(row_ptr && col && mark && work && result, GDX_INPUT, "gdx_induced_count: null pointer");
    cudaStream_t s = as_cuda(stream);
    GDX_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long), s));
    if (n) {
        induced_count_kernel<<<grid_for(static_cast<uint64_t>(n) * 32), 256, 0, s>>>(row_ptr, col, n,
                                                                                     mark, work);
        note_launch();
        GDX_CUDA(cudaGetLastError());
    }
    unsigned long long h = 0;
    GDX_CUDA(cudaMemcpyAsync(&h, work, sizeof(h), cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    *result = h;
    return GDX_OK;
}

extern "C" int gdx_peel_mfg(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                            const uint8_t* in_batch, const uint32_t* targets, uint64_t nt,
                            uint32_t layers, uint32_t* work, uint64_t* counts, gdx_stream stream) {
    GDX_REQUIRE(row_ptr && col && in_batch && work && counts, GDX_INPUT, "gdx_peel_mfg: null pointer");
    GDX_REQUIRE(nt <= n, GDX_INPUT, "gdx_peel_mfg: more targets than vertices");
    cudaStream_t s = as_cuda(stream);
    uint32_t* in_set = work;
    uint32_t* fa = work + n;
    uint32_t* fb = work + 2 * static_cast<uint64_t>(n);
    uint32_t* cnt = work + 3 * static_cast<uint64_t>(n);
    GDX_CUDA(cudaMemsetAsync(in_set, 0, sizeof(uint32_t) * n, s));
    if (nt) {
        peel_init<<<grid_for(nt), 256, 0, s>>>(targets, nt, in_set, fa);
        note_launch();
        GDX_CUDA(cudaGetLastError());
    }
    // every back-peel step enqueued with device-resident frontier sizes (no host round
    // trip per step); each step's number of added vertices is copied aside and read back
    // once at the end
    uint32_t* adds = nullptr;
    GDX_CUDA(cudaMallocAsync(&adds, sizeof(uint32_t) * (layers + 1), s));
    GDX_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(uint32_t), s));
    if (nt) {
        const uint32_t nt32 = static_cast<uint32_t>(nt);
        GDX_CUDA(cudaMemcpyAsync(cnt, &nt32, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    }
    const unsigned grid = static_cast<unsigned>(device_sms()) * 8;
    for (uint32_t back = 1; back <= layers; ++back) {
        uint32_t* cin = cnt + ((back - 1) & 1);
        uint32_t* cout = cnt + (back & 1);
        GDX_CUDA(cudaMemsetAsync(cout, 0, sizeof(uint32_t), s));
        peel_step<<<grid, 256, 0, s>>>(row_ptr, col, in_batch, fa, cin, in_set, fb, cout);
        note_launch();
        GDX_CUDA(cudaGetLastError());
        GDX_CUDA(cudaMemcpyAsync(adds + back, cout, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        uint32_t* t = fa;
        fa = fb;
        fb = t;
    }
    std::vector<uint32_t> h(layers + 1, 0);
    if (layers) GDX_CUDA(cudaMemcpyAsync(h.data() + 1, adds + 1, sizeof(uint32_t) * layers, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaFreeAsync(adds, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    counts[layers] = nt;
    uint64_t total = nt;
    for (uint32_t back = 1; back <= layers; ++back) {
        total += h[back];
        counts[layers - back] = total;
    }
    return GDX_OK;
}

extern "C" int gdx_split_batch(const uint32_t* bv, uint64_t nb, const uint32_t* sp,
                               const uint32_t* gp, uint32_t server, uint32_t gpus,
                               uint32_t* share_of, uint32_t* work, gdx_stream stream) {
    GDX_REQUIRE(gpus >= 1 && gpus <= 1024, GDX_INPUT, "gdx_split_batch: gpus must be in [1, 1024]");
    GDX_REQUIRE(nb == 0 || (bv && sp && gp && share_of && work), GDX_INPUT,
                "gdx_split_batch: null pointer");
    if (nb == 0) return GDX_OK;
    cudaStream_t s = as_cuda(stream);
    // work layout (u32 units): [flag nb][pad][wide u64 nb][rank u64 nb][inner u64 gpus]
    uint32_t* flag = work;
    uint64_t* wide = reinterpret_cast<uint64_t*>(work + ((nb + 1) & ~1ull));
    uint64_t* rank = wide + nb;
    unsigned long long* ic = reinterpret_cast<unsigned long long*>(rank + nb);
    GDX_CUDA(cudaMemsetAsync(ic, 0, sizeof(unsigned long long) * gpus, s));
    split_classify<<<grid_for(nb), 256, 0, s>>>(bv, nb, sp, gp, server, gpus, share_of, flag, ic);
    note_launch();
    GDX_CUDA(cudaGetLastError());
    widen_u32<<<grid_for(nb), 256, 0, s>>>(flag, nb, wide);
    note_launch();
    GDX_CUDA(cudaGetLastError());
    int rc = scan_exclusive<uint64_t>(wide, rank, nb, s);
    if (rc) return rc;
    split_assign<<<grid_for(nb), 256, 0, s>>>(nb, gpus, flag, rank, ic, share_of);
    note_launch();
    return check_launch("gdx_split_batch");
}

extern "C" int gdx_exclusive_scan_u64(const uint64_t* counts, uint64_t n, uint64_t* out,
                                      uint64_t* total, gdx_stream stream) {
    GDX_REQUIRE(counts && out, GDX_INPUT, "gdx_exclusive_scan_u64: null pointer");
    cudaStream_t s = as_cuda(stream);
    if (n) {
        int rc = scan_exclusive<uint64_t>(counts, out, n, s);
        if (rc) return rc;
        // out[n] = out[n-1] + counts[n-1]
        tail_total<<<1, 1, 0, s>>>(counts, out, n);
        note_launch();
        GDX_CUDA(cudaGetLastError());
    } else {
        GDX_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    }
    if (total) {
        GDX_CUDA(cudaMemcpyAsync(total, out + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
    }
    return GDX_OK;
}

extern "C" int gdx_order_by_hop(const uint32_t* hop, uint32_t n, uint32_t max_hop,
                                uint32_t* local_to_global, uint32_t* local_of, uint64_t* hop_start,
                                uint32_t* local_n, gdx_stream stream) {
    GDX_REQUIRE(hop && local_to_global && local_of && hop_start && local_n, GDX_INPUT,
                "gdx_order_by_hop: null pointer");
    cudaStream_t s = as_cuda(stream);
    *local_n = 0;
    hop_start[0] = 0;
    if (n == 0) {
        for (uint32_t h = 0; h <= max_hop; ++h) hop_start[h + 1] = 0;
        return GDX_OK;
    }
    fill_u32<<<grid_for(n), 256, 0, s>>>(local_of, n, GDX_UNSEEN);
    note_launch();
    uint32_t* flag = nullptr;
    uint32_t* rank = nullptr;
    GDX_CUDA(cudaMallocAsync(&flag, sizeof(uint32_t) * (static_cast<uint64_t>(n) + 1), s));
    GDX_CUDA(cudaMallocAsync(&rank, sizeof(uint32_t) * (static_cast<uint64_t>(n) + 1), s));
    uint32_t base = 0;
    int rc = GDX_OK;
    for (uint32_t h = 0; h <= max_hop && rc == GDX_OK; ++h) {
        hop_flags<<<grid_for(n), 256, 0, s>>>(hop, n, h, flag);
        note_launch();
        rc = scan_exclusive<uint32_t>(flag, rank, n, s);
        if (rc) break;
        hop_scatter<<<grid_for(n), 256, 0, s>>>(hop, n, h, rank, base, local_to_global, local_of);
        note_launch();
        uint32_t last_rank = 0, last_flag = 0;
        cudaMemcpyAsync(&last_rank, rank + n - 1, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) rc = gdx::fail(GDX_INTERNAL, "gdx_order_by_hop: sync failed");
        base += last_rank + last_flag;
        hop_start[h + 1] = base;
    }
    cudaFreeAsync(flag, s);
    cudaFreeAsync(rank, s);
    if (rc) return rc;
    *local_n = base;
    return check_launch("gdx_order_by_hop");
}

extern "C" int gdx_local_csr(const uint64_t* row_ptr, const uint32_t* col,
                             const uint32_t* local_to_global, uint32_t local_n,
                             const uint32_t* local_of, uint64_t* counts, const uint64_t* lptr,
                             uint32_t* lcol, gdx_stream stream) {
    GDX_REQUIRE(row_ptr && col && local_to_global && local_of, GDX_INPUT, "gdx_local_csr: null pointer");
    GDX_REQUIRE(lptr ? lcol != nullptr : counts != nullptr, GDX_INPUT,
                "gdx_local_csr: pass 1 needs counts, pass 2 needs lptr and lcol");
    if (!local_n) return GDX_OK;
    local_csr_kernel<<<grid_for(static_cast<uint64_t>(local_n) * 32), 256, 0, as_cuda(stream)>>>(
        row_ptr, col, local_to_global, local_n, local_of, counts, lptr, lcol);
    note_launch();
    return check_launch("gdx_local_csr");
}

extern "C" int gdx_gather_split_rows(const uint16_t* src_hi, const uint16_t* src_lo, uint64_t ld_src,
                                     const uint32_t* idx, uint32_t rows, uint32_t cols,
                                     uint16_t* out_hi, uint16_t* out_lo, uint64_t ld_out,
                                     gdx_stream stream) {
    GDX_REQUIRE(src_hi && src_lo && idx && out_hi && out_lo, GDX_INPUT,
                "gdx_gather_split_rows: null pointer");
    GDX_REQUIRE(ld_src % 8 == 0 && ld_out % 8 == 0 && ld_src >= cols && ld_out >= cols, GDX_INPUT,
                "gdx_gather_split_rows: pitches must be multiples of 8 elements and >= cols");
    GDX_REQUIRE(((reinterpret_cast<uintptr_t>(src_hi) | reinterpret_cast<uintptr_t>(src_lo) |
                  reinterpret_cast<uintptr_t>(out_hi) | reinterpret_cast<uintptr_t>(out_lo)) & 15) == 0,
                GDX_INPUT, "gdx_gather_split_rows: planes must be 16-byte aligned");
    if (!rows || !cols) return GDX_OK;
    const uint32_t vecs = (cols + 7) / 8;  // whole 16-byte vectors (pitch padding included)
    gather_split_rows_kernel<<<grid_for(static_cast<uint64_t>(rows) * 32), 256, 0, as_cuda(stream)>>>(
        src_hi, src_lo, ld_src, idx, rows, vecs, out_hi, out_lo, ld_out);
    note_launch();
    return check_launch("gdx_gather_split_rows");
}

extern "C" int gdx_gather_rows(const float* src, uint64_t ld_src, const uint32_t* idx, uint32_t rows,
                               uint32_t cols, float* out, uint64_t ld_out, gdx_stream stream) {
    GDX_REQUIRE(src && idx && out, GDX_INPUT, "gdx_gather_rows: null pointer");
    if (!rows || !cols) return GDX_OK;
    gather_rows_kernel<<<grid_for(static_cast<uint64_t>(rows) * cols), 256, 0, as_cuda(stream)>>>(
        src, ld_src, idx, rows, cols, out, ld_out);
    note_launch();
    return check_launch("gdx_gather_rows");
}
