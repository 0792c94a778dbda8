// host.cpp -- host-side C++ of libgdx: error plumbing, launch accounting and
// the host preprocessing that stays on the CPU: the
// G(n,p) generator and the random partition, parallelised with OpenMP and
// bit-identical to the reference.
//
// gen_random_graph (graph.cpp:137-154) keys every vertex's stream by
// (seed, u), so vertices can be sampled in any order.  assemble_undirected
// (graph.cpp:116-132) produces rows sorted ascending without a sort pass; the
// parallel fill appends with atomic cursors and then sorts each row, which
// yields the identical CSR because every row is a set of distinct ids.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <mutex>
#include <numeric>
#include <queue>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gdx.h"

namespace gdx {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
inline uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t mix64(uint64_t x) { return fin(x + kGamma); }

// rng.hpp:18-52 KeyedRng
struct Stream {
    uint64_t s;
    Stream(uint64_t seed, uint64_t k1, uint64_t k2) {
        s = mix64(seed);
        s = mix64(s ^ (k1 + kGamma));
        s = mix64(s ^ (k2 + 0xc2b2ae3d27d4eb4fULL));
    }
    uint64_t next() {
        s += kGamma;
        return fin(s);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
    }
};

// graph.cpp:86-94
inline uint64_t geometric_skip(Stream& r, double p, double log1mp) {
    if (p >= 1.0) return 0;
    double u = r.unit();
    if (u <= 0.0) u = 0x1.0p-53;
    double skip = std::floor(std::log(u) / log1mp);
    if (skip < 0.0) skip = 0.0;
    if (skip > 1e18) skip = 1e18;
    return static_cast<uint64_t>(skip);
}

// graph.cpp:99-111, for one u
template <class Emit>
void sample_range(uint64_t seed, uint32_t u, uint32_t start, uint32_t limit, double p, Emit&& emit) {
    if (p <= 0.0 || start >= limit) return;
    Stream r(seed, u, 0);
    const double log1mp = (p < 1.0) ? std::log1p(-p) : 0.0;
    uint64_t v = start + geometric_skip(r, p, log1mp);
    while (v < limit) {
        emit(static_cast<uint32_t>(v));
        v += 1 + geometric_skip(r, p, log1mp);
    }
}

double edge_probability(uint32_t n, double d) {
    double p = d / static_cast<double>(n - 1);
    return p > 1.0 ? 1.0 : p;
}

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int device_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
    if (dev >= 64) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

int ensure_smem_attr(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(GDX_INTERNAL, "cudaGetDevice failed");
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, kernel})) return GDX_OK;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess)
        return fail(GDX_INTERNAL, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    done.insert({dev, kernel});
    return GDX_OK;
}

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GDX_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
    return GDX_OK;
}

}  // namespace gdx

using namespace gdx;

extern "C" const char* gdx_last_error(void) { return g_last_error.c_str(); }
extern "C" int gdx_version(void) { return 1; }
extern "C" uint64_t gdx_launch_count(void) { return g_launches.load(); }

extern "C" uint64_t gdx_host_gen_random_graph_count(uint32_t n, double d, uint64_t seed,
                                                    uint64_t* ro) {
    if (n == 0 || d < 0.0 || d >= static_cast<double>(n) || !ro) {
        fail(GDX_INPUT, "gen_random_graph: need n >= 1 and 0 <= avg_degree < n");
        return ~0ull;
    }
    std::memset(ro, 0, sizeof(uint64_t) * (static_cast<size_t>(n) + 1));
    if (n == 1 || d == 0.0) return 0;
    const double p = edge_probability(n, d);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t uu = 0; uu < static_cast<int64_t>(n) - 1; ++uu) {
        const uint32_t u = static_cast<uint32_t>(uu);
        uint64_t mine = 0;
        sample_range(seed, u, u + 1, n, p, [&](uint32_t v) {
            ++mine;
            __atomic_fetch_add(&ro[v + 1], 1, __ATOMIC_RELAXED);
        });
        __atomic_fetch_add(&ro[u + 1], mine, __ATOMIC_RELAXED);
    }
    for (uint32_t i = 0; i < n; ++i) ro[i + 1] += ro[i];
    return ro[n];
}

extern "C" int gdx_host_gen_random_graph_fill(uint32_t n, double d, uint64_t seed,
                                              const uint64_t* ro, uint32_t* cols) {
    if (n == 0 || d < 0.0 || d >= static_cast<double>(n) || !ro)
        return fail(GDX_INPUT, "gen_random_graph: need n >= 1 and 0 <= avg_degree < n");
    if (n == 1 || d == 0.0 || ro[n] == 0) return GDX_OK;
    const double p = edge_probability(n, d);
    std::vector<uint64_t> cursor(ro, ro + n);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t uu = 0; uu < static_cast<int64_t>(n) - 1; ++uu) {
        const uint32_t u = static_cast<uint32_t>(uu);
        sample_range(seed, u, u + 1, n, p, [&](uint32_t v) {
            cols[__atomic_fetch_add(&cursor[u], 1, __ATOMIC_RELAXED)] = v;
            cols[__atomic_fetch_add(&cursor[v], 1, __ATOMIC_RELAXED)] = u;
        });
    }
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < static_cast<int64_t>(n); ++v) std::sort(cols + ro[v], cols + ro[v + 1]);
    return GDX_OK;
}

// SampleTrace of extract_sampled (extract.hpp:49-64; the attribution order of
// extract.cpp:158-178): frontier vertices hop by hop in ascending order, each taking the
// not-yet-included vertices of its sampled prefix.  Host diagnostics: the set of taken
// vertices is what the device growth computes; this replays the sequential order only
// to attribute each one to its first exposing frontier vertex.
extern "C" int gdx_host_sample_trace(uint32_t n, const uint64_t* ro, const uint32_t* cols, const uint8_t* inner,
                                     uint32_t max_hop, uint32_t fanout, uint64_t seed, uint64_t cap_steps,
                                     uint64_t cap_taken, uint64_t* nsteps, uint64_t* ntaken, uint32_t* step_vertex,
                                     uint32_t* step_hop, uint64_t* step_off, uint32_t* taken) {
    if (!ro || (!cols && n && ro[n]) || !inner || !nsteps || !ntaken)
        return fail(GDX_INPUT, "gdx_host_sample_trace: null pointer");
    std::vector<uint8_t> incl(inner, inner + n);
    std::vector<uint32_t> frontier, added, cand;
    for (uint32_t v = 0; v < n; ++v) {
        if (!inner[v]) continue;
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e)
            if (!inner[cols[e]]) {
                frontier.push_back(v);
                break;
            }
    }
    uint64_t ns = 0, nt = 0;
    for (uint32_t hop = 1; hop <= max_hop && !frontier.empty(); ++hop) {
        added.clear();
        for (uint32_t v : frontier) {
            cand.clear();
            for (uint64_t e = ro[v]; e < ro[v + 1]; ++e)
                if (!inner[cols[e]]) cand.push_back(cols[e]);
            if (fanout != GDX_UNLIMITED_FANOUT && cand.size() > fanout) {
                Stream r(seed, v, 0x73616d70ULL);   // keyed_shuffle (rng.hpp:55-61)
                for (size_t i = cand.size(); i > 1; --i) std::swap(cand[i - 1], cand[r.below(i)]);
                cand.resize(fanout);
            }
            if (step_vertex && ns < cap_steps) {
                step_vertex[ns] = v;
                step_hop[ns] = hop;
                step_off[ns] = nt;
            }
            ++ns;
            for (uint32_t u : cand) {
                if (incl[u]) continue;
                incl[u] = 1;
                if (taken && nt < cap_taken) taken[nt] = u;
                ++nt;
                added.push_back(u);
            }
        }
        std::sort(added.begin(), added.end());
        frontier.swap(added);
    }
    if (step_off && ns <= cap_steps) step_off[ns < cap_steps ? ns : cap_steps] = nt;
    *nsteps = ns;
    *ntaken = nt;
    if ((step_vertex && ns > cap_steps) || (taken && nt > cap_taken))
        return fail(GDX_CAPACITY, "gdx_host_sample_trace: output capacity too small");
    return GDX_OK;
}

// partition.cpp:51-61
extern "C" int gdx_host_partition_random(uint32_t n, uint32_t parts, uint64_t seed,
                                         uint32_t* assignment) {
    if (parts == 0) return fail(GDX_INPUT, "partition: parts must be >= 1");
    if (parts > n)
        return fail(GDX_INPUT, "partition: parts (" + std::to_string(parts) +
                                   ") exceeds vertex count (" + std::to_string(n) + ")");
    std::vector<uint32_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0u);
    Stream r(seed, 0x7061727469ULL, 0);
    for (uint64_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[r.below(i)]);
    for (uint32_t i = 0; i < n; ++i) assignment[perm[i]] = i % parts;
    return GDX_OK;
}

// Gain-bucket queue for the region growth: one two-level bitmap of vertex ids per gain
// value.  An increment only sets the vertex's bit at its new gain; the bits it leaves at
// lower gains go stale and are dropped when a pop meets them (a stale bit is never the
// answer: the vertex's valid bit sits at a higher, non-empty gain, or it is assigned).
// pop() therefore returns the unassigned frontier vertex with the largest gain, ties to
// the lowest id -- exactly the valid top of the reference's lazy priority_queue of
// (gain, MAX - v) (partition.cpp:95-125) -- with one bitmap store per edge instead of a
// heap push.
class GainBuckets {
public:
    explicit GainBuckets(uint32_t n) : n_(n), words_((n + 63) / 64), sums_((words_ + 63) / 64) {}
    void set(uint32_t g, uint32_t v) {
        Level& L = level(g);
        const uint32_t w = v >> 6;
        if (!L.w[w]) {
            L.s[w >> 6] |= 1ull << (w & 63);
            if (w >> 6 < L.lo) L.lo = w >> 6;
        }
        L.w[w] |= 1ull << (v & 63);
        ++L.count;  // bits set (valid + stale); a vertex's bit per gain is set at most once
        if (g > top_) top_ = g;
    }
    // Lowest valid id at the highest gain holding one (removed); n if none.
    template <class Valid>
    uint32_t pop(Valid valid) {
        while (top_ > 0) {
            Level& L = lv_[top_];
            if (L.count == 0) {
                --top_;
                continue;
            }
            while (!L.s[L.lo]) ++L.lo;
            const uint32_t w = (L.lo << 6) + static_cast<uint32_t>(__builtin_ctzll(L.s[L.lo]));
            const uint32_t v = (w << 6) + static_cast<uint32_t>(__builtin_ctzll(L.w[w]));
            L.w[w] &= L.w[w] - 1;  // v is the lowest bit of its word
            if (!L.w[w]) L.s[w >> 6] &= ~(1ull << (w & 63));
            --L.count;
            if (valid(v, top_)) return v;
        }
        return n_;
    }
    // empty every bucket (a new region starts with all gains 0)
    void reset() {
        for (Level& L : lv_)
            if (L.count) {
                std::fill(L.w.begin(), L.w.end(), 0ull);
                std::fill(L.s.begin(), L.s.end(), 0ull);
                L.count = 0;
                L.lo = sums_;
            }
        top_ = 0;
    }
private:
    struct Level {
        std::vector<uint64_t> w, s;
        uint32_t lo = 0;
        uint64_t count = 0;
    };
    Level& level(uint32_t g) {
        if (g >= lv_.size()) lv_.resize(g + 1);
        Level& L = lv_[g];
        if (L.w.empty()) {
            L.w.assign(words_, 0);
            L.s.assign(sums_, 0);
            L.lo = sums_;
        }
        return L;
    }
    uint32_t n_, words_, sums_, top_ = 0;
    std::vector<Level> lv_;
};

// partition_mincut (partition.cpp:63-170): greedy region growing from high-degree
// seeds (frontier vertex with the most edges into the region next, ties to the
// lowest id), then <= 10 boundary-refinement passes under the size cap
// floor(ceil(n/parts) * (1 + eps)).  Host preprocessing, deterministic; the growth
// order comes from GainBuckets instead of a heap, the assignment is bit-identical to
// the reference's (tests/test_abi.py against the compiled reference).
extern "C" int gdx_host_partition_mincut(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                                         uint32_t parts, uint64_t seed, double eps,
                                         uint32_t* assignment) {
    (void)seed;  // the reference ignores it: growth and refinement are deterministic
    if (parts == 0) return fail(GDX_INPUT, "partition: parts must be >= 1");
    if (parts > n)
        return fail(GDX_INPUT, "partition: parts (" + std::to_string(parts) +
                                   ") exceeds vertex count (" + std::to_string(n) + ")");
    if (eps < 0.0) return fail(GDX_INPUT, "partition: epsilon must be >= 0");
    const uint32_t unassigned = parts;
    std::vector<uint32_t> a(n, unassigned);
    const uint32_t base = n / parts, rem = n % parts;
    auto deg = [&](uint32_t v) { return static_cast<uint32_t>(ro[v + 1] - ro[v]); };
    std::vector<uint32_t> by_degree(n);
    std::iota(by_degree.begin(), by_degree.end(), 0u);
    std::stable_sort(by_degree.begin(), by_degree.end(),
                     [&](uint32_t x, uint32_t y) { return deg(x) > deg(y); });
    size_t seed_scan = 0;
    // st[u]: the gain of an unassigned vertex, or kAssigned | part -- one random access
    // per edge for the "unassigned?" test and the gain update together; neighbours'
    // entries are prefetched a few edges ahead (the growth is latency-bound at the
    // products shape, 2.4 M vertices)
    constexpr uint32_t kAssigned = 0x80000000u;
    std::vector<uint32_t> st(n, 0), touched;
    GainBuckets q(n);
    constexpr uint64_t kAhead = 16;
    for (uint32_t part = 0; part < parts; ++part) {
        const uint32_t target = base + (part < rem ? 1 : 0);
        for (uint32_t taken = 0; taken < target; ++taken) {
            uint32_t v = q.pop([&](uint32_t c, uint32_t g) { return st[c] == g; });
            if (v == n) {  // empty frontier: next unassigned vertex by degree
                while (st[by_degree[seed_scan]] & kAssigned) ++seed_scan;
                v = by_degree[seed_scan];
            }
            st[v] = kAssigned | part;
            const uint64_t e1 = ro[v + 1];
            for (uint64_t e = ro[v]; e < e1; ++e) {
                if (e + kAhead < e1) __builtin_prefetch(&st[ci[e + kAhead]], 1, 3);
                const uint32_t u = ci[e];
                const uint32_t g = st[u];
                if (g & kAssigned) continue;
                if (g == 0) touched.push_back(u);
                st[u] = g + 1;
                q.set(g + 1, u);
            }
        }
        // the next region starts from an empty frontier with all gains 0
        for (uint32_t u : touched)
            if (!(st[u] & kAssigned)) st[u] = 0;
        touched.clear();
        q.reset();
    }
    for (uint32_t v = 0; v < n; ++v) a[v] = st[v] & ~kAssigned;
    std::vector<uint32_t> size(parts, 0);
    for (uint32_t v = 0; v < n; ++v) ++size[a[v]];
    uint32_t cap = static_cast<uint32_t>(
        std::floor(static_cast<double>((n + parts - 1) / parts) * (1.0 + eps)));
    cap = std::max<uint32_t>(cap, (n + parts - 1) / parts);
    std::vector<uint64_t> conn(parts, 0);
    const uint64_t nnz = ro[n];
    std::vector<uint32_t> tparts;
    for (int pass = 0; pass < 10; ++pass) {
        bool moved = false;
        for (uint32_t v = 0; v < n; ++v) {
            const uint32_t own = a[v];
            if (size[own] <= 1) continue;
            tparts.clear();
            const uint64_t e1 = ro[v + 1];
            for (uint64_t e = ro[v]; e < e1; ++e) {
                if (e + kAhead < nnz) __builtin_prefetch(&a[ci[e + kAhead]], 0, 3);  // across rows
                const uint32_t q = a[ci[e]];
                if (conn[q] == 0) tparts.push_back(q);
                ++conn[q];
            }
            uint32_t best = own;
            const uint64_t own_conn = conn[own];
            uint64_t best_gain = 0;
            for (uint32_t q : tparts) {
                if (q == own || size[q] + 1 > cap) continue;
                if (conn[q] > own_conn && conn[q] - own_conn > best_gain) {
                    best_gain = conn[q] - own_conn;
                    best = q;
                } else if (conn[q] > own_conn && conn[q] - own_conn == best_gain && q < best) {
                    best = q;
                }
            }
            for (uint32_t q : tparts) conn[q] = 0;
            if (best != own) {
                a[v] = best;
                --size[own];
                ++size[best];
                moved = true;
            }
        }
        if (!moved) break;
    }
    std::copy(a.begin(), a.end(), assignment);
    return GDX_OK;
}
