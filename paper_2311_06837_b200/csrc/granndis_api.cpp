// granndis_api.cpp -- the reference's C++ API (include/granndis_b200/granndis.hpp)
// implemented over the C ABI of libgdx (include/gdx.h).  This is the binding a
// maintainer of the reference would drop in for proj/src/{reference_gnn,extract}.cpp
// (INTEGRATION.md): same signatures, same validation and error types, compute
// on the GPU, results returned by value as fp64 Matrix / index vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <set>

#include "gdx.h"
#include "granndis_b200/granndis.hpp"

namespace granndis {
namespace {

void check(int rc) {
    if (rc == GDX_OK) return;
    const std::string m = gdx_last_error();
    switch (rc) {
        case GDX_INPUT: throw InputError(m);
        case GDX_CAPACITY: throw CapacityError(m);
        case GDX_CONTRACT: throw ContractError(m);
        default: throw InternalError(m);
    }
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw InternalError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count, bool zero = true) : n(count) {
        cuda(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
        if (zero) cuda(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)), "cudaMemset");
    }
    Dev(const T* host, size_t count) : Dev(count, host == nullptr) {
        if (count && host) cuda(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        if (this != &o) {
            if (p) cudaFree(p);
            p = o.p;
            n = o.n;
            o.p = nullptr;
        }
        return *this;
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    std::vector<T> download() const {
        std::vector<T> h(n);
        if (n) cuda(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
        return h;
    }
};

size_t pad4(size_t x) { return (x + 3) / 4 * 4; }
size_t pad8(size_t x) { return (x + 7) / 8 * 8; }

struct DevCSR {
    Dev<uint64_t> rp;
    Dev<uint32_t> col;
    uint32_t rows = 0;
};

}  // namespace

// The device copy of a Graph's CSR, uploaded once per graph (Graph::device_).
struct GraphDevice {
    static const DevCSR& get(const Graph& g) {
        if (!g.device_) {
            auto d = std::make_shared<DevCSR>();
            d->rp = Dev<uint64_t>(g.row_offsets().data(), g.row_offsets().size());
            d->col = g.col_indices().empty() ? Dev<uint32_t>(1)
                                             : Dev<uint32_t>(g.col_indices().data(), g.col_indices().size());
            d->rows = g.num_vertices();
            g.device_ = d;
        }
        return *static_cast<const DevCSR*>(g.device_.get());
    }
};

namespace {

const DevCSR& upload(const Graph& g) { return GraphDevice::get(g); }

// split-bf16 copy of an fp32 device matrix (rows x cols, pitch ld) with pitch pad8(cols)
struct Split {
    Dev<uint16_t> hi, lo;
    size_t ld = 0;
    Split(const float* src, size_t ld_src, uint32_t rows, uint32_t cols)
        : hi(std::max<size_t>(rows, 1) * pad8(cols)), lo(std::max<size_t>(rows, 1) * pad8(cols)),
          ld(pad8(cols)) {
        if (rows && cols) check(gdx_split_bf16(src, ld_src, rows, cols, hi.p, lo.p, ld, 0, nullptr));
    }
    Split(uint32_t rows, uint32_t cols)
        : hi(std::max<size_t>(rows, 1) * pad8(cols)), lo(std::max<size_t>(rows, 1) * pad8(cols)),
          ld(pad8(cols)) {}
};

// reference_gnn.cpp:36-50
void check_shapes(const DenseFeatures& x, const LayerWeights& w, std::uint32_t layers) {
    if (layers == 0) return;
    if (w.layers.size() < layers)
        throw InputError("forward: " + std::to_string(layers) + " layers requested, " +
                         std::to_string(w.layers.size()) + " weight matrices given");
    std::uint32_t width = x.cols;
    for (std::uint32_t l = 0; l < layers; ++l) {
        if (w.layers[l].cols != width)
            throw InputError("forward: layer " + std::to_string(l + 1) + " expects width " +
                             std::to_string(w.layers[l].cols) + ", got " + std::to_string(width));
        width = w.layers[l].rows;
    }
}

// Layer loop shared by forward_full and forward_server_local: rows outside the
// computed prefix stay zero (the hop mask of reference_gnn.cpp:123-131).
Dev<float> run_layers(const DevCSR& csr, uint32_t n_local, Dev<float> h, uint32_t width,
                      const LayerWeights& w, std::uint32_t layers, const std::vector<uint32_t>& rows_in,
                      const std::vector<uint32_t>& rows_out, uint32_t* out_width) {
    for (std::uint32_t l = 0; l < layers; ++l) {
        const Matrix& W = w.layers[l];
        const uint32_t H = W.rows;
        std::vector<float> wf(W.data.begin(), W.data.end());
        Dev<float> wdev(wf.data(), wf.size());
        Split B(wdev.p, W.cols, H, W.cols);
        const uint32_t r_in = rows_in[l], r_out = rows_out[l];
        Dev<float> out(size_t(std::max(n_local, 1u)) * pad4(H));
        gdx_gemm_args g{};
        gdx_aggregate_args a{};
        a.row_ptr = csr.rp.p;
        a.col = csr.col.p;
        a.rows = r_out;
        a.self_coef = 1.0f;
        if (H <= width) {
            Split A(h.p, pad4(width), n_local, width);
            Dev<float> Z(size_t(std::max(n_local, 1u)) * pad4(H));
            if (r_in) {
                g.a_hi = A.hi.p; g.a_lo = A.lo.p; g.lda = A.ld;
                g.b_hi = B.hi.p; g.b_lo = B.lo.p; g.ldb = B.ld;
                g.m = r_in; g.n = H; g.k = width;
                g.c0 = Z.p; g.ldc0 = pad4(H); g.split = H;
                check(gdx_gemm_tn(&g, nullptr));
            }
            if (r_out) {
                a.width = H; a.src = Z.p; a.ld_src = pad4(H); a.relu = 1;
                a.out = out.p; a.ld_out = pad4(H);
                check(gdx_aggregate(&a, nullptr));
            }
        } else if (r_out) {
            Split A(n_local, width);
            a.width = width; a.src = h.p; a.ld_src = pad4(width);
            a.out_hi = A.hi.p; a.out_lo = A.lo.p; a.ld_split = A.ld;
            check(gdx_aggregate(&a, nullptr));
            g.a_hi = A.hi.p; g.a_lo = A.lo.p; g.lda = A.ld;
            g.b_hi = B.hi.p; g.b_lo = B.lo.p; g.ldb = B.ld;
            g.m = r_out; g.n = H; g.k = width; g.relu = 1;
            g.c0 = out.p; g.ldc0 = pad4(H); g.split = H;
            check(gdx_gemm_tn(&g, nullptr));
        }
        h = std::move(out);
        width = H;
    }
    cuda(cudaDeviceSynchronize(), "forward");
    *out_width = width;
    return h;
}

Dev<float> upload_features(const DenseFeatures& x) {
    const size_t ld = pad4(x.cols);
    std::vector<float> f(size_t(x.rows) * ld, 0.f);
    for (uint32_t r = 0; r < x.rows; ++r)
        for (uint32_t c = 0; c < x.cols; ++c) f[r * ld + c] = static_cast<float>(x.at(r, c));
    return Dev<float>(f.data(), f.size());
}

DenseFeatures download_rows(const Dev<float>& d, uint32_t rows, uint32_t width) {
    std::vector<float> h = d.download();
    DenseFeatures m(rows, width);
    const size_t ld = pad4(width);
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < width; ++c) m.at(r, c) = h[r * ld + c];
    return m;
}

void check_server(const Graph& g, const Partition& p, std::uint32_t server_id) {
    if (p.assignment.size() != g.num_vertices())
        throw InputError("extract: partition size does not match graph");
    if (server_id >= p.num_parts)
        throw InputError("extract: server id " + std::to_string(server_id) + " out of range (" +
                         std::to_string(p.num_parts) + " parts)");
}

Partition finish(std::vector<std::uint32_t> a, std::uint32_t parts) {
    Partition p;
    p.assignment = std::move(a);
    p.num_parts = parts;
    p.part_sizes.assign(parts, 0);
    for (std::uint32_t id : p.assignment) p.part_sizes[id]++;
    return p;
}

// Device hop loop (extract.cpp:135-182 / :87-113) -> subgraph with induced-edge count.
DependencySubgraph grow(const Graph& g, const Partition& p, std::uint32_t server, std::uint32_t max_hop,
                        std::uint32_t fanout, std::uint64_t seed, bool sampled) {
    const uint32_t n = g.num_vertices();
    const DevCSR& csr = upload(g);
    std::vector<uint8_t> inner(n);
    std::vector<uint32_t> mark(n);
    for (uint32_t v = 0; v < n; ++v) {
        inner[v] = p.assignment[v] == server;
        mark[v] = inner[v] ? 0u : GDX_UNSEEN;
    }
    Dev<uint8_t> dinner(inner.data(), n);
    Dev<uint32_t> dmark(mark.data(), n);
    Dev<uint32_t> work(size_t(3) * n + 64);
    check(gdx_sampled_growth(csr.rp.p, csr.col.p, n, dinner.p, nullptr, max_hop, fanout, seed, dmark.p,
                             work.p, nullptr));
    uint64_t induced = 0;
    Dev<unsigned long long> w64(1);
    check(gdx_induced_count(csr.rp.p, csr.col.p, n, dmark.p, w64.p, &induced, nullptr));
    mark = dmark.download();
    DependencySubgraph sub;
    sub.server_id = server;
    for (uint32_t v = 0; v < n; ++v) {
        if (mark[v] == 0) sub.inner_vertices.push_back(v);
        else if (mark[v] != GDX_UNSEEN) {
            sub.halo_vertices.push_back(v);
            sub.halo_hops.push_back(mark[v]);
        }
    }
    sub.induced_edges = induced;
    sub.hop_limit = max_hop;
    sub.sampled = sampled;
    return sub;
}

// Host-side SampleTrace: the reference attributes each taken vertex to the first
// frontier vertex (ascending) exposing it, hop by hop.  The device result fixes
// the frontiers; the attribution is recomputed here only when a trace is asked
// for (diagnostics; extract.hpp:49-54).
void build_trace(const Graph& g, const std::vector<uint8_t>& inner, const DependencySubgraph& sub,
                 const SamplingConfig& cfg, SampleTrace* trace) {
    (void)sub;
    const uint32_t n = g.num_vertices();
    const uint32_t* cols = g.col_indices().empty() ? nullptr : g.col_indices().data();
    uint64_t ns = 0, nt = 0;
    check(gdx_host_sample_trace(n, g.row_offsets().data(), cols, inner.data(), cfg.max_hop, cfg.fanout, cfg.seed,
                                0, 0, &ns, &nt, nullptr, nullptr, nullptr, nullptr));
    std::vector<uint32_t> sv(std::max<uint64_t>(ns, 1)), sh(std::max<uint64_t>(ns, 1)), tk(std::max<uint64_t>(nt, 1));
    std::vector<uint64_t> so(ns + 1);
    check(gdx_host_sample_trace(n, g.row_offsets().data(), cols, inner.data(), cfg.max_hop, cfg.fanout, cfg.seed,
                                ns, nt, &ns, &nt, sv.data(), sh.data(), so.data(), tk.data()));
    for (uint64_t i = 0; i < ns; ++i)
        trace->push_back({sv[i], sh[i], std::vector<VertexId>(tk.begin() + so[i], tk.begin() + so[i + 1])});
}

// G(n,p) scan of graph.cpp:86-111 for the planted generator (host preprocessing)
template <class Emit>
void sample_range(std::uint64_t seed, VertexId u, VertexId start, VertexId limit, double p,
                  std::uint64_t tag, Emit&& emit) {
    if (p <= 0.0 || start >= limit) return;
    KeyedRng rng(seed, u, tag);
    const double log1mp = (p < 1.0) ? std::log1p(-p) : 0.0;
    auto skip = [&]() -> std::uint64_t {
        if (p >= 1.0) return 0;
        double r = rng.next_double();
        if (r <= 0.0) r = 0x1.0p-53;
        double s = std::floor(std::log(r) / log1mp);
        if (s < 0.0) s = 0.0;
        if (s > 1e18) s = 1e18;
        return static_cast<std::uint64_t>(s);
    };
    std::uint64_t v = start + skip();
    while (v < limit) {
        emit(static_cast<VertexId>(v));
        v += 1 + skip();
    }
}

}  // namespace

// ======================= graph ==========================================
Graph Graph::from_csr(VertexId n, std::vector<EdgeIndex> offsets, std::vector<VertexId> cols,
                      bool undirected) {
    Graph g;
    g.n_ = n;
    g.offsets_ = std::move(offsets);
    g.cols_ = std::move(cols);
    g.undirected_ = undirected;
    return g;
}

// graph.cpp:25-67 semantics: self loops dropped, rows sorted and deduplicated
Graph Graph::from_edges(const std::vector<std::pair<VertexId, VertexId>>& edges, VertexId n,
                        bool undirected) {
    if (n == 0) throw InputError("graph must have at least one vertex");
    std::vector<std::vector<VertexId>> rows(n);
    for (const auto& [u, v] : edges) {
        if (u >= n || v >= n)
            throw InputError("edge endpoint " + std::to_string(std::max(u, v)) + " out of range for " +
                             std::to_string(n) + " vertices");
    }
    for (const auto& [u, v] : edges) {
        if (u == v) continue;
        rows[u].push_back(v);
        if (undirected) rows[v].push_back(u);
    }
    std::vector<EdgeIndex> off(n + 1, 0);
    std::vector<VertexId> cols;
    for (VertexId v = 0; v < n; ++v) {
        std::sort(rows[v].begin(), rows[v].end());
        rows[v].erase(std::unique(rows[v].begin(), rows[v].end()), rows[v].end());
        cols.insert(cols.end(), rows[v].begin(), rows[v].end());
        off[v + 1] = cols.size();
    }
    return from_csr(n, std::move(off), std::move(cols), undirected);
}

Graph gen_random_graph(VertexId n, double avg_degree, std::uint64_t seed) {
    if (n == 0) throw InputError("gen_random_graph: n must be >= 1");
    if (avg_degree < 0.0) throw InputError("gen_random_graph: avg_degree must be >= 0");
    if (avg_degree >= static_cast<double>(n))
        throw InputError("gen_random_graph: avg_degree " + std::to_string(avg_degree) +
                         " >= n, simple graph impossible");
    std::vector<EdgeIndex> off(n + 1);
    const uint64_t nnz = gdx_host_gen_random_graph_count(n, avg_degree, seed, off.data());
    std::vector<VertexId> cols(nnz);
    check(gdx_host_gen_random_graph_fill(n, avg_degree, seed, off.data(), cols.data()));
    return Graph::from_csr(n, std::move(off), std::move(cols), true);
}

std::uint32_t planted_block_of(VertexId v, VertexId n, std::uint32_t parts) {
    return static_cast<std::uint32_t>(((static_cast<std::uint64_t>(v) + 1) * parts - 1) / n);
}

// graph.cpp:156-185: within-block p_in (tag 1), cross-block p_out (tag 2)
Graph gen_planted_partition_graph(VertexId n, std::uint32_t parts, double p_in, double p_out,
                                  std::uint64_t seed) {
    if (n == 0) throw InputError("gen_planted_partition_graph: n must be >= 1");
    if (parts == 0 || parts > n) throw InputError("gen_planted_partition_graph: parts must be in [1, n]");
    if (p_in < 0.0 || p_in > 1.0 || p_out < 0.0 || p_out > 1.0)
        throw InputError("gen_planted_partition_graph: probabilities must lie in [0, 1]");
    std::vector<std::vector<VertexId>> rows(n);
    for (VertexId u = 0; u + 1 < n; ++u) {
        const VertexId be = static_cast<VertexId>(
            (static_cast<std::uint64_t>(planted_block_of(u, n, parts)) + 1) * n / parts);
        auto emit = [&](VertexId v) {
            rows[u].push_back(v);
            rows[v].push_back(u);
        };
        sample_range(seed, u, u + 1, be, p_in, 1, emit);
        sample_range(seed, u, be, n, p_out, 2, emit);
    }
    std::vector<EdgeIndex> off(n + 1, 0);
    std::vector<VertexId> cols;
    for (VertexId v = 0; v < n; ++v) {
        cols.insert(cols.end(), rows[v].begin(), rows[v].end());  // already ascending
        off[v + 1] = cols.size();
    }
    return Graph::from_csr(n, std::move(off), std::move(cols), true);
}

// ======================= partition ======================================
std::vector<VertexId> Partition::members(std::uint32_t part) const {
    std::vector<VertexId> out;
    for (VertexId v = 0; v < assignment.size(); ++v)
        if (assignment[v] == part) out.push_back(v);
    return out;
}

Partition partition_random(const Graph& g, std::uint32_t parts, std::uint64_t seed) {
    std::vector<std::uint32_t> a(g.num_vertices());
    check(gdx_host_partition_random(g.num_vertices(), parts, seed, a.data()));
    return finish(std::move(a), parts);
}

Partition partition_mincut(const Graph& g, std::uint32_t parts, std::uint64_t seed, double eps) {
    std::vector<std::uint32_t> a(std::max<VertexId>(g.num_vertices(), 1));
    check(gdx_host_partition_mincut(g.num_vertices(), g.row_offsets().data(), g.col_indices().data(),
                                    parts, seed, eps, a.data()));
    a.resize(g.num_vertices());
    return finish(std::move(a), parts);
}

InducedSubgraph induced_subgraph(const Graph& g, std::span<const VertexId> vs) {
    InducedSubgraph out;
    out.global_ids.assign(vs.begin(), vs.end());
    std::vector<std::int64_t> local(g.num_vertices(), -1);
    for (size_t i = 0; i < vs.size(); ++i) local[vs[i]] = static_cast<std::int64_t>(i);
    std::vector<EdgeIndex> off(vs.size() + 1, 0);
    std::vector<VertexId> cols;
    for (size_t i = 0; i < vs.size(); ++i) {
        for (VertexId u : g.neighbors(vs[i]))
            if (local[u] >= 0) cols.push_back(static_cast<VertexId>(local[u]));
        off[i + 1] = cols.size();
    }
    out.graph = Graph::from_csr(static_cast<VertexId>(vs.size()), std::move(off), std::move(cols), true);
    return out;
}

HierarchicalPartition hierarchical_partition(const Graph& g, std::uint32_t servers,
                                             std::uint32_t gpus_per_server, PartitionMode mode,
                                             std::uint64_t seed, double eps) {
    if (servers == 0 || gpus_per_server == 0)
        throw InputError("hierarchical_partition: servers and gpus_per_server must be >= 1");
    if (static_cast<std::uint64_t>(servers) * gpus_per_server > g.num_vertices())
        throw InputError("hierarchical_partition: more workers than vertices");
    auto run = [&](const Graph& gr, std::uint32_t parts, std::uint64_t s) {
        return mode == PartitionMode::Random ? partition_random(gr, parts, s)
                                             : partition_mincut(gr, parts, s, eps);
    };
    HierarchicalPartition h;
    h.gpus_per_server = gpus_per_server;
    h.server = run(g, servers, seed);
    std::vector<std::uint32_t> gpu(g.num_vertices(), 0);
    for (std::uint32_t s = 0; s < servers; ++s) {
        std::vector<VertexId> inner = h.server.members(s);
        InducedSubgraph sub = induced_subgraph(g, inner);
        Partition local = run(sub.graph, gpus_per_server, mix64(seed ^ (s + 1)));
        for (VertexId i = 0; i < sub.global_ids.size(); ++i)
            gpu[sub.global_ids[i]] = s * gpus_per_server + local.assignment[i];
    }
    h.gpu = finish(std::move(gpu), servers * gpus_per_server);
    return h;
}

// ======================= extraction =====================================
bool DependencySubgraph::is_inner(VertexId v) const {
    return std::binary_search(inner_vertices.begin(), inner_vertices.end(), v);
}
bool DependencySubgraph::is_halo(VertexId v) const {
    return std::binary_search(halo_vertices.begin(), halo_vertices.end(), v);
}
std::uint32_t DependencySubgraph::hop_of(VertexId v) const {
    if (is_inner(v)) return 0;
    auto it = std::lower_bound(halo_vertices.begin(), halo_vertices.end(), v);
    if (it == halo_vertices.end() || *it != v)
        throw InputError("hop_of: vertex " + std::to_string(v) + " not in subgraph");
    return halo_hops[static_cast<size_t>(it - halo_vertices.begin())];
}
std::vector<VertexId> DependencySubgraph::all_vertices() const {
    std::vector<VertexId> out;
    out.reserve(inner_vertices.size() + halo_vertices.size());
    std::merge(inner_vertices.begin(), inner_vertices.end(), halo_vertices.begin(), halo_vertices.end(),
               std::back_inserter(out));
    return out;
}

DependencySubgraph extract_full(const Graph& g, const Partition& p, std::uint32_t server,
                                std::uint32_t layers) {
    check_server(g, p, server);
    return grow(g, p, server, layers, kUnlimitedFanout, 0, false);
}

DependencySubgraph extract_sampled(const Graph& g, const Partition& p, std::uint32_t server,
                                   const SamplingConfig& cfg, SampleTrace* trace) {
    check_server(g, p, server);
    DependencySubgraph sub = grow(g, p, server, cfg.max_hop, cfg.fanout, cfg.seed, !cfg.unlimited());
    if (trace) {
        std::vector<uint8_t> inner(g.num_vertices(), 0);
        for (VertexId v : sub.inner_vertices) inner[v] = 1;
        build_trace(g, inner, sub, cfg, trace);
    }
    return sub;
}

std::vector<std::pair<std::uint32_t, std::uint64_t>> neighbor_explosion_profile(
    const Graph& g, const Partition& p, std::uint32_t server, std::uint32_t max_layers) {
    if (max_layers == 0) throw InputError("neighbor_explosion_profile: max_layers must be >= 1");
    check_server(g, p, server);
    DependencySubgraph deep = extract_full(g, p, server, max_layers);
    std::vector<std::uint64_t> added(max_layers + 1, 0);
    for (std::uint32_t h : deep.halo_hops) added[h]++;
    std::vector<std::pair<std::uint32_t, std::uint64_t>> out;
    std::uint64_t size = deep.inner_vertices.size();
    for (std::uint32_t l = 1; l <= max_layers; ++l) {
        size += added[l];
        out.emplace_back(l, size);
    }
    return out;
}

// ======================= reference GNN ==================================
DenseFeatures make_features(VertexId n, std::uint32_t dim, std::uint64_t seed) {
    Matrix m(n, dim);
    if (!n || !dim) return m;
    Dev<double> d(size_t(n) * dim, false);
    check(gdx_init_uniform_f64(seed, 0x66656174ULL, 0, 0, n, dim, -0.5, 0.5, d.p, dim, nullptr));
    m.data = d.download();
    return m;
}

LayerWeights make_layer_weights(std::uint32_t num_layers, std::uint32_t F, std::uint32_t H,
                                std::uint64_t seed) {
    if (F == 0 || H == 0) throw InputError("make_layer_weights: dimensions must be >= 1");
    LayerWeights w;
    std::uint64_t first = 0;
    for (std::uint32_t l = 0; l < num_layers; ++l) {
        const std::uint32_t in = l == 0 ? F : H;
        Matrix m(H, in);
        Dev<double> d(size_t(H) * in, false);
        check(gdx_init_uniform_f64(seed, 0x77656967ULL, 0, first, H, in, -0.5, 0.5, d.p, in, nullptr));
        m.data = d.download();
        first += std::uint64_t(H) * in;
        w.layers.push_back(std::move(m));
    }
    return w;
}

DenseFeatures forward_full(const Graph& g, const DenseFeatures& x, const LayerWeights& w,
                           std::uint32_t layers) {
    if (x.rows != g.num_vertices()) throw InputError("forward_full: feature rows do not match vertex count");
    check_shapes(x, w, layers);
    if (layers == 0) return x;
    const DevCSR& csr = upload(g);
    const uint32_t n = g.num_vertices();
    uint32_t width = 0;
    Dev<float> out = run_layers(csr, n, upload_features(x), x.cols, w, layers,
                                std::vector<uint32_t>(layers, n), std::vector<uint32_t>(layers, n), &width);
    return download_rows(out, n, width);
}

DenseFeatures forward_server_local(const DependencySubgraph& sub, const Graph& g,
                                   const DenseFeatures& x, const LayerWeights& w,
                                   std::uint32_t layers, bool require_exact) {
    if (x.rows != g.num_vertices())
        throw InputError("forward_server_local: feature rows do not match vertex count");
    check_shapes(x, w, layers);
    if (require_exact && (sub.sampled || sub.hop_limit < layers))
        throw ContractError("forward_server_local: subgraph too shallow or sampled for exact " +
                            std::to_string(layers) + "-layer computation");
    const uint32_t n = g.num_vertices();
    if (layers == 0) {  // no layer runs: the inner rows verbatim (reference_gnn.cpp:140-146)
        DenseFeatures out(static_cast<uint32_t>(sub.inner_vertices.size()), x.cols);
        for (VertexId r = 0; r < sub.inner_vertices.size(); ++r)
            std::copy(x.row(sub.inner_vertices[r]).begin(), x.row(sub.inner_vertices[r]).end(),
                      out.row(r).begin());
        return out;
    }
    std::vector<uint32_t> hop(n, GDX_UNSEEN);
    for (VertexId v : sub.inner_vertices) hop[v] = 0;
    uint32_t max_hop = 0;
    for (size_t i = 0; i < sub.halo_vertices.size(); ++i) {
        hop[sub.halo_vertices[i]] = sub.halo_hops[i];
        max_hop = std::max(max_hop, sub.halo_hops[i]);
    }
    const DevCSR& gcsr = upload(g);
    Dev<uint32_t> dhop(hop.data(), n);
    Dev<uint32_t> l2g(n), local_of(n);
    std::vector<uint64_t> hop_start(max_hop + 2, 0);
    uint32_t local_n = 0;
    check(gdx_order_by_hop(dhop.p, n, max_hop, l2g.p, local_of.p, hop_start.data(), &local_n, nullptr));
    Dev<uint64_t> counts(std::max(local_n, 1u));
    check(gdx_local_csr(gcsr.rp.p, gcsr.col.p, l2g.p, local_n, local_of.p, counts.p, nullptr, nullptr, nullptr));
    DevCSR lcsr;
    lcsr.rp = Dev<uint64_t>(size_t(local_n) + 1);
    uint64_t total = 0;
    check(gdx_exclusive_scan_u64(counts.p, local_n, lcsr.rp.p, &total, nullptr));
    lcsr.col = Dev<uint32_t>(std::max<uint64_t>(total, 1));
    check(gdx_local_csr(gcsr.rp.p, gcsr.col.p, l2g.p, local_n, local_of.p, nullptr, lcsr.rp.p, lcsr.col.p,
                        nullptr));
    lcsr.rows = local_n;
    auto upto = [&](std::int64_t h) -> uint32_t {
        if (h < 0) return 0;
        return static_cast<uint32_t>(hop_start[std::min<std::int64_t>(h, max_hop) + 1]);
    };
    // layer-1 inputs: rows with hop <= L gathered, others zero
    Dev<float> xg = upload_features(x);
    Dev<float> h(size_t(std::max(local_n, 1u)) * pad4(x.cols));
    const uint32_t first = upto(layers);
    if (first) check(gdx_gather_rows(xg.p, pad4(x.cols), l2g.p, first, x.cols, h.p, pad4(x.cols), nullptr));
    std::vector<uint32_t> rin(layers), rout(layers);
    for (std::uint32_t l = 0; l < layers; ++l) {
        rin[l] = upto(std::int64_t(layers) - l);
        rout[l] = upto(std::int64_t(layers) - l - 1);
    }
    uint32_t width = x.cols;
    Dev<float> out = layers ? run_layers(lcsr, local_n, std::move(h), x.cols, w, layers, rin, rout, &width)
                            : std::move(h);
    cuda(cudaDeviceSynchronize(), "forward_server_local");
    return download_rows(out, upto(0), width);
}

EquivalenceReport equivalence_check(const Graph& g, const Partition& p, std::uint32_t layers,
                                    std::uint64_t seed, std::uint32_t F, std::uint32_t H) {
    DenseFeatures x = make_features(g.num_vertices(), F, seed);
    LayerWeights w = make_layer_weights(layers, F, H, mix64(seed + 1));
    DenseFeatures full = forward_full(g, x, w, layers);
    EquivalenceReport rep;
    for (std::uint32_t s = 0; s < p.num_parts; ++s) {
        DependencySubgraph sub = extract_full(g, p, s, layers);
        DenseFeatures local = forward_server_local(sub, g, x, w, layers, true);
        double dev = 0.0;
        for (VertexId r = 0; r < sub.inner_vertices.size(); ++r)
            for (std::uint32_t c = 0; c < local.cols; ++c)
                dev = std::max(dev, std::abs(local.at(r, c) - full.at(sub.inner_vertices[r], c)));
        rep.per_server_max_dev.push_back(dev);
        rep.max_deviation = std::max(rep.max_deviation, dev);
    }
    return rep;
}

// ======================= cooperative batch planning ========================
std::uint64_t estimate_batch_memory(const Batch& b, const ModelSpec& model) {
    std::uint64_t bytes = 0;
    for (std::size_t l = 0; l < b.mfg_vertices_per_layer.size(); ++l)
        bytes += b.mfg_vertices_per_layer[l] * (l == 0 ? model.feature_dim : model.hidden_dim) * kBytesPerScalar;
    return bytes;
}

namespace {

// Target groups of one R (batch_plan.cpp:114-126): the inner vertices split by the
// host min-cut of their induced subgraph (bit-identical to the reference's).
std::vector<std::vector<VertexId>> target_groups(const Graph& g, const std::vector<VertexId>& targets,
                                                 std::uint32_t r, std::uint64_t seed) {
    if (r <= 1 || targets.size() <= 1) return {targets};
    InducedSubgraph inner = induced_subgraph(g, targets);
    Partition p = partition_mincut(inner.graph, r, seed);
    std::vector<std::vector<VertexId>> groups(r);
    for (VertexId i = 0; i < inner.global_ids.size(); ++i) groups[p.assignment[i]].push_back(inner.global_ids[i]);
    for (auto& grp : groups) std::sort(grp.begin(), grp.end());
    return groups;
}

// The planner's device context: graph + server universe resident for the whole R scan.
struct PlanDevice {
    const DevCSR& csr;
    Dev<uint8_t> universe;
    uint32_t n = 0;
    PlanDevice(const Graph& g, const DependencySubgraph& sub) : csr(upload(g)), n(g.num_vertices()) {
        std::vector<uint8_t> u(n, 0);
        for (VertexId v : sub.inner_vertices) u[v] = 1;
        for (VertexId v : sub.halo_vertices) u[v] = 1;
        universe = Dev<uint8_t>(u.data(), n);
    }
};

uint64_t workspace_budget() {
    size_t free_b = 0, total = 0;
    if (cudaMemGetInfo(&free_b, &total) != cudaSuccess) return 1ull << 28;
    return std::max<uint64_t>(1ull << 26, std::min<uint64_t>(free_b / 4, 32ull << 30));
}

// One batched device evaluation of every group (gdx_cobatch_eval).  With plan: the
// batches (vertex lists included) are written into it.
std::vector<std::vector<std::uint64_t>> eval_groups(const PlanDevice& d,
                                                    const std::vector<std::vector<VertexId>>& groups,
                                                    std::uint32_t layers, const SamplingConfig& cfg,
                                                    const ModelSpec& model, BatchPlan* plan) {
    const uint32_t G = static_cast<uint32_t>(groups.size());
    std::vector<uint64_t> off(G + 1, 0);
    std::vector<uint32_t> flat;
    for (uint32_t i = 0; i < G; ++i) {
        flat.insert(flat.end(), groups[i].begin(), groups[i].end());
        off[i + 1] = flat.size();
    }
    Dev<uint32_t> t(flat.data(), flat.size());
    std::vector<uint64_t> sizes(G), mfg(size_t(G) * (layers + 1));
    const uint64_t ws = workspace_budget();
    check(gdx_cobatch_eval(d.csr.rp.p, d.csr.col.p, d.n, d.universe.p, t.p, off.data(), G, cfg.max_hop,
                           cfg.fanout, cfg.seed, layers, ws, sizes.data(), mfg.data(), nullptr, nullptr,
                           nullptr));
    std::vector<std::vector<std::uint64_t>> counts(G);
    for (uint32_t i = 0; i < G; ++i)
        counts[i].assign(mfg.begin() + size_t(i) * (layers + 1), mfg.begin() + size_t(i + 1) * (layers + 1));
    if (plan) {
        std::vector<uint64_t> voff(G + 1, 0);
        for (uint32_t i = 0; i < G; ++i) voff[i + 1] = voff[i] + sizes[i];
        Dev<uint32_t> verts(std::max<uint64_t>(voff[G], 1), false);
        check(gdx_cobatch_eval(d.csr.rp.p, d.csr.col.p, d.n, d.universe.p, t.p, off.data(), G, cfg.max_hop,
                               cfg.fanout, cfg.seed, layers, ws, sizes.data(), mfg.data(), verts.p,
                               voff.data(), nullptr));
        std::vector<uint32_t> hv = verts.download();
        for (uint32_t i = 0; i < G; ++i) {
            Batch b;
            b.target_vertices = groups[i];
            b.vertices.assign(hv.begin() + voff[i], hv.begin() + voff[i + 1]);
            b.mfg_vertices_per_layer = counts[i];
            b.est_memory_bytes = estimate_batch_memory(b, model);
            plan->batches.push_back(std::move(b));
        }
    }
    return counts;
}

BatchPlan empty_plan(const DependencySubgraph& sub, std::uint32_t layers) {
    BatchPlan plan;
    plan.worker_id = sub.server_id;
    plan.strategy = BatchStrategy::FetchThenSplit;
    plan.layers = layers;
    return plan;
}

[[noreturn]] void capacity_failure(const std::vector<VertexId>& worst_targets, std::uint64_t bytes,
                                   std::uint64_t budget) {
    throw CapacityError("single-target batch for vertex " +
                        std::to_string(worst_targets.empty() ? 0 : worst_targets.front()) + " needs " +
                        std::to_string(bytes) + " bytes, budget is " + std::to_string(budget));
}

}  // namespace

BatchPlan plan_cobatch_fixed_r(const DependencySubgraph& sub, const Graph& g, std::uint32_t layers,
                               const SamplingConfig& cfg, std::uint32_t r, const ModelSpec& model) {
    if (r == 0) throw InputError("plan_cobatch: batch count must be >= 1");
    const std::uint32_t capped =
        std::min<std::uint32_t>(r, std::max<std::uint32_t>(1, static_cast<std::uint32_t>(sub.inner_vertices.size())));
    PlanDevice d(g, sub);
    BatchPlan plan = empty_plan(sub, layers);
    eval_groups(d, target_groups(g, sub.inner_vertices, capped, cfg.seed), layers, cfg, model, &plan);
    return plan;
}

// batch_plan.cpp:155-180: the reference's linear scan over R (the worst batch's bytes
// are not monotone in R); each R is one batched device evaluation, only the first R
// that fits is materialised.
BatchPlan plan_cobatch(const DependencySubgraph& sub, const Graph& g, std::uint32_t layers,
                       const SamplingConfig& cfg, std::uint64_t mem_budget, const ModelSpec& model) {
    if (mem_budget == 0) throw InputError("plan_cobatch: mem_budget must be > 0");
    const std::uint32_t max_r = std::max<std::uint32_t>(1, static_cast<std::uint32_t>(sub.inner_vertices.size()));
    PlanDevice d(g, sub);
    std::vector<std::vector<VertexId>> groups;
    std::uint64_t worst = 0;
    std::size_t worst_i = 0;
    for (std::uint32_t r = 1; r <= max_r; ++r) {
        groups = target_groups(g, sub.inner_vertices, r, cfg.seed);
        auto counts = eval_groups(d, groups, layers, cfg, model, nullptr);
        worst = 0;
        worst_i = 0;
        for (std::size_t i = 0; i < counts.size(); ++i) {
            Batch b;
            b.mfg_vertices_per_layer = counts[i];
            const std::uint64_t bytes = estimate_batch_memory(b, model);
            if (bytes > worst) {
                worst = bytes;
                worst_i = i;
            }
        }
        if (worst <= mem_budget) {
            BatchPlan plan = empty_plan(sub, layers);
            eval_groups(d, groups, layers, cfg, model, &plan);
            return plan;
        }
    }
    capacity_failure(groups[worst_i], worst, mem_budget);
}

// The split-then-fetch baseline (the planner the paper compares against): each chunk
// of the GPU's own vertices grows GraphSAGE-style layered dependency sets from the
// whole graph -- at every step each vertex already in the set keeps at most
// fanout_per_layer neighbours of its (seed, vertex, layer)-keyed permutation.  Host
// code: a visited stamp per vertex (no O(V) clearing per batch), one scan per chunk.
BatchPlan plan_minibatch_baseline(const Graph& g, const Partition& gpu_partition, std::uint32_t gpu_id,
                                  std::uint32_t layers, std::uint32_t fanout_per_layer,
                                  std::uint64_t mem_budget, const ModelSpec& model, std::uint64_t seed) {
    if (mem_budget == 0) throw InputError("plan_minibatch_baseline: mem_budget must be > 0");
    if (gpu_id >= gpu_partition.num_parts) throw InputError("plan_minibatch_baseline: gpu id out of range");
    const std::vector<VertexId> own = gpu_partition.members(gpu_id);
    std::vector<std::uint32_t> stamp(g.num_vertices(), 0);
    std::uint32_t epoch = 0;
    auto build = [&](std::vector<VertexId> targets) {
        ++epoch;
        Batch b;
        b.target_vertices = std::move(targets);
        std::vector<VertexId> set = b.target_vertices;
        for (VertexId v : set) stamp[v] = epoch;
        b.mfg_vertices_per_layer.assign(layers + 1, 0);
        b.mfg_vertices_per_layer[layers] = set.size();
        std::vector<VertexId> picks;
        for (std::uint32_t step = 1; step <= layers; ++step) {
            const std::uint32_t key = layers - step + 1;
            const std::size_t before = set.size();
            for (std::size_t i = 0; i < before; ++i) {
                const auto nb = g.neighbors(set[i]);
                picks.assign(nb.begin(), nb.end());
                if (fanout_per_layer != kUnlimitedFanout && picks.size() > fanout_per_layer) {
                    KeyedRng rng(seed, set[i], key);
                    keyed_shuffle(picks, rng);
                    picks.resize(fanout_per_layer);
                }
                for (VertexId u : picks)
                    if (stamp[u] != epoch) {
                        stamp[u] = epoch;
                        set.push_back(u);
                    }
            }
            b.mfg_vertices_per_layer[layers - step] = set.size();
        }
        std::sort(set.begin(), set.end());
        b.vertices = std::move(set);
        b.est_memory_bytes = estimate_batch_memory(b, model);
        return b;
    };
    BatchPlan plan;
    plan.worker_id = gpu_id;
    plan.strategy = BatchStrategy::SplitThenFetch;
    plan.layers = layers;
    const std::uint32_t max_r = std::max<std::uint32_t>(1, static_cast<std::uint32_t>(own.size()));
    for (std::uint32_t r = 1; r <= max_r; ++r) {
        plan.batches.clear();
        std::uint64_t worst = 0;
        const std::size_t base = own.size() / r, rem = own.size() % r;
        std::size_t pos = 0;
        for (std::uint32_t i = 0; i < r; ++i) {
            const std::size_t len = base + (i < rem ? 1 : 0);
            plan.batches.push_back(build({own.begin() + pos, own.begin() + pos + len}));
            pos += len;
            worst = std::max(worst, plan.batches.back().est_memory_bytes);
        }
        if (worst <= mem_budget) return plan;
    }
    const Batch* w = &plan.batches.front();
    for (const Batch& b : plan.batches)
        if (b.est_memory_bytes > w->est_memory_bytes) w = &b;
    capacity_failure(w->target_vertices, w->est_memory_bytes, mem_budget);
}

std::string plan_to_json(const BatchPlan& plan) {
    std::string o = "{\n  \"worker_id\": " + std::to_string(plan.worker_id) + ",\n  \"strategy\": \"" +
                    (plan.strategy == BatchStrategy::FetchThenSplit ? "fetch_then_split" : "split_then_fetch") +
                    "\",\n  \"layers\": " + std::to_string(plan.layers) + ",\n  \"batch_count\": " +
                    std::to_string(plan.batch_count()) + ",\n  \"batches\": [";
    for (std::size_t i = 0; i < plan.batches.size(); ++i) {
        const Batch& b = plan.batches[i];
        o += (i ? ",\n    {" : "\n    {");
        o += "\"targets\": " + std::to_string(b.target_vertices.size()) + ", \"vertices\": " +
             std::to_string(b.vertices.size()) + ", \"mfg_vertices_per_layer\": [";
        for (std::size_t l = 0; l < b.mfg_vertices_per_layer.size(); ++l)
            o += (l ? ", " : "") + std::to_string(b.mfg_vertices_per_layer[l]);
        o += "], \"est_memory_bytes\": " + std::to_string(b.est_memory_bytes) + "}";
    }
    o += plan.batches.empty() ? "]\n}" : "\n  ]\n}";
    return o;
}

void save_plan_json(const BatchPlan& plan, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw InputError("cannot open output file: " + path);
    const std::string s = plan_to_json(plan);
    std::fputs(s.c_str(), f);
    std::fputs("\n", f);
    std::fclose(f);
}

// ======================= cooperative split ================================
std::vector<std::vector<VertexId>> split_batch(const std::vector<VertexId>& bv, const Partition& sp,
                                               const Partition& gp, std::uint32_t server,
                                               std::uint32_t gpus) {
    std::vector<std::vector<VertexId>> shares(gpus);
    if (bv.empty()) return shares;
    Dev<uint32_t> dbv(bv.data(), bv.size()), dsp(sp.assignment.data(), sp.assignment.size()),
        dgp(gp.assignment.data(), gp.assignment.size()), share(bv.size()), work(5 * bv.size() + 2 * gpus + 8);
    check(gdx_split_batch(dbv.p, bv.size(), dsp.p, dgp.p, server, gpus, share.p, work.p, nullptr));
    std::vector<uint32_t> s = share.download();
    for (size_t i = 0; i < bv.size(); ++i) shares[s[i]].push_back(bv[i]);  // bv ascending
    return shares;
}

}  // namespace granndis
