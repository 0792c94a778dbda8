// ref_shim.cpp -- extern "C" bridge onto the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles the reference sources in
// place (/root/reference/proj/src/*.cpp, never copied) together with this file
// into oracle/_ref/libgranndis_ref.so.  Tests call it through ctypes to pin the
// C restatement (granndis_oracle.c) and to generate golden fixtures; bench.py
// --impl reference times the reference's own forward_full through it.
//
// Graphs, partitions, subgraphs and plans cross the boundary as opaque heap
// handles with copy-out accessors; errors are caught and reported as the
// reference's category string (errors.hpp:11-44) via grr_last_error().

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "granndis/batch_plan.hpp"
#include "granndis/errors.hpp"
#include "granndis/extract.hpp"
#include "granndis/graph.hpp"
#include "granndis/partition.hpp"
#include "granndis/reference_gnn.hpp"
#include "granndis/rng.hpp"
#include "granndis/sim.hpp"

namespace granndis {
// Defined in graph.cpp (friend of Graph); declared here to wrap a caller CSR.
Graph make_csr_direct(VertexId n, std::vector<EdgeIndex> offsets, std::vector<VertexId> cols,
                      bool undirected);
}  // namespace granndis

using namespace granndis;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const CapacityError& e) {
        g_err = std::string("capacity: ") + e.what();
        return 2;
    } catch (const ContractError& e) {
        g_err = std::string("contract: ") + e.what();
        return 3;
    } catch (const Error& e) {
        g_err = e.category() + ": " + e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = std::string("internal: ") + e.what();
        return 4;
    }
}

Partition make_partition(const std::uint32_t* assign, std::uint32_t n, std::uint32_t parts) {
    Partition p;
    p.assignment.assign(assign, assign + n);
    p.num_parts = parts;
    p.part_sizes.assign(parts, 0);
    for (std::uint32_t i = 0; i < n; ++i) p.part_sizes[assign[i]]++;
    return p;
}

void hops_out(const Graph& g, const DependencySubgraph& sub, std::uint32_t* hop) {
    for (VertexId v = 0; v < g.num_vertices(); ++v) hop[v] = 0xFFFFFFFFu;
    for (VertexId v : sub.inner_vertices) hop[v] = 0;
    for (std::size_t i = 0; i < sub.halo_vertices.size(); ++i)
        hop[sub.halo_vertices[i]] = sub.halo_hops[i];
}

DependencySubgraph sub_from_hops(const Graph& g, const std::uint32_t* hop, std::uint32_t server,
                                 std::uint32_t hop_limit, int sampled) {
    DependencySubgraph sub;
    sub.server_id = server;
    for (VertexId v = 0; v < g.num_vertices(); ++v) {
        if (hop[v] == 0) sub.inner_vertices.push_back(v);
        else if (hop[v] != 0xFFFFFFFFu) {
            sub.halo_vertices.push_back(v);
            sub.halo_hops.push_back(hop[v]);
        }
    }
    sub.hop_limit = hop_limit;
    sub.sampled = sampled != 0;
    return sub;
}

Matrix to_matrix(const double* x, std::uint32_t rows, std::uint32_t cols) {
    Matrix m(rows, cols);
    std::memcpy(m.data.data(), x, sizeof(double) * std::size_t(rows) * cols);
    return m;
}

LayerWeights to_weights(const double* w, std::uint32_t layers, std::uint32_t F, std::uint32_t H) {
    LayerWeights lw;
    for (std::uint32_t l = 0; l < layers; ++l) {
        std::uint32_t in = l == 0 ? F : H;
        lw.layers.push_back(to_matrix(w, H, in));
        w += std::size_t(H) * in;
    }
    return lw;
}
}  // namespace

extern "C" {

const char* grr_last_error() { return g_err.c_str(); }

// ---- graphs -------------------------------------------------------------
void* grr_gen_random_graph(std::uint32_t n, double d, std::uint64_t seed) {
    Graph* out = nullptr;
    if (guarded([&] { out = new Graph(gen_random_graph(n, d, seed)); })) return nullptr;
    return out;
}
void* grr_gen_planted(std::uint32_t n, std::uint32_t parts, double pin, double pout,
                      std::uint64_t seed) {
    Graph* out = nullptr;
    if (guarded([&] { out = new Graph(gen_planted_partition_graph(n, parts, pin, pout, seed)); }))
        return nullptr;
    return out;
}
void* grr_graph_from_edges(const std::uint32_t* edges, std::uint64_t m, std::uint32_t n) {
    Graph* out = nullptr;
    std::vector<std::pair<VertexId, VertexId>> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {edges[2 * i], edges[2 * i + 1]};
    if (guarded([&] { out = new Graph(Graph::from_edges(e, n, true)); })) return nullptr;
    return out;
}
void* grr_graph_from_csr(std::uint32_t n, const std::uint64_t* ro, const std::uint32_t* ci) {
    std::vector<EdgeIndex> off(ro, ro + n + 1);
    std::vector<VertexId> cols(ci, ci + ro[n]);
    return new Graph(make_csr_direct(n, std::move(off), std::move(cols), true));
}
std::uint32_t grr_graph_n(void* g) { return static_cast<Graph*>(g)->num_vertices(); }
std::uint64_t grr_graph_nnz(void* g) { return static_cast<Graph*>(g)->num_edges(); }
void grr_graph_copy(void* h, std::uint64_t* ro, std::uint32_t* ci) {
    const Graph& g = *static_cast<Graph*>(h);
    std::memcpy(ro, g.row_offsets().data(), sizeof(std::uint64_t) * (g.num_vertices() + 1));
    std::memcpy(ci, g.col_indices().data(), sizeof(std::uint32_t) * g.num_edges());
}
void grr_graph_free(void* g) { delete static_cast<Graph*>(g); }

// ---- partitions -----------------------------------------------------------
int grr_partition_random(void* g, std::uint32_t parts, std::uint64_t seed, std::uint32_t* out) {
    return guarded([&] {
        Partition p = partition_random(*static_cast<Graph*>(g), parts, seed);
        std::memcpy(out, p.assignment.data(), sizeof(std::uint32_t) * p.assignment.size());
    });
}
int grr_partition_mincut(void* g, std::uint32_t parts, std::uint64_t seed, double eps,
                         std::uint32_t* out) {
    return guarded([&] {
        Partition p = partition_mincut(*static_cast<Graph*>(g), parts, seed, eps);
        std::memcpy(out, p.assignment.data(), sizeof(std::uint32_t) * p.assignment.size());
    });
}
int grr_hierarchical_partition(void* g, std::uint32_t servers, std::uint32_t gpus, int mincut,
                               std::uint64_t seed, std::uint32_t* server_out,
                               std::uint32_t* gpu_out) {
    return guarded([&] {
        HierarchicalPartition h = hierarchical_partition(
            *static_cast<Graph*>(g), servers, gpus,
            mincut ? PartitionMode::MinCut : PartitionMode::Random, seed);
        std::memcpy(server_out, h.server.assignment.data(),
                    sizeof(std::uint32_t) * h.server.assignment.size());
        std::memcpy(gpu_out, h.gpu.assignment.data(),
                    sizeof(std::uint32_t) * h.gpu.assignment.size());
    });
}

// ---- rng / init --------------------------------------------------------------
std::uint64_t grr_mix64(std::uint64_t x) { return mix64(x); }
void grr_rng_draws(std::uint64_t seed, std::uint64_t k1, std::uint64_t k2, std::uint64_t count,
                   std::uint64_t* out) {
    KeyedRng r(seed, k1, k2);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void grr_shuffle(std::uint64_t seed, std::uint64_t k1, std::uint64_t k2, std::uint32_t* items,
                 std::uint64_t count) {
    KeyedRng r(seed, k1, k2);
    std::vector<std::uint32_t> v(items, items + count);
    keyed_shuffle(v, r);
    std::memcpy(items, v.data(), sizeof(std::uint32_t) * count);
}
void grr_make_features(std::uint32_t n, std::uint32_t dim, std::uint64_t seed, double* out) {
    Matrix m = make_features(n, dim, seed);
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
}
int grr_make_layer_weights(std::uint32_t layers, std::uint32_t F, std::uint32_t H,
                           std::uint64_t seed, double* out) {
    return guarded([&] {
        LayerWeights w = make_layer_weights(layers, F, H, seed);
        for (const Matrix& m : w.layers) {
            std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
            out += m.data.size();
        }
    });
}

// ---- reference GNN ----------------------------------------------------------
int grr_forward_full(void* g, const double* x, std::uint32_t rows, std::uint32_t F,
                     const double* w, std::uint32_t wl, std::uint32_t H, std::uint32_t layers,
                     double* out) {
    return guarded([&] {
        Matrix xm = to_matrix(x, rows, F);
        Matrix r = forward_full(*static_cast<Graph*>(g), xm, to_weights(w, wl, F, H), layers);
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    });
}
int grr_forward_server_local(void* g, const std::uint32_t* hop, std::uint32_t server,
                             std::uint32_t hop_limit, int sampled, const double* x,
                             std::uint32_t F, const double* w, std::uint32_t H,
                             std::uint32_t layers, int require_exact, double* out) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        DependencySubgraph sub = sub_from_hops(gr, hop, server, hop_limit, sampled);
        Matrix xm = to_matrix(x, gr.num_vertices(), F);
        Matrix r = forward_server_local(sub, gr, xm, to_weights(w, layers, F, H), layers,
                                        require_exact != 0);
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    });
}
double grr_equivalence_check(void* g, const std::uint32_t* assign, std::uint32_t parts,
                             std::uint32_t layers, std::uint64_t seed, std::uint32_t F,
                             std::uint32_t H) {
    double dev = -1.0;
    guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        dev = equivalence_check(gr, make_partition(assign, gr.num_vertices(), parts), layers, seed,
                                F, H)
                  .max_deviation;
    });
    return dev;
}

// ---- extraction ---------------------------------------------------------------
int grr_extract_full(void* g, const std::uint32_t* assign, std::uint32_t parts,
                     std::uint32_t server, std::uint32_t layers, std::uint32_t* hop,
                     std::uint64_t* induced) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        DependencySubgraph s =
            extract_full(gr, make_partition(assign, gr.num_vertices(), parts), server, layers);
        hops_out(gr, s, hop);
        *induced = s.induced_edges;
    });
}
int grr_extract_sampled(void* g, const std::uint32_t* assign, std::uint32_t parts,
                        std::uint32_t server, std::uint32_t max_hop, std::uint32_t fanout,
                        std::uint64_t seed, std::uint32_t* hop, std::uint64_t* induced) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        DependencySubgraph s =
            extract_sampled(gr, make_partition(assign, gr.num_vertices(), parts), server,
                            SamplingConfig{max_hop, fanout, seed});
        hops_out(gr, s, hop);
        *induced = s.induced_edges;
    });
}
int grr_neighbor_explosion_profile(void* g, const std::uint32_t* assign, std::uint32_t parts,
                                   std::uint32_t server, std::uint32_t max_layers,
                                   std::uint64_t* sizes) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        auto prof = neighbor_explosion_profile(
            gr, make_partition(assign, gr.num_vertices(), parts), server, max_layers);
        for (std::size_t i = 0; i < prof.size(); ++i) sizes[i] = prof[i].second;
    });
}

// ---- cooperative batching -------------------------------------------------------
// Plan handle: flattened (targets, vertices, mfg, bytes) per batch.
struct PlanOut {
    BatchPlan plan;
};
void* grr_plan_cobatch_fixed_r(void* g, const std::uint32_t* hop, std::uint32_t server,
                               std::uint32_t hop_limit, int sampled, std::uint32_t layers,
                               std::uint32_t max_hop, std::uint32_t fanout, std::uint64_t seed,
                               std::uint32_t r, std::uint32_t hidden, std::uint32_t feat) {
    PlanOut* out = nullptr;
    if (guarded([&] {
            const Graph& gr = *static_cast<Graph*>(g);
            DependencySubgraph sub = sub_from_hops(gr, hop, server, hop_limit, sampled);
            ModelSpec m{layers, hidden, feat, 1.5};
            out = new PlanOut{plan_cobatch_fixed_r(sub, gr, layers,
                                                   SamplingConfig{max_hop, fanout, seed}, r, m)};
        }))
        return nullptr;
    return out;
}
// plan_cobatch (batch_plan.cpp:155-180): the budgeted R scan; nullptr + error on
// failure (grr_last_error names the category, e.g. capacity).
void* grr_plan_cobatch(void* g, const std::uint32_t* hop, std::uint32_t server, std::uint32_t hop_limit,
                       int sampled, std::uint32_t layers, std::uint32_t max_hop, std::uint32_t fanout,
                       std::uint64_t seed, std::uint64_t budget, std::uint32_t hidden, std::uint32_t feat) {
    PlanOut* out = nullptr;
    if (guarded([&] {
            const Graph& gr = *static_cast<Graph*>(g);
            DependencySubgraph sub = sub_from_hops(gr, hop, server, hop_limit, sampled);
            ModelSpec m{layers, hidden, feat, 1.5};
            out = new PlanOut{plan_cobatch(sub, gr, layers, SamplingConfig{max_hop, fanout, seed}, budget, m)};
        }))
        return nullptr;
    return out;
}
std::uint32_t grr_plan_batches(void* p) { return static_cast<PlanOut*>(p)->plan.batch_count(); }
void grr_plan_batch_sizes(void* p, std::uint32_t b, std::uint64_t* nt, std::uint64_t* nv,
                          std::uint64_t* bytes) {
    const Batch& bt = static_cast<PlanOut*>(p)->plan.batches[b];
    *nt = bt.target_vertices.size();
    *nv = bt.vertices.size();
    *bytes = bt.est_memory_bytes;
}
void grr_plan_batch_copy(void* p, std::uint32_t b, std::uint32_t* targets, std::uint32_t* verts,
                         std::uint64_t* mfg) {
    const Batch& bt = static_cast<PlanOut*>(p)->plan.batches[b];
    std::memcpy(targets, bt.target_vertices.data(), 4 * bt.target_vertices.size());
    std::memcpy(verts, bt.vertices.data(), 4 * bt.vertices.size());
    std::memcpy(mfg, bt.mfg_vertices_per_layer.data(), 8 * bt.mfg_vertices_per_layer.size());
}
void grr_plan_free(void* p) { delete static_cast<PlanOut*>(p); }

// ---- simulator (indirect pin for split_batch, sim.cpp:223-266) -------------------
// Cobatch simulation of one plan per server given as flat batch vertex lists.
int grr_simulate_cobatch_moved(void* g, const std::uint32_t* sp, const std::uint32_t* gp,
                               std::uint32_t servers, std::uint32_t gpus, std::uint32_t layers,
                               void** plans, std::uint64_t* internal_moved,
                               std::uint64_t* preloaded) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        Partition spp = make_partition(sp, gr.num_vertices(), servers);
        Partition gpp = make_partition(gp, gr.num_vertices(), servers * gpus);
        ClusterSpec c;
        c.num_servers = servers;
        c.gpus_per_server = gpus;
        ModelSpec m{layers, 8, 8, 1.5};
        std::vector<BatchPlan> ps;
        for (std::uint32_t s = 0; s < servers; ++s) {
            BatchPlan p = static_cast<PlanOut*>(plans[s])->plan;
            p.worker_id = s;
            ps.push_back(std::move(p));
        }
        CostBreakdown b = simulate_epoch(gr, spp, gpp, c, m, Strategy::Cobatch, std::nullopt, &ps);
        for (std::size_t i = 0; i < b.workers.size(); ++i) {
            internal_moved[i] = b.workers[i].internal_moved;
            preloaded[i] = b.workers[i].features_preloaded;
        }
    });
}

// ---- simulator calibration: simulate_epoch (sim.cpp:165-283) with
// caller-supplied rates.  strategy: 0 baseline, 1 shared preload, 2 preload+EAS.
// totals[5] = compute, internal, external, grad sync, total (s); workers[6*i..] =
// compute_s, internal_s, external_s, sync_s, internal_moved, external_moved.
int grr_simulate_epoch(void* g, const std::uint32_t* sp, const std::uint32_t* gp, std::uint32_t servers,
                       std::uint32_t gpus, double compute_vps, double internal_bw_vps,
                       double external_bw_vps, std::uint32_t layers, std::uint32_t hidden,
                       std::uint32_t feature, int strategy, std::uint32_t max_hop, std::uint32_t fanout,
                       std::uint64_t sseed, double* totals, double* workers) {
    return guarded([&] {
        const Graph& gr = *static_cast<Graph*>(g);
        Partition spp = make_partition(sp, gr.num_vertices(), servers);
        Partition gpp = make_partition(gp, gr.num_vertices(), servers * gpus);
        ClusterSpec c;
        c.num_servers = servers;
        c.gpus_per_server = gpus;
        c.compute_vps = compute_vps;
        c.internal_bw_vps = internal_bw_vps;
        c.external_bw_vps = external_bw_vps;
        ModelSpec m{layers, hidden, feature, 1.5};
        Strategy st = strategy == 0 ? Strategy::FullGraphBaseline
                                    : (strategy == 1 ? Strategy::SharedPreload : Strategy::PreloadEas);
        std::optional<SamplingConfig> cfg;
        if (strategy == 2) cfg = SamplingConfig{max_hop, fanout, sseed};
        CostBreakdown b = simulate_epoch(gr, spp, gpp, c, m, st, cfg);
        totals[0] = b.compute_s;
        totals[1] = b.internal_comm_s;
        totals[2] = b.external_comm_s;
        totals[3] = b.grad_sync_s;
        totals[4] = b.total_s;
        for (std::size_t i = 0; i < b.workers.size(); ++i) {
            const WorkerCost& w = b.workers[i];
            double* o = workers + 6 * i;
            o[0] = w.compute_s;
            o[1] = w.internal_s;
            o[2] = w.external_s;
            o[3] = w.sync_s;
            o[4] = static_cast<double>(w.internal_moved);
            o[5] = static_cast<double>(w.external_moved);
        }
    });
}

}  // extern "C"
