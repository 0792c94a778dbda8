// granndis.hpp -- the reference's C++ hot-path API (proj/include/granndis/*.hpp,
// SURVEY.md §8b) re-declared over the B200 engine.
//
// Same namespace, type names, member layout and function signatures as the
// reference, so code written against granndis_core (including its own doctest
// suites, see tests/cxx/) compiles unchanged and links against
// libgranndis_b200.so instead.  Compute runs on the GPU through include/gdx.h;
// host preprocessing (generation, partitioning) runs in libgdx's C++.
// Matrices stay fp64 at the API (the reference's Matrix); the engine computes
// in fp32 with split-bf16 tcgen05 GEMMs.
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace granndis {

// ---- errors (errors.hpp:11-44) ----------------------------------------------
class Error : public std::runtime_error {
public:
    Error(std::string category, const std::string& detail)
        : std::runtime_error(detail), category_(std::move(category)) {}
    const std::string& category() const noexcept { return category_; }

private:
    std::string category_;
};
struct InputError : Error { explicit InputError(const std::string& d) : Error("input", d) {} };
struct ParseError : Error { explicit ParseError(const std::string& d) : Error("parse", d) {} };
struct CapacityError : Error { explicit CapacityError(const std::string& d) : Error("capacity", d) {} };
struct ContractError : Error { explicit ContractError(const std::string& d) : Error("contract", d) {} };
struct InternalError : Error { explicit InternalError(const std::string& d) : Error("internal", d) {} };

// ---- keyed RNG (rng.hpp:11-61) -------------------------------------------------
constexpr std::uint64_t mix64(std::uint64_t x) noexcept {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

class KeyedRng {
public:
    explicit KeyedRng(std::uint64_t seed, std::uint64_t k1 = 0, std::uint64_t k2 = 0) noexcept
        : s_(mix64(mix64(mix64(seed) ^ (k1 + 0x9e3779b97f4a7c15ULL)) ^ (k2 + 0xc2b2ae3d27d4eb4fULL))) {}
    std::uint64_t next_u64() noexcept {
        s_ += 0x9e3779b97f4a7c15ULL;
        std::uint64_t z = s_;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_double() noexcept { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    std::uint64_t next_below(std::uint64_t n) noexcept {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
    }
    double uniform(double lo, double hi) noexcept { return lo + (hi - lo) * next_double(); }

private:
    std::uint64_t s_;
};

template <typename T>
void keyed_shuffle(std::vector<T>& items, KeyedRng& rng) {
    for (std::size_t i = items.size(); i > 1; --i) {
        std::size_t j = static_cast<std::size_t>(rng.next_below(i));
        std::swap(items[i - 1], items[j]);
    }
}

// ---- graph (graph.hpp:11-87) ------------------------------------------------------
using VertexId = std::uint32_t;
using EdgeIndex = std::uint64_t;

class Graph {
public:
    Graph() = default;
    static Graph from_edges(const std::vector<std::pair<VertexId, VertexId>>& edges,
                            VertexId num_vertices, bool undirected);
    static Graph from_csr(VertexId n, std::vector<EdgeIndex> offsets, std::vector<VertexId> cols,
                          bool undirected = true);

    VertexId num_vertices() const noexcept { return n_; }
    EdgeIndex num_edges() const noexcept { return static_cast<EdgeIndex>(cols_.size()); }
    bool undirected() const noexcept { return undirected_; }
    std::span<const VertexId> neighbors(VertexId v) const {
        return {cols_.data() + offsets_[v], cols_.data() + offsets_[v + 1]};
    }
    VertexId degree(VertexId v) const { return static_cast<VertexId>(offsets_[v + 1] - offsets_[v]); }
    const std::vector<EdgeIndex>& row_offsets() const noexcept { return offsets_; }
    const std::vector<VertexId>& col_indices() const noexcept { return cols_; }
    std::uint32_t feature_dim() const noexcept { return feature_dim_; }
    void set_feature_dim(std::uint32_t d) noexcept { feature_dim_ = d; }
    bool operator==(const Graph& o) const noexcept {
        return n_ == o.n_ && offsets_ == o.offsets_ && cols_ == o.cols_;
    }

private:
    VertexId n_ = 0;
    std::vector<EdgeIndex> offsets_{0};
    std::vector<VertexId> cols_;
    bool undirected_ = true;
    std::uint32_t feature_dim_ = 0;
    // The engine's device copy of this (immutable) CSR: uploaded on first use and kept,
    // shared by copies of the graph, so repeated calls do not re-upload it.
    mutable std::shared_ptr<void> device_;
    friend struct GraphDevice;
};

Graph gen_random_graph(VertexId n, double avg_degree, std::uint64_t seed);
Graph gen_planted_partition_graph(VertexId n, std::uint32_t parts, double p_in, double p_out,
                                  std::uint64_t seed);
std::uint32_t planted_block_of(VertexId v, VertexId n, std::uint32_t parts);

// ---- partition (partition.hpp:15-71) -------------------------------------------------
inline constexpr double kDefaultBalanceEps = 0.05;

struct Partition {
    std::vector<std::uint32_t> assignment;
    std::uint32_t num_parts = 0;
    std::vector<VertexId> part_sizes;
    std::uint32_t part_of(VertexId v) const { return assignment[v]; }
    std::vector<VertexId> members(std::uint32_t part) const;
};

enum class PartitionMode { Random, MinCut };
Partition partition_random(const Graph& g, std::uint32_t parts, std::uint64_t seed);
Partition partition_mincut(const Graph& g, std::uint32_t parts, std::uint64_t seed,
                           double epsilon = kDefaultBalanceEps);
struct HierarchicalPartition {
    Partition server;
    Partition gpu;
    std::uint32_t gpus_per_server = 1;
};
HierarchicalPartition hierarchical_partition(const Graph& g, std::uint32_t servers,
                                             std::uint32_t gpus_per_server, PartitionMode mode,
                                             std::uint64_t seed, double epsilon = kDefaultBalanceEps);
struct InducedSubgraph {
    Graph graph;
    std::vector<VertexId> global_ids;
};
InducedSubgraph induced_subgraph(const Graph& g, std::span<const VertexId> vertices_sorted);

// ---- extraction (extract.hpp:13-73) ----------------------------------------------------
inline constexpr std::uint32_t kUnlimitedFanout = std::numeric_limits<std::uint32_t>::max();

struct SamplingConfig {
    std::uint32_t max_hop = 1;
    std::uint32_t fanout = 15;
    std::uint64_t seed = 0;
    bool unlimited() const noexcept { return fanout == kUnlimitedFanout; }
};

struct DependencySubgraph {
    std::uint32_t server_id = 0;
    std::vector<VertexId> inner_vertices;
    std::vector<VertexId> halo_vertices;
    std::vector<std::uint32_t> halo_hops;
    EdgeIndex induced_edges = 0;
    std::uint32_t hop_limit = 0;
    bool sampled = false;

    bool is_inner(VertexId v) const;
    bool is_halo(VertexId v) const;
    bool contains(VertexId v) const { return is_inner(v) || is_halo(v); }
    std::uint32_t hop_of(VertexId v) const;
    std::vector<VertexId> all_vertices() const;
};

DependencySubgraph extract_full(const Graph& g, const Partition& server_partition,
                                std::uint32_t server_id, std::uint32_t layers);

struct SampleTraceStep {
    VertexId frontier_vertex;
    std::uint32_t hop;
    std::vector<VertexId> taken;
};
using SampleTrace = std::vector<SampleTraceStep>;

DependencySubgraph extract_sampled(const Graph& g, const Partition& server_partition,
                                   std::uint32_t server_id, const SamplingConfig& cfg,
                                   SampleTrace* trace = nullptr);
std::vector<std::pair<std::uint32_t, std::uint64_t>> neighbor_explosion_profile(
    const Graph& g, const Partition& server_partition, std::uint32_t server_id,
    std::uint32_t max_layers);

// ---- reference GNN (reference_gnn.hpp:13-66) -----------------------------------------
struct Matrix {
    std::uint32_t rows = 0;
    std::uint32_t cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(std::uint32_t r, std::uint32_t c) : rows(r), cols(c), data(std::size_t(r) * c, 0.0) {}
    double& at(std::uint32_t r, std::uint32_t c) { return data[std::size_t(r) * cols + c]; }
    double at(std::uint32_t r, std::uint32_t c) const { return data[std::size_t(r) * cols + c]; }
    std::span<double> row(std::uint32_t r) { return {data.data() + std::size_t(r) * cols, cols}; }
    std::span<const double> row(std::uint32_t r) const {
        return {data.data() + std::size_t(r) * cols, cols};
    }
};
using DenseFeatures = Matrix;
struct LayerWeights {
    std::vector<Matrix> layers;
};

DenseFeatures make_features(VertexId n, std::uint32_t dim, std::uint64_t seed);
LayerWeights make_layer_weights(std::uint32_t num_layers, std::uint32_t feature_dim,
                                std::uint32_t hidden_dim, std::uint64_t seed);
DenseFeatures forward_full(const Graph& g, const DenseFeatures& x, const LayerWeights& w,
                           std::uint32_t layers);
DenseFeatures forward_server_local(const DependencySubgraph& sub, const Graph& g,
                                   const DenseFeatures& x, const LayerWeights& w,
                                   std::uint32_t layers, bool require_exact = false);
struct EquivalenceReport {
    std::vector<double> per_server_max_dev;
    double max_deviation = 0.0;
};
EquivalenceReport equivalence_check(const Graph& g, const Partition& server_partition,
                                    std::uint32_t layers, std::uint64_t seed,
                                    std::uint32_t feature_dim = 8, std::uint32_t hidden_dim = 8);

// ---- model description (cost_model.hpp:24-29) ------------------------------------------
struct ModelSpec {
    std::uint32_t layers = 1;
    std::uint32_t hidden_dim = 64;
    std::uint32_t feature_dim = 64;
    double expansion_factor = 1.5;  // per-layer dependency growth rate
};

// ---- cooperative batch planning (batch_plan.hpp:13-69) ----------------------------------
// Device implementation: every group of one R is evaluated in batched launches
// (gdx_cobatch_eval), the R scan reads one count array per R back; only the chosen
// R's vertex lists are materialised.
inline constexpr std::uint64_t kUnlimitedMemory = std::numeric_limits<std::uint64_t>::max();
inline constexpr std::uint32_t kBytesPerScalar = 4;

enum class BatchStrategy { FetchThenSplit, SplitThenFetch };

struct Batch {
    std::vector<VertexId> target_vertices;              // sorted
    std::vector<VertexId> vertices;                     // sorted dependency universe
    std::vector<std::uint64_t> mfg_vertices_per_layer;  // [0] inputs .. [L] targets
    std::uint64_t est_memory_bytes = 0;
};

struct BatchPlan {
    std::uint32_t worker_id = 0;
    BatchStrategy strategy = BatchStrategy::FetchThenSplit;
    std::uint32_t layers = 0;
    std::vector<Batch> batches;
    std::uint32_t batch_count() const noexcept { return static_cast<std::uint32_t>(batches.size()); }
};

std::uint64_t estimate_batch_memory(const Batch& b, const ModelSpec& model);
BatchPlan plan_cobatch(const DependencySubgraph& sub, const Graph& g, std::uint32_t layers,
                       const SamplingConfig& cfg, std::uint64_t mem_budget, const ModelSpec& model);
BatchPlan plan_cobatch_fixed_r(const DependencySubgraph& sub, const Graph& g, std::uint32_t layers,
                               const SamplingConfig& cfg, std::uint32_t r, const ModelSpec& model);
// The paper's split-then-fetch comparison baseline (per-GPU chunks, layer-wise fanout);
// host C++, not on the training path.
BatchPlan plan_minibatch_baseline(const Graph& g, const Partition& gpu_partition, std::uint32_t gpu_id,
                                  std::uint32_t layers, std::uint32_t fanout_per_layer,
                                  std::uint64_t mem_budget, const ModelSpec& model, std::uint64_t seed);
std::string plan_to_json(const BatchPlan& plan);
void save_plan_json(const BatchPlan& plan, const std::string& path);

// ---- cooperative split (sim.cpp:81-102, re-exported) ------------------------------------
std::vector<std::vector<VertexId>> split_batch(const std::vector<VertexId>& batch_vertices,
                                               const Partition& server_partition,
                                               const Partition& gpu_partition,
                                               std::uint32_t server, std::uint32_t gpus);

}  // namespace granndis
