/*
 * granndis_oracle.h -- CPU restatement of the GraNNDis reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against; nothing in the product (paper_2311_06837_b200/) may link or call it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs use it.
 *
 * Every function restates the reference algorithm (file:line under
 * /root/reference/proj) in plain C.  The pinned subset (RNG, generators,
 * forward_full, forward_server_local, extract_full, extract_sampled,
 * batch_closure, peel_mfg, split_batch) is checked bit-for-bit against the
 * compiled reference (oracle/_ref, built by oracle/Makefile) and against the
 * reference unit tests' known answers (tests/golden/).  The training extension
 * (GraphSAGE-mean, normalised GCN, softmax cross-entropy, backward, SGD) has no
 * reference implementation: parity there is UNPINNED beyond
 * the reduction to forward_full for the Sum model, and is backed by
 * finite-difference gradient checks in tests/test_oracle.py.
 *
 * Conventions: CSR = row_offsets u64[n+1] + col_indices u32[nnz] (graph.hpp:21-60);
 * all buffers are caller-allocated; hop arrays use GRO_UNSEEN for outsiders.
 */
#ifndef GRANNDIS_ORACLE_H
#define GRANNDIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRO_UNSEEN 0xFFFFFFFFu
#define GRO_UNLIMITED_FANOUT 0xFFFFFFFFu

/* ---- rng.hpp:11-61 ---------------------------------------------------- */
typedef struct { uint64_t state; } gro_rng;
uint64_t gro_mix64(uint64_t x);
void gro_rng_init(gro_rng* r, uint64_t seed, uint64_t k1, uint64_t k2);
uint64_t gro_next_u64(gro_rng* r);
double gro_next_double(gro_rng* r);
uint64_t gro_next_below(gro_rng* r, uint64_t n);
void gro_shuffle_u32(uint32_t* items, uint64_t count, gro_rng* r);

/* ---- graph.cpp ---------------------------------------------------------- */
/* Two calls: *_count fills row_offsets (n+1) and returns nnz; *_fill writes cols. */
uint64_t gro_gen_random_graph_count(uint32_t n, double avg_degree, uint64_t seed,
                                    uint64_t* row_offsets);
void gro_gen_random_graph_fill(uint32_t n, double avg_degree, uint64_t seed,
                               const uint64_t* row_offsets, uint32_t* cols);
uint64_t gro_gen_planted_count(uint32_t n, uint32_t parts, double p_in, double p_out,
                               uint64_t seed, uint64_t* row_offsets);
void gro_gen_planted_fill(uint32_t n, uint32_t parts, double p_in, double p_out, uint64_t seed,
                          const uint64_t* row_offsets, uint32_t* cols);
/* Graph::from_edges, undirected: edges u32[2*m]; returns nnz, cols must hold 2*m. */
uint64_t gro_from_edges(const uint32_t* edges, uint64_t m, uint32_t n, uint64_t* row_offsets,
                        uint32_t* cols);

/* ---- partition.cpp:51-61 ------------------------------------------------ */
void gro_partition_random(uint32_t n, uint32_t parts, uint64_t seed, uint32_t* assignment);

/* ---- reference_gnn.cpp -------------------------------------------------- */
void gro_make_features(uint32_t n, uint32_t dim, uint64_t seed, double* out);
void gro_feature_rows(const uint32_t* ids, uint64_t count, uint32_t dim, uint64_t seed,
                      double* out, int nthreads);
void gro_make_layer_weights(uint32_t layers, uint32_t feature_dim, uint32_t hidden_dim,
                            uint64_t seed, double* out);
/* out: n x (layers ? hidden : F).  nthreads>1 keeps per-row order, so bit-identical. */
void gro_forward_full(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                      uint32_t F, const double* w, uint32_t H, uint32_t layers, double* out,
                      int nthreads);
/* hop[v]: 0 inner, >=1 halo, GRO_UNSEEN outside.  out: n_inner rows (ascending inner id). */
void gro_forward_server_local(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                              const double* x, uint32_t F, const double* w, uint32_t H,
                              uint32_t layers, const uint32_t* hop, double* out);

/* ---- extract.cpp -------------------------------------------------------- */
/* Both write hop[n] (0 inner / h halo / GRO_UNSEEN) and return induced_edges. */
uint64_t gro_extract_full(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                          const uint32_t* assignment, uint32_t server, uint32_t layers,
                          uint32_t* hop);
uint64_t gro_extract_sampled(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                             const uint32_t* assignment, uint32_t server, uint32_t max_hop,
                             uint32_t fanout, uint64_t seed, uint32_t* hop);

/* ---- batch_plan.cpp:28-101, sim.cpp:81-102 ------------------------------ */
/* in_closure[n] := 1 for targets and sampled closure members. returns closure size */
uint64_t gro_batch_closure(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                           const uint8_t* universe, const uint32_t* targets, uint64_t nt,
                           uint32_t max_hop, uint32_t fanout, uint64_t seed, uint8_t* in_closure);
void gro_peel_mfg(uint32_t n, const uint64_t* ro, const uint32_t* ci, const uint8_t* in_batch,
                  const uint32_t* targets, uint64_t nt, uint32_t layers, uint64_t* counts);
/* share_of[i] = local GPU of batch_vertices[i] (batch_vertices sorted ascending). */
void gro_split_batch(const uint32_t* batch_vertices, uint64_t nb, const uint32_t* server_assign,
                     const uint32_t* gpu_assign, uint32_t server, uint32_t gpus,
                     uint32_t* share_of);

/* ---- training extension (UNPINNED; no reference implementation) --------- */
enum { GRO_SUM = 0, GRO_SAGE = 1, GRO_GCN = 2 };
typedef struct {
    int kind;
    uint32_t layers;
    const uint32_t* dims; /* layers + 1 widths: dims[0] = feature dim */
    int relu_last;        /* 1: ReLU on the last layer too (reference Sum semantics) */
} gro_model;

/* Number of doubles in the flat weight vector (SAGE: W_self then W_neigh per layer). */
uint64_t gro_weight_count(const gro_model* m);
/* acts: if non-null, receives H^1..H^L concatenated (n x dims[l] each). */
void gro_model_forward(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                       const gro_model* m, const double* w, double* acts, int nthreads);
/*
 * One full-graph epoch: forward, mean softmax cross-entropy over rows < row_limit
 * (labels int32), backward, SGD (w -= lr*dW) in place.  Returns the loss.
 * grads (nullable) receives dW; dacts (nullable) receives dL/dH^1..dL/dH^L.
 * row_limit < n restricts every phase to destination rows < row_limit (used
 * only to time a bounded sample for the CPU baseline).
 */
double gro_train_epoch(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                       const int32_t* labels, uint32_t num_classes, const gro_model* m,
                       double* w, double lr, double* grads, double* acts, double* dacts,
                       uint32_t row_limit, int nthreads);
/* Same epoch with the loss restricted to rows < loss_rows and normalised by
 * loss_count (>= loss_rows: the global count when several subgraphs train
 * together); SGD is skipped when lr == 0 (gradients only, for summing across
 * subgraphs).  layer_rows (nullable, [layers]): layer l produces only rows <
 * layer_rows[l] -- the hop masking of forward_server_local (reference_gnn.cpp:119-137)
 * when local ids are ordered by hop.  Returns the (partial) loss sum / loss_count. */
double gro_train_epoch_masked(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                              const int32_t* labels, uint32_t num_classes, const gro_model* m,
                              double* w, double lr, double* grads, uint32_t loss_rows,
                              double loss_count, const uint32_t* layer_rows, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
