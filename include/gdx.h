/*
 * gdx.h -- C ABI of the B200 GraNNDis hot-path engine (libgdx.so).
 *
 * The reference (/root/reference/proj) exposes its hot path only as C++
 * free functions in namespace granndis; it has no FFI.  This
 * header is the thin extern "C" layer those functions are re-implemented on:
 * plain pointers and sizes, caller-allocated DEVICE buffers (unless a name
 * says host), stream-ordered, no allocation inside per-layer calls, no
 * exceptions.  Each entry point cites the reference code it replaces.
 *
 * Status codes mirror the reference error taxonomy (errors.hpp:11-44):
 *   GDX_OK 0, GDX_INPUT 1 (InputError), GDX_CAPACITY 2 (CapacityError),
 *   GDX_CONTRACT 3 (ContractError), GDX_INTERNAL 4 (InternalError / CUDA).
 * gdx_last_error() returns the thread-local message of the last failure.
 *
 * Layouts: CSR row_ptr u64[rows+1] (absolute offsets) + col u32[nnz]
 * (graph.hpp:21-60).  Dense matrices are row-major fp32 with a row pitch in
 * elements.  GEMM operands are "split bf16": x = hi + lo with
 * hi = bf16(x), lo = bf16(x - hi), stored as two uint16 arrays.
 */
#ifndef GDX_H
#define GDX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gdx_stream; /* == cudaStream_t; NULL = legacy default stream */

enum { GDX_OK = 0, GDX_INPUT = 1, GDX_CAPACITY = 2, GDX_CONTRACT = 3, GDX_INTERNAL = 4 };
#define GDX_UNSEEN 0xFFFFFFFFu
#define GDX_UNLIMITED_FANOUT 0xFFFFFFFFu

const char* gdx_last_error(void);
int gdx_version(void);
/* Number of GPU kernel launches issued by this library in this process. */
uint64_t gdx_launch_count(void);

/* ------------------------------------------------------------------------
 * Host preprocessing (C++, OpenMP).  Bit-identical to the reference.
 * ---------------------------------------------------------------------- */
/* gen_random_graph (graph.cpp:137-154, assemble_undirected :116-132).
 * Pass 1 fills row_offsets[n+1] and returns nnz; pass 2 fills cols[nnz]. */
uint64_t gdx_host_gen_random_graph_count(uint32_t n, double avg_degree, uint64_t seed,
                                         uint64_t* row_offsets);
int gdx_host_gen_random_graph_fill(uint32_t n, double avg_degree, uint64_t seed,
                                   const uint64_t* row_offsets, uint32_t* cols);
/* SampleTrace of extract_sampled (extract.hpp:49-64): per step (frontier vertex, hop,
 * taken[step_off[i] .. step_off[i+1])) in the reference's sequential attribution order.
 * Call with null outputs to get nsteps / ntaken, then with capacities (step_off has
 * cap_steps + 1 entries).  Host diagnostics (the taken sets equal the device growth's). */
int gdx_host_sample_trace(uint32_t n, const uint64_t* row_offsets, const uint32_t* cols, const uint8_t* inner,
                          uint32_t max_hop, uint32_t fanout, uint64_t seed, uint64_t cap_steps, uint64_t cap_taken,
                          uint64_t* nsteps, uint64_t* ntaken, uint32_t* step_vertex, uint32_t* step_hop,
                          uint64_t* step_off, uint32_t* taken);
/* partition_random (partition.cpp:51-61). */
int gdx_host_partition_random(uint32_t n, uint32_t parts, uint64_t seed, uint32_t* assignment);
/* partition_mincut (partition.cpp:63-170) over a host CSR (bit-identical assignment). */
int gdx_host_partition_mincut(uint32_t n, const uint64_t* row_offsets, const uint32_t* cols,
                              uint32_t parts, uint64_t seed, double epsilon, uint32_t* assignment);

/* ------------------------------------------------------------------------
 * K7 initialisation: make_features / make_layer_weights (reference_gnn.cpp:11-32)
 * out[r*ld + c] = float(lo + (hi-lo)*next_double()) of stream (seed,k1,k2) at draw
 * index first_draw + r*cols + c (SplitMix64 jump-ahead; bit-exact double math).
 * ---------------------------------------------------------------------- */
int gdx_init_uniform(uint64_t seed, uint64_t k1, uint64_t k2, uint64_t first_draw,
                     uint32_t rows, uint32_t cols, double lo, double hi, float* out,
                     uint64_t ld, gdx_stream stream);
/* Same stream, written as fp64 (the reference Matrix element type). */
int gdx_init_uniform_f64(uint64_t seed, uint64_t k1, uint64_t k2, uint64_t first_draw,
                         uint32_t rows, uint32_t cols, double lo, double hi, double* out,
                         uint64_t ld, gdx_stream stream);
/* Builder-defined labels: KeyedRng(seed, base+v, "labl").next_below(classes). */
int gdx_init_labels(uint64_t seed, uint64_t base, uint32_t rows, uint32_t classes,
                    int32_t* out, gdx_stream stream);

/* ------------------------------------------------------------------------
 * K1/K3 aggregation: the forward_full inner loop (reference_gnn.cpp:76-83),
 * forward_server_local's masked loop (:123-134) and the transposed backward.
 *   out[v] = act( post_scale[v] * (self_coef * src[self_base+v] + partial[v]
 *                                  + sum_{e in [row_ptr[v], row_end[v]) \ skip} src[col[e]])
 *                 + add[v] )
 * The skip range / partial pair splits a row into the locally owned column block
 * (aggregated while the all-gather of remote rows is in flight) and the rest.
 * ---------------------------------------------------------------------- */
typedef struct gdx_aggregate_args {
    const uint64_t* row_ptr;  /* [rows+1] */
    const uint64_t* row_end;  /* nullable: per-row end, else row_ptr[v+1] */
    const uint64_t* skip_lo;  /* nullable pair: per-row sub-range [skip_lo, skip_hi) excluded */
    const uint64_t* skip_hi;
    const float* partial;     /* nullable: partial sums [rows x ld_partial] added before scaling */
    uint64_t ld_partial;
    const uint32_t* col;
    uint32_t rows;
    uint32_t width;           /* feature width F (any; fast paths for F % 4 == 0) */
    const float* src;         /* gathered matrix, row pitch ld_src (16 B aligned rows) */
    uint64_t ld_src;
    float self_coef;          /* 1: reference self term, 0: none (SAGE mean) */
    uint64_t self_base;       /* src row of destination 0 (owned-row offset) */
    const float* post_scale;  /* nullable, [rows] */
    const float* add;         /* nullable, [rows x ld_add] (SAGE self path) */
    uint64_t ld_add;
    int relu;
    float* out;               /* nullable fp32 [rows x ld_out] */
    uint64_t ld_out;
    uint16_t* out_hi;         /* nullable split-bf16 copy [rows x ld_split] */
    uint16_t* out_lo;
    uint64_t ld_split;
    /* Packed-24 rows (fp32 rounded to 24 bits: 15 mantissa bits, relative error <= 2^-16,
     * the split-bf16 GEMM operands' precision) in two planes of the same pitch: u16 high
     * bits + u8 next bits -- 6 of a 64-wide row's 8 sectors.  src_lo8 non-null: src is
     * the u16 high plane (pitch ld_src elements) of the gathered matrix, self term
     * included; out24_*: packed-24 copy of the output.  Width a multiple of 8. */
    const uint8_t* src_lo8;
    uint16_t* out24_hi;
    uint8_t* out24_lo;
    uint64_t ld_out24;
    /* pitch of the packed-24 source's low plane in bytes (0: ld_src) -- e.g. one
     * interleaved 3F-byte row per vertex (high plane then low plane), so a block of
     * rows is one contiguous range (the trainer's exchanged buffers) */
    uint64_t ld_src_lo8;
} gdx_aggregate_args;
/* Degree-binned load balancing for skewed graphs (replaces the reference's uniform
 * per-vertex loop, reference_gnn.cpp:76-83, for hub-heavy inputs): rows with more
 * than heavy_degree edges are cut into chunks of chunk_edges edges; one warp per chunk
 * gathers an fp32 partial row, one warp per heavy row sums its chunks in order
 * (deterministic) and applies the epilogue; the other rows run the normal kernels
 * through a row list.  Built once per CSR from its HOST row offsets. */
typedef struct gdx_row_bins {
    uint32_t rows, n_light, n_heavy, n_chunks, chunk_edges;
    uint32_t* light_rows;       /* device, ascending */
    uint32_t* heavy_rows;       /* device, ascending */
    uint32_t* chunk_row;        /* device [n_chunks]: position in heavy_rows */
    uint64_t* chunk_beg;        /* device [n_chunks]: first edge of the chunk */
    uint64_t* chunk_off;        /* device [n_heavy+1]: chunks of each heavy row */
    float* partial;             /* device workspace [n_chunks x ld_partial] */
    uint64_t ld_partial;
    uint32_t* light_host;       /* host copies (prefix sizes per call) */
    uint32_t* heavy_host;
    uint64_t* chunk_off_host;
} gdx_row_bins;
int gdx_row_bins_build(const uint64_t* row_ptr_host, uint32_t rows, uint32_t heavy_degree, uint32_t chunk_edges,
                       uint32_t max_width, gdx_row_bins** out);
int gdx_row_bins_free(gdx_row_bins* bins);
/* gdx_aggregate_variant over the bins (bins NULL or no heavy row: the plain call).
 * Rows >= a->rows are skipped (hop prefixes).  fp32 rows only. */
int gdx_aggregate_balanced(const gdx_aggregate_args* a, int variant, const gdx_row_bins* bins, gdx_stream stream);
/* fp32 <-> packed-24 conversion (round to nearest even at bit 8). */
int gdx_pack24(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols, uint16_t* hi, uint8_t* lo,
               uint64_t ld_dst, gdx_stream stream);
int gdx_unpack24(const uint16_t* hi, const uint8_t* lo, uint64_t ld_src, uint32_t rows, uint32_t cols, float* dst,
                 uint64_t ld_dst, gdx_stream stream);
int gdx_aggregate(const gdx_aggregate_args* a, gdx_stream stream);
/* seg_lo[v], seg_hi[v] = sub-range of row v's (sorted) column ids inside [lo, hi). */
int gdx_row_split(const uint64_t* row_ptr, const uint32_t* col, uint32_t rows, uint32_t lo,
                  uint32_t hi, uint64_t* seg_lo, uint64_t* seg_hi, gdx_stream stream);
/* Kernel selection.  variant GDX_AGG_ROWS: one lane group per destination row
 * (EPW rows per warp at once) -- for low-degree CSRs such as cooperative-batch
 * subgraphs (a few in-batch edges per row), where the warp-per-row kernel is
 * bound by the per-row row_ptr -> col -> row latency chain.  4 / 8: unroll depth
 * of the warp-per-row kernel (tuning).  0 = gdx_aggregate. */
#define GDX_AGG_ROWS 1
/* GDX_AGG_ROWS2: lane groups of half the row (two 16-byte chunks per lane), twice the rows
 * per warp (degree ~8-20).  GDX_AGG_FLAT: a lane group walks the edges of LPE-1
 * consecutive rows in order with gathers in flight across row boundaries (degree < 6);
 * plain CSR rows only (falls back to GDX_AGG_ROWS with row_end / skip / row lists). */
#define GDX_AGG_ROWS2 2
#define GDX_AGG_FLAT 3
/* GDX_AGG_P24_WIDE: 48-wide packed-24 rows whose planes are readable to 64 columns (pitch
 * >= 64 in both planes, e.g. the trainer's 192-byte interleaved rows) gathered as whole
 * 64-wide rows; columns 48..63 are read but never stored. */
#define GDX_AGG_P24_WIDE 16
int gdx_aggregate_variant(const gdx_aggregate_args* a, int variant, gdx_stream stream);

/* ------------------------------------------------------------------------
 * K2 dense transform on tcgen05 (apply_layer, reference_gnn.cpp:53-60):
 *   C[m][n] = sum_k (A_hi+A_lo)(m,k) * (B_hi+B_lo)(n,k)   (3 bf16 MMAs, fp32 TMEM acc)
 * with each operand K-major or MN-major (so G^T H needs no transposes).
 * Persistent: one CTA per SM, double-buffered TMEM accumulator.
 * Epilogue: C = mask ? (mask > 0 ? C : 0) : C; [split copy if split_unscaled];
 * C *= row_scale[m]; relu; columns [0,split) -> c0, [split,n) -> c1; optional split-bf16
 * copy (after scaling unless split_unscaled).  The mask form fuses the ReLU backward
 * and degree scaling of the next aggregation into the dH GEMM.  split_k > 1 writes raw partials to
 * c0 + z*m*ldc0 (z < split_k) for gdx_splitk_reduce.
 * Constraints: lda, ldb multiples of 8 elements; device pointers 16 B aligned.
 * Note: inputs are read by TMA through tensor maps built per call on the host.
 * ---------------------------------------------------------------------- */
typedef struct gdx_gemm_args {
    const uint16_t* a_hi; const uint16_t* a_lo; uint64_t lda;
    const uint16_t* b_hi; const uint16_t* b_lo; uint64_t ldb;
    int a_mn_major;           /* 0: A stored [m][k] (K-major); 1: A stored [k][m] */
    int b_mn_major;           /* 0: B stored [n][k];           1: B stored [k][n] */
    uint32_t m, n, k;
    float* c0; uint64_t ldc0;
    float* c1; uint64_t ldc1;
    uint32_t split;           /* == n when c1 unused */
    const float* row_scale;   /* nullable */
    int relu;
    uint16_t* out_hi; uint16_t* out_lo; uint64_t ld_split;   /* nullable */
    uint32_t split_k;         /* 0/1: none */
    const float* mask;        /* nullable [m x ld_mask]: C = 0 where mask <= 0 (ReLU backward) */
    uint64_t ld_mask;
    int split_unscaled;       /* 1: the split-bf16 copy is taken before row_scale */
    /* Fused exchange: every value stored to output `peer_target` (0: c0, 1: c1) is also
     * stored at the same offset in npeers peer buffers (address + peer_delta[r] bytes;
     * CUDA IPC mappings over NVLink), see gdx_peer_signal/gdx_peer_wait. */
    uint32_t npeers;
    int peer_target;
    int64_t peer_delta[7];
    /* Row gather (the cooperative batch's feature LOAD fused into its GEMMs, TMA
     * tile::gather4): nullable. a_rows [m]: row i of a K-major A is row a_rows[i] of a
     * source with a_src_rows rows (pitch lda); b_rows [k]: k-row i of an MN-major B is
     * row b_rows[i] of a source with b_src_rows rows (pitch ldb). Same results as
     * gdx_gather_split_rows followed by the plain GEMM. */
    const uint32_t* a_rows; uint64_t a_src_rows;
    const uint32_t* b_rows; uint64_t b_src_rows;
    /* Packed-24 output (nullable; the aggregation's packed-24 source format): the columns
     * of output p24_target (0: c0's [0, split), 1: c1's [split, n)) are stored as the
     * high-16 plane p24_hi (pitch ld_p24_hi u16) + low-8 plane p24_lo (pitch ld_p24_lo
     * bytes) instead of fp32; that output's fp32 pointer must be null. */
    uint16_t* p24_hi; uint8_t* p24_lo; uint64_t ld_p24_hi, ld_p24_lo; int p24_target;
} gdx_gemm_args;
int gdx_gemm_tn(const gdx_gemm_args* g, gdx_stream stream);
/* Reference-precision SIMT fallback of the same contract, for tests only. */
int gdx_gemm_tn_simt(const gdx_gemm_args* g, gdx_stream stream);
/* out[i] = sum_z ws[z*stride + i] for i < rows*cols (pitch ld); then optional SGD:
 * if w: w[i] -= lr * out[i] and (w_hi,w_lo) split copies are refreshed. */
int gdx_splitk_reduce(const float* ws, uint32_t split_k, uint64_t stride, uint32_t rows,
                      uint32_t cols, uint64_t ld, float* out, float* w, float lr,
                      uint16_t* w_hi, uint16_t* w_lo, gdx_stream stream);

/* ------------------------------------------------------------------------
 * Row exchange over NVLink peer memory (the a13 exchange of the trainer, fused
 * into the producing GEMM / softmax epilogues instead of a separate all-gather).
 * ---------------------------------------------------------------------- */
int gdx_device_alloc(uint64_t bytes, void** out);      /* zeroed cudaMalloc (IPC-able base) */
int gdx_device_free(void* p);
int gdx_ipc_get_handle(const void* base, void* handle64);   /* 64-byte cudaIpcMemHandle */
int gdx_ipc_open(const void* handle64, void** out);         /* lazy peer access enabled */
int gdx_ipc_close(void* p);
/* Per-source wait of a pipelined exchange: advance=1 starts the round (*expected += 1)
 * before waiting; every wait then blocks until slots[src] >= *expected. */
int gdx_peer_wait_src(unsigned long long* slots, unsigned long long* expected, uint32_t src, int advance,
                      uint64_t timeout_ns, gdx_stream stream);
/* SM-driven push of `bytes` at src to src + peer_delta[r] (IPC-mapped peer buffers)
 * for r < npeers, fused with gdx_peer_signal: the last of `ctas` CTAs releases the
 * stores (system fence) and bumps our slot in every peer's arrival array.
 * `done`: a device u32, zero before the first call (re-armed by the kernel). */
int gdx_push_peers(const void* src, uint64_t bytes, const int64_t* peer_delta, uint32_t npeers,
                   unsigned long long* const* peer_slots_dev, unsigned int* done, uint32_t ctas,
                   gdx_stream stream);
/* Sparse push: rows idx[off[r] .. off[r+1]) of this rank's block (row pitch row_bytes)
 * to the same offsets in peer r's buffer (base + peer_delta[r]), then signal as
 * gdx_push_peers.  For exchanges where each peer reads only part of the block. */
int gdx_push_rows(const void* base, uint64_t row_bytes, const uint32_t* idx, const uint64_t* off,
                  const int64_t* peer_delta, uint32_t npeers, unsigned long long* const* peer_slots_dev,
                  unsigned int* done, uint32_t ctas, gdx_stream stream);
/* NVSwitch multicast push: `bytes` at src stored once through the buffer's multicast
 * mapping (mc_dst = same offset in it; multimem.st), replicated by the switch into every
 * GPU's copy; fused signal as gdx_push_peers. */
int gdx_push_multicast(const void* src, uint64_t bytes, void* mc_dst, uint32_t npeers,
                       unsigned long long* const* peer_slots_dev, unsigned int* done, uint32_t ctas,
                       gdx_stream stream);
/* The layer exchange and the aggregation in ONE cooperative kernel: every block pushes
 * its share of this rank's row block (push_src, push_bytes) into every peer's copy
 * (push_src + peer_delta[r]), aggregates the locally owned source segment of its rows
 * ([seg_lo, seg_hi), into `partial`) while the stores drain, releases them (the last
 * block bumps this rank's slot in every peer), waits until every peer's slot reached
 * the round (*expected + 1; the last block to finish stores it), then aggregates the
 * remote segments with the fused epilogue of `a` (a->row_end / skip / partial unused).
 * Widths 32, 48, 64, 128.  counters: 2 zeroed u32.  Replaces gdx_push_peers +
 * two gdx_aggregate passes + gdx_peer_wait. */
int gdx_aggregate_exchange(const gdx_aggregate_args* a, const uint64_t* seg_lo, const uint64_t* seg_hi,
                           float* partial, uint64_t ld_partial, const void* push_src, uint64_t push_bytes,
                           const int64_t* peer_delta, uint32_t npeers, unsigned long long* const* peer_slots_dev,
                           unsigned long long* slots, unsigned long long* expected, uint32_t world, uint32_t self,
                           unsigned int* counters, uint64_t timeout_ns, gdx_stream stream);
/* One copy-engine push (cudaMemcpyAsync D2D; dst may be an IPC-mapped peer address). */
int gdx_memcpy_async(void* dst, const void* src, uint64_t bytes, gdx_stream stream);
/* rows x width_bytes of a pitched buffer set to `value` (stream-ordered, graph-capturable). */
int gdx_memset2d_async(void* dst, uint64_t pitch_bytes, int value, uint64_t width_bytes, uint64_t rows,
                       gdx_stream stream);
/* After the producing kernel: release its peer stores and increment this rank's slot
 * in every peer's arrival array (peer_slots_dev: device array of npeers IPC-mapped
 * u64 slot pointers). */
int gdx_peer_signal(unsigned long long* const* peer_slots_dev, uint32_t npeers, gdx_stream stream);
/* Before gathering remote rows: *expected += 1, spin (acquire, system scope) until
 * slots[r] >= *expected for every r != self; traps after timeout_ns.  Device-side
 * state only, so it can be captured in a CUDA graph and replayed. */
int gdx_peer_wait(unsigned long long* slots, unsigned long long* expected, uint32_t world,
                  uint32_t self, uint64_t timeout_ns, gdx_stream stream);

/* ------------------------------------------------------------------------
 * Layout / elementwise helpers of the training extension (no reference code).
 * ---------------------------------------------------------------------- */
/* dst (rows x cols, pitch ld_dst) = split(src); transpose=1 writes dst[c][r]. */
int gdx_split_bf16(const float* src, uint64_t ld_src, uint32_t rows, uint32_t cols,
                   uint16_t* hi, uint16_t* lo, uint64_t ld_dst, int transpose, gdx_stream stream);
/* Transpose a split-bf16 pair: dst[c][r] = src[r][c]. */
int gdx_transpose_split(const uint16_t* src_hi, const uint16_t* src_lo, uint64_t ld_src,
                        uint32_t rows, uint32_t cols, uint16_t* dst_hi, uint16_t* dst_lo,
                        uint64_t ld_dst, gdx_stream stream);
/* Backward through act and the aggregation's destination scale:
 *   g = dH * (mask ? (H > 0) : 1)          -> g_hi/g_lo (split, pitch ld_g) and g_out (fp32, nullable)
 *   gs = g * dst_scale[v]                  -> gs (fp32, nullable; the rows to gather) */
int gdx_grad_prepare(const float* dH, uint64_t ld_dh, const float* H, uint64_t ld_h,
                     uint32_t rows, uint32_t width, const float* dst_scale,
                     float* g_out, uint64_t ld_gout, float* gs, uint64_t ld_gs,
                     uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g, gdx_stream stream);
/* Softmax cross-entropy over rows: dlogits = (softmax - onehot) * inv_count,
 * loss_sum[0] += sum of per-row losses (fp64 atomics). */
int gdx_softmax_xent(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                     const int32_t* labels, float inv_count, float* dlogits, uint64_t ld_d,
                     double* loss_sum, gdx_stream stream);
/* Same, fused with the backward prep of the last layer: g = dlogits is written as a
 * split-bf16 copy (g_hi/g_lo, nullable) and as gs = g * row_scale[v] (gs, nullable;
 * row_scale nullable = 1); dlogits itself is optional. */
int gdx_softmax_xent_fused(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                           const int32_t* labels, float inv_count, float* dlogits, uint64_t ld_d,
                           const float* row_scale, float* gs, uint64_t ld_gs, uint16_t* g_hi,
                           uint16_t* g_lo, uint64_t ld_g, double* loss_sum, gdx_stream stream);
/* Same, with gs stored as packed-24 rows (u16 high plane, pitch ld_hi24 elements; u8 low
 * plane, pitch ld_lo8 bytes; the trainer's interleaved layout) instead of fp32 -- the
 * gathered source of the output layer's transposed aggregation.  classes <= 128. */
int gdx_softmax_xent_fused_p24(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                               const int32_t* labels, float inv_count, const float* row_scale,
                               uint16_t* gs_hi24, uint64_t ld_hi24, uint8_t* gs_lo8, uint64_t ld_lo8,
                               uint16_t* g_hi, uint16_t* g_lo, uint64_t ld_g, double* loss_sum,
                               gdx_stream stream);
/* Same, with gs also stored into npeers peer buffers (gs + gs_peer_delta[r] bytes). */
int gdx_softmax_xent_fused_peers(const float* logits, uint64_t ld, uint32_t rows, uint32_t classes,
                                 const int32_t* labels, float inv_count, const float* row_scale,
                                 float* gs, uint64_t ld_gs, uint16_t* g_hi, uint16_t* g_lo,
                                 uint64_t ld_g, double* loss_sum, uint32_t npeers,
                                 const int64_t* gs_peer_delta, gdx_stream stream);
/* Bandwidth probe for roofline denominators: reads `bytes` of buf `reps` times,
 * mode 0 = coalesced stream, mode 1 = random 256 B row gathers (bytes moved =
 * reps * bytes in both modes), mode 2 = random 192 B packed-24 row gathers (16 B + 8 B
 * per lane, 8 lanes per row; bytes moved = steps * 8 * T * 24 with T = 2048 * SMs
 * threads and steps = ceil(reps * bytes / (8 * T * 24))).  Time it with events on
 * `stream`. */
/* L2 access-policy window (persisting) on `stream` for the matrix the next kernels gather
 * (bytes = 0 clears it); carves the device's persisting L2 set-aside on first use. */
int gdx_set_l2_window(const void* base, uint64_t bytes, float hit_ratio, gdx_stream stream);
int gdx_probe_bandwidth(const float* buf, uint64_t bytes, uint32_t reps, int mode, float* sink,
                        gdx_stream stream);
/* Per-vertex scales from CSR degrees: kind 0 -> 1/deg (0 if deg=0), 1 -> (deg+1)^-1/2. */
int gdx_degree_scale(const uint64_t* row_ptr, uint32_t rows, int kind, float* out,
                     gdx_stream stream);

/* ------------------------------------------------------------------------
 * K4/K5 sampling and closure (integer, bit-exact).  Host-synchronising:
 * frontier sizes are read back once per hop.
 * ---------------------------------------------------------------------- */
/* Shared hop loop of extract_sampled (extract.cpp:135-182) and batch_closure
 * (batch_plan.cpp:28-70).  mark[n] in: 0 for excluded (inner / targets) vertices,
 * GDX_UNSEEN otherwise; out: hop label of every vertex taken.  allowed (nullable)
 * restricts candidates (the batch universe).  fanout GDX_UNLIMITED_FANOUT gives the
 * unsampled closure (extract_full, extract.cpp:87-113).  work: >= 2*n + 64 u32. */
int gdx_sampled_growth(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                       const uint8_t* excluded, const uint8_t* allowed, uint32_t max_hop,
                       uint32_t fanout, uint64_t seed, uint32_t* mark, uint32_t* work,
                       gdx_stream stream);
/* count_induced_edges (extract.cpp:49-58): sum over v with mark[v] != UNSEEN of
 * |{u in N(v): mark[u] != UNSEEN}|.  result: host pointer. work >= 1 u64. */
int gdx_induced_count(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                      const uint32_t* mark, unsigned long long* work, uint64_t* result,
                      gdx_stream stream);
/* peel_mfg (batch_plan.cpp:75-101): counts[layers+1] (host) of the back-peeled
 * MFG sets.  in_batch[n] u8; targets[nt]; work >= 3*n + 64 u32. */
int gdx_peel_mfg(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                 const uint8_t* in_batch, const uint32_t* targets, uint64_t nt, uint32_t layers,
                 uint32_t* work, uint64_t* counts, gdx_stream stream);
/* Cooperative-batch evaluation of one target grouping on the device: for every
 * group g (targets[group_off[g] .. group_off[g+1]), ascending ids, device; group_off
 * is a HOST array of groups+1 offsets) the sampled closure of the group's targets
 * inside universe[n] (candidates: universe minus the group's own targets; keyed
 * shuffle as EAS) -- batch_closure, batch_plan.cpp:28-70 -- and its back-peeled MFG
 * counts -- peel_mfg, :75-101 -- for all groups of a chunk in the same launches,
 * with no host synchronisation until the end (the body of plan_cobatch's R scan,
 * :155-180, and of plan_cobatch_fixed_r, :146-153).
 * Outputs (HOST): sizes[groups] = |batch vertices|, mfg[groups*(layers+1)] (row g is
 * the reference's mfg_vertices_per_layer).  If vertices (device) is non-NULL, batch
 * g's ascending vertex list is written at vertices + vertex_off[g] (host offsets,
 * from a previous call's sizes).  workspace_bytes bounds the per-call device
 * workspace (20 bytes per vertex per group evaluated together; >= one group). */
int gdx_cobatch_eval(const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                     const uint8_t* universe, const uint32_t* targets, const uint64_t* group_off,
                     uint32_t groups, uint32_t max_hop, uint32_t fanout, uint64_t seed,
                     uint32_t layers, uint64_t workspace_bytes, uint64_t* sizes, uint64_t* mfg,
                     uint32_t* vertices, const uint64_t* vertex_off, gdx_stream stream);
/* split_batch (sim.cpp:81-102): share_of[i] for sorted batch_vertices[i]; inner
 * vertices to their home GPU, halo vertices (ascending) to the least-loaded GPU,
 * computed in closed form (greedy == (level, gpu)-ordered slot filling).
 * work >= 5*nb + 2*gpus + 8 u32. */
int gdx_split_batch(const uint32_t* batch_vertices, uint64_t nb, const uint32_t* server_assign,
                    const uint32_t* gpu_assign, uint32_t server, uint32_t gpus,
                    uint32_t* share_of, uint32_t* work, gdx_stream stream);
/* Local numbering of a dependency subgraph for forward_server_local
 * (reference_gnn.cpp:103-116): vertices with hop[v] != UNSEEN ordered by
 * (hop, id), so the rows valid at layer l are a prefix.  Writes
 * local_to_global[local_n], local_of[n] (UNSEEN outside), hop_start[max_hop+2]
 * (host: first local id of each hop class) and returns local_n via *local_n. */
int gdx_order_by_hop(const uint32_t* hop, uint32_t n, uint32_t max_hop, uint32_t* local_to_global,
                     uint32_t* local_of, uint64_t* hop_start, uint32_t* local_n, gdx_stream stream);
/* Induced local CSR over that numbering (reference_gnn.cpp:125-131): row i lists
 * the in-subgraph neighbours of local_to_global[i] as local ids, in the global
 * row's (ascending-id) order, so a row whose neighbours are all present reduces
 * in exactly the same order as in the whole graph.
 * Pass 1 (lptr == NULL): counts[i] = in-subgraph degree of local vertex i.
 * Pass 2: writes the row at lptr[i]. */
int gdx_local_csr(const uint64_t* row_ptr, const uint32_t* col, const uint32_t* local_to_global,
                  uint32_t local_n, const uint32_t* local_of, uint64_t* counts, const uint64_t* lptr,
                  uint32_t* lcol, gdx_stream stream);
/* Exclusive prefix sum of counts[n] into out[n+1] (out[n] = total, also in *total). */
int gdx_exclusive_scan_u64(const uint64_t* counts, uint64_t n, uint64_t* out, uint64_t* total,
                           gdx_stream stream);
/* out[i*ld_out + c] = src[idx[i]*ld_src + c] for i < rows, c < cols (row gather). */
int gdx_gather_rows(const float* src, uint64_t ld_src, const uint32_t* idx, uint32_t rows,
                    uint32_t cols, float* out, uint64_t ld_out, gdx_stream stream);
/* Cooperative-batch feature LOAD (the LOAD step of the paper's Alg. 1 over a
 * resident split-bf16 feature store): out_{hi,lo}[i] = src_{hi,lo}[idx[i]] for
 * i < rows, whole 8-element vectors up to cols.  Pitches in elements, multiples of 8. */
int gdx_gather_split_rows(const uint16_t* src_hi, const uint16_t* src_lo, uint64_t ld_src,
                          const uint32_t* idx, uint32_t rows, uint32_t cols, uint16_t* out_hi,
                          uint16_t* out_lo, uint64_t ld_out, gdx_stream stream);

/* ------------------------------------------------------------------------
 * Training epoch as a C-ABI object (the benchmarked step, driven from C/C++ with
 * no Python): the reference's layer model (reference_gnn.cpp:64-147) plus the
 * north_star's softmax cross-entropy, backward and SGD, on this library's
 * kernels.  One trainer per GPU; world > 1 ranks exchange rows and weight
 * gradients through CUDA-IPC-shared buffers (gdx_trainer_ipc_export on every rank,
 * the blobs gathered by the caller -- MPI, sockets, torch -- then
 * gdx_trainer_connect on every rank).  No NCCL on the data path.
 * ---------------------------------------------------------------------- */
enum { GDX_MODEL_SUM = 0, GDX_MODEL_GCN = 1, GDX_MODEL_SAGE = 2 };
typedef struct gdx_trainer gdx_trainer;
typedef struct gdx_trainer_config {
    int kind;                 /* GDX_MODEL_*: Sum (reference), normalised GCN, SAGE-mean */
    uint32_t layers;          /* L */
    const uint32_t* dims;     /* [L+1]: feature width, hidden widths, classes (<= 256) */
    float lr;                 /* SGD step */
    uint32_t rank, world;     /* world <= 8 (<= 7 peers) */
    int device;               /* CUDA ordinal */
    uint64_t feature_seed;    /* make_features stream seed of the inputs (reference_gnn.cpp:11-16) */
    uint64_t label_seed;      /* labels: KeyedRng(seed, v, "labl").next_below(classes) */
    int use_graph;            /* capture the epoch as a CUDA graph after two eager epochs */
    int no_agg_first;         /* 1: widening SAGE output layers stay transform-first */
    uint32_t push_ctas;       /* CTAs of the NVLink push kernel (0: 32) */
    double peer_timeout_s;    /* peer wait traps after this (0: 20 s); a trap poisons the context */
    uint32_t heavy_degree;    /* rows above this degree run chunked (gdx_row_bins); 0: auto
                               * (max(4096, 32 x mean degree)), 0xFFFFFFFF: never */
    int fused_exchange;       /* world > 1: 1 = gdx_aggregate_exchange (one kernel per layer
                               * exchange), 0 = push kernel + two passes + wait kernel */
    int packed24;             /* 1: the gathered Z / dZ rows of 64k- and 64k+48-wide transform-first layers
                               * are stored packed-24 (fp32 rounded to 24 bits, relative 2^-16:
                               * the GEMM operands' precision) -- 25% fewer gathered bytes on
                               * L2-resident graphs; off with fused_exchange or heavy rows */
} gdx_trainer_config;
typedef struct gdx_trainer_graph {
    uint32_t num_vertices;          /* V of the whole graph */
    uint64_t nnz;                   /* full graph: row_offsets[V] */
    const uint64_t* row_offsets;    /* HOST. full graph: [V+1]; local subgraph: [local_rows+1] */
    const uint32_t* cols;           /* HOST. full graph: global ids; local subgraph: local ids */
    /* local subgraph (EAS / preload mode) when local_rows > 0: local ids ordered so that
     * the rows layer l reads / writes are prefixes rows_in[l] / rows_out[l]
     * (forward_server_local's hop mask, reference_gnn.cpp:119-137); the loss covers rows
     * < loss_rows, normalised by loss_count (the loss rows of all ranks). */
    uint64_t local_rows;
    const uint32_t* rows_in;        /* HOST [layers], nullable (= local_rows) */
    const uint32_t* rows_out;       /* HOST [layers] */
    uint32_t loss_rows;
    double loss_count;
    const uint32_t* global_ids;     /* HOST [local_rows]: stream row of each local row */
} gdx_trainer_graph;
int gdx_trainer_create(const gdx_trainer_config* cfg, const gdx_trainer_graph* graph, gdx_trainer** out);
int gdx_trainer_destroy(gdx_trainer* t);
/* Weights in reference order: per layer W [out x in] (Sum, GCN) or W_self, W_neigh (SAGE),
 * row-major fp64, all layers concatenated; count = gdx_trainer_weight_count. */
uint64_t gdx_trainer_weight_count(const gdx_trainer* t);
int gdx_trainer_init_weights(gdx_trainer* t, uint64_t seed, int he_init);  /* (seed, "weig") stream */
int gdx_trainer_set_weights(gdx_trainer* t, const double* w, uint64_t count);
int gdx_trainer_get_weights(gdx_trainer* t, double* w, uint64_t count);
int gdx_trainer_get_grads(gdx_trainer* t, double* g, uint64_t count);   /* last epoch's dW (summed) */
/* Each rank's shared buffers travel as a blob of CUDA IPC handles (same size on every rank). */
uint64_t gdx_trainer_ipc_blob_bytes(const gdx_trainer* t);
int gdx_trainer_ipc_export(gdx_trainer* t, void* blob);
int gdx_trainer_connect(gdx_trainer* t, const void* blobs);  /* world blobs, rank order */
/* One epoch (forward, loss, backward, gradient all-reduce, SGD) on the trainer's stream.
 * loss_out (nullable): the mean loss, read back (synchronising). */
int gdx_trainer_epoch(gdx_trainer* t, double* loss_out);
/* End-to-end inputs from HOST memory: stage_inputs enqueues one contiguous H2D of this
 * rank's feature block [local rows x F] fp32 (pinned memory overlaps the running epoch)
 * and labels (nullable) on a copy stream, double-buffered; step_staged consumes the
 * oldest staged block (split into the GEMM operand) and runs one epoch. */
int gdx_trainer_stage_inputs(gdx_trainer* t, const float* x_host, const int32_t* labels_host);
int gdx_trainer_step_staged(gdx_trainer* t, int with_labels, double* loss_out);
/* The trainer's stream (cudaStream_t) for event timing by the caller. */
void* gdx_trainer_stream(gdx_trainer* t);
/* out[0..]: local rows, local nnz, first row, gathered rows, loss rows, loss count,
 * graph captured, aggregate-first output layer, local-source nnz, heavy (chunked) rows. */
int gdx_trainer_info(const gdx_trainer* t, uint64_t* out, uint32_t count);
/* Per-aggregation CUDA events on eager epochs (on = 1); reading (non-null outputs)
 * returns the total ms, launch count and algorithmic bytes since on. */
int gdx_trainer_profile(gdx_trainer* t, int on, double* ms, uint64_t* launches, double* bytes);
/* The tcgen05 GEMMs of the same profiled epochs: total ms, launches, useful flops
 * (2 m n k each; read it BEFORE the gdx_trainer_profile read that resets the events). */
int gdx_trainer_profile_gemm(gdx_trainer* t, double* ms, uint64_t* launches, double* flops);

#ifdef __cplusplus
}
#endif
#endif /* GDX_H */
