// trainer.cu -- the training epoch as a C-ABI object (gdx_trainer_*, include/gdx.h):
// the layer model of reference_gnn.cpp:64-147 (forward_full / forward_server_local)
// extended with the loss, backward and SGD of BASELINE.json's north_star, driven
// from C++ so a host program runs the benchmarked epoch with no Python or torch.
//
// One object per GPU.  Two problem shapes:
//  * full graph, row partitioned: rank r owns rows [r*B, r*B+nloc) of
//    the whole CSR, B = ceil(V / world); each layer's rows are pushed into every
//    peer's copy of the gathered buffer over NVLink (CUDA IPC, SM push kernel with
//    a fused arrival signal), the locally owned sources are aggregated while the
//    push is in flight, then the remote ones;
//  * local subgraph (EAS / shared preloading, reference_gnn.cpp:91-147): the rank's
//    preloaded inner + halo rows with their hop-prefix masks; no per-layer exchange.
// Either way the weight gradients (and the loss) are summed across ranks through
// the same IPC arena: every rank pushes its slot to all peers, waits, and reduces
// the world slots in rank order (so every rank applies bit-identical SGD).
// Every launch is stream-ordered on the trainer's stream; after two eager epochs
// an epoch is captured once as a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gdx_common.cuh"

namespace gdx {
namespace {

constexpr uint64_t kFeatTag = 0x66656174ULL;   // "feat", reference_gnn.cpp:13
constexpr uint64_t kWeigTag = 0x77656967ULL;   // "weig", reference_gnn.cpp:24
constexpr uint64_t kL2Resident = 96ull << 20;  // gathered matrices up to this size stay in L2

uint64_t pad4(uint64_t x) { return (x + 3) / 4 * 4; }
uint64_t pad8(uint64_t x) { return (x + 7) / 8 * 8; }
uint64_t pad64(uint64_t x) { return (x + 63) / 64 * 64; }

__global__ void loss_to_slot(const double* loss, float* slot) { *slot = static_cast<float>(*loss); }
__global__ void slot_to_loss(const float* slot, double* loss) { *loss = static_cast<double>(*slot); }
__global__ void zero_f64(double* p) { *p = 0.0; }

struct Mat {  // fp32 rows x cols, row pitch ld (elements)
    float* p = nullptr;
    uint64_t ld = 0;
    // p24: the rows are packed-24 instead (cfg.packed24), interleaved so that a block of
    // rows is one contiguous range: row r at byte 3 ld r, high plane (ld u16) then low
    // plane (ld u8)
    int p24 = 0;
    float* row(uint64_t r) const { return p + r * ld; }
    uint64_t row_bytes() const { return p24 ? 3 * ld : 4 * ld; }
    Mat rows_from(uint64_t r) const {  // view starting at row r
        Mat v = *this;
        v.p = reinterpret_cast<float*>(reinterpret_cast<char*>(p) + r * row_bytes());
        return v;
    }
    uint16_t* hi24() const { return reinterpret_cast<uint16_t*>(p); }
    uint8_t* lo24() const { return reinterpret_cast<uint8_t*>(p) + 2 * ld; }
};
struct Spl {  // split-bf16 operand
    uint16_t* hi = nullptr;
    uint16_t* lo = nullptr;
    uint64_t ld = 0;
    uint32_t rows = 0, cols = 0;
    Spl col_view(uint32_t off, uint32_t ncols) const {
        Spl v = *this;
        v.hi += off;
        v.lo += off;
        v.cols = ncols;
        return v;
    }
    Spl rows_view(uint32_t r) const {
        Spl v = *this;
        v.rows = r;
        return v;
    }
};

struct Layer {
    bool agg_first = false;
    uint32_t fin = 0, fout = 0, k = 0, w = 0, nz = 0, fin_ld = 0, upd_cols = 0, split_k = 1;
    float* W = nullptr;
    Spl Wsp;
    float* dW = nullptr;     // this rank's reduced split-K partials (the all-reduce slot)
    float* dWsum = nullptr;  // world > 1: the all-reduced gradient (get_grads)
    uint64_t grad_off = 0;   // offset of dW inside a grad slot (floats)
    float* ws = nullptr;
    // transform-first layer
    Mat S, Zfull, dfull, Hout;
    Spl Hsp, G;
    // aggregate-first output layer
    Mat Xin_full, dAfull, dself, dtmp;
    Spl C, Gl;
};

}  // namespace
}  // namespace gdx

using namespace gdx;

struct gdx_trainer {
    gdx_trainer_config cfg{};
    std::vector<uint32_t> dims;
    int dev = 0;
    uint32_t rank = 0, world = 1;
    bool subgraph = false;
    uint32_t n = 0, F = 0, classes = 0, L = 0;
    uint64_t B = 0, lo = 0, nloc = 0, nfull = 0, nnz = 0, nnz_src = 0;
    uint32_t loss_rows = 0;
    double loss_count = 1.0;
    std::vector<uint32_t> rows_in, rows_out;
    // device state
    std::vector<void*> owned;
    uint64_t* row_ptr = nullptr;
    uint32_t* col = nullptr;
    uint64_t* seg_lo = nullptr;
    uint64_t* seg_hi = nullptr;
    float* inv_deg = nullptr;
    float* gcn_s = nullptr;
    Mat X;
    Spl Xsp;
    int32_t* labels = nullptr;
    Mat partial;
    double* loss_acc = nullptr;
    std::vector<Layer> layers;
    // IPC-shared regions, each its own cudaMalloc: region 0 = [grad slots: world x gstride
    // floats][arrival slots]; regions 1.. = the gathered buffers (full-graph mode, world > 1)
    std::vector<char*> regions;
    std::vector<uint64_t> region_bytes;
    std::vector<std::vector<int64_t>> region_delta;  // [region][peer]: peer base - our base
    char* arena = nullptr;                             // == regions[0]
    uint64_t arena_bytes = 0, gstride = 0;
    float* grad_slots = nullptr;
    unsigned long long* slots = nullptr;
    unsigned long long* expected = nullptr;
    unsigned int* push_done = nullptr;
    unsigned long long** peer_slots_dev = nullptr;
    std::vector<void*> opened;
    bool connected = false;
    // streams, graph, staging
    cudaStream_t stream = nullptr, side = nullptr, copy = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int eager_epochs = 0;
    float* stage[2] = {nullptr, nullptr};
    int32_t* stage_labels[2] = {nullptr, nullptr};
    cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    bool staged_labels[2] = {false, false};
    uint64_t issued = 0, consumed = 0;
    double* loss_host = nullptr;  // pinned
    gdx_row_bins* bins = nullptr;  // degree bins (skewed graphs), else null
    // fused exchange (cfg.fused_exchange): the pending push of the last publish, done by
    // the next exchange_aggregate's kernel
    const float* pending = nullptr;
    uint64_t pending_bytes = 0;
    unsigned int* xcounters = nullptr;
    // kernel profiling (eager epochs)
    bool profile = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    std::vector<double> prof_bytes;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gemm_events;  // tcgen05 GEMMs (useful flops)
    std::vector<double> gemm_flops;

    ~gdx_trainer();
};

namespace {

int err(int code, const std::string& m) { return fail(code, "gdx_trainer: " + m); }

#define TR_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess) return err(GDX_INTERNAL, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)
#define TR_OK(call)                 \
    do {                            \
        int _rc = (call);           \
        if (_rc != GDX_OK) return _rc; \
    } while (0)

template <class T>
int dalloc(gdx_trainer* t, T** p, uint64_t count) {
    void* q = nullptr;
    TR_CUDA(cudaMalloc(&q, std::max<uint64_t>(count, 1) * sizeof(T)));
    TR_CUDA(cudaMemset(q, 0, std::max<uint64_t>(count, 1) * sizeof(T)));
    t->owned.push_back(q);
    *p = static_cast<T*>(q);
    return GDX_OK;
}
int dmat(gdx_trainer* t, Mat* m, uint64_t rows, uint64_t cols) {
    m->ld = pad4(cols);
    return dalloc(t, &m->p, std::max<uint64_t>(rows, 1) * m->ld);
}
int dspl(gdx_trainer* t, Spl* s, uint64_t rows, uint64_t cols, uint64_t ld = 0) {
    s->ld = ld ? ld : pad8(cols);
    s->rows = static_cast<uint32_t>(rows);
    s->cols = static_cast<uint32_t>(cols);
    TR_OK(dalloc(t, &s->hi, std::max<uint64_t>(rows, 1) * s->ld));
    return dalloc(t, &s->lo, std::max<uint64_t>(rows, 1) * s->ld);
}

// Row width of a gathered matrix: 32-byte sectors when L2-resident, whole 128-byte
// lines otherwise (a misaligned row costs an extra DRAM line per gather).
uint32_t agg_width(uint32_t fout, uint64_t rows) {
    const uint64_t w8 = pad8(fout);
    if (rows * w8 * 4 <= kL2Resident) return static_cast<uint32_t>(w8);
    return fout <= 32 ? 32u : static_cast<uint32_t>((w8 + 31) / 32 * 32);
}
// Kernel per CSR shape (train.agg_variant): row groups (predicated tail) below degree 7,
// half-width row groups below 20, row groups for 48-wide rows, warp per row otherwise.
int agg_variant(uint32_t width, uint64_t nnz, uint64_t rows) {
    const double deg = rows ? static_cast<double>(nnz) / static_cast<double>(rows) : 0.0;
    if (rows && deg < 7.0) return GDX_AGG_ROWS;
    if (rows && deg < 20.0) return GDX_AGG_ROWS2;
    return pad4(width) == 48 ? GDX_AGG_ROWS : 0;
}
bool p24_wide() {  // GDX_P24_WIDE=0: 48-wide packed-24 rows through the 6-lane row groups
    static const bool on = [] {
        const char* e = std::getenv("GDX_P24_WIDE");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}
uint32_t splitk_eff(uint32_t split_k, uint64_t k) {
    const uint64_t kb = (k + 63) / 64;
    if (kb <= 1) return 1;
    const uint64_t per = (kb + std::min<uint64_t>(split_k, kb) - 1) / std::min<uint64_t>(split_k, kb);
    return static_cast<uint32_t>((kb + per - 1) / per);
}
uint32_t splitk_for(uint64_t nloc, uint32_t fin, int sms) {
    const uint64_t kb = std::max<uint64_t>(1, (nloc + 63) / 64);
    const uint32_t tile = fin > 128 ? 256 : (fin > 64 ? 128 : 64);
    const uint64_t ntiles = std::max<uint64_t>(1, (fin + tile - 1) / tile);
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kb, (2ull * sms) / ntiles)));
}

// ---- kernel calls ------------------------------------------------------------------
struct AggEpi {
    Mat out;
    Spl out_split;
    bool has_out = false, has_split = false;
    float self_coef = 0.f;
    const float* post_scale = nullptr;
    Mat add;
    bool relu = false;
};

int gemm(gdx_trainer* t, const Spl& A, const Spl& B, bool a_mn, bool b_mn, uint32_t m, Mat c0, Mat c1,
         uint32_t split, const float* row_scale, bool relu, const Spl* out_split, uint32_t split_k,
         const Mat* mask, bool split_unscaled) {
    gdx_gemm_args g{};
    g.a_hi = A.hi; g.a_lo = A.lo; g.lda = A.ld;
    g.b_hi = B.hi; g.b_lo = B.lo; g.ldb = B.ld;
    g.a_mn_major = a_mn; g.b_mn_major = b_mn;
    const uint32_t kA = a_mn ? A.rows : A.cols;
    const uint32_t nB = b_mn ? B.cols : B.rows;
    const uint32_t kB = b_mn ? B.rows : B.cols;
    if (kA != kB) return err(GDX_INTERNAL, "gemm K mismatch");
    g.m = m; g.n = nB; g.k = kA;
    g.c0 = c0.p; g.ldc0 = c0.ld;
    g.c1 = c1.p; g.ldc1 = c1.ld;
    for (int which = 0; which < 2; ++which) {  // a packed-24 output replaces its fp32 form
        const Mat& c = which ? c1 : c0;
        if (!c.p24) continue;
        if (which) g.c1 = nullptr;
        else g.c0 = nullptr;
        g.p24_hi = c.hi24(); g.p24_lo = c.lo24();
        g.ld_p24_hi = 3 * c.ld / 2; g.ld_p24_lo = 3 * c.ld;
        g.p24_target = which;
    }
    g.split = split ? split : nB;
    g.row_scale = row_scale;
    g.relu = relu;
    if (out_split) { g.out_hi = out_split->hi; g.out_lo = out_split->lo; g.ld_split = out_split->ld; }
    g.split_k = split_k;
    if (mask) { g.mask = mask->p; g.ld_mask = mask->ld; }
    g.split_unscaled = split_unscaled;
    if (!t->profile) return gdx_gemm_tn(&g, reinterpret_cast<gdx_stream>(t->stream));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    TR_CUDA(cudaEventCreate(&e0));
    TR_CUDA(cudaEventCreate(&e1));
    TR_CUDA(cudaEventRecord(e0, t->stream));
    TR_OK(gdx_gemm_tn(&g, reinterpret_cast<gdx_stream>(t->stream)));
    TR_CUDA(cudaEventRecord(e1, t->stream));
    t->gemm_events.push_back({e0, e1});
    t->gemm_flops.push_back(2.0 * m * nB * kA);  // useful flops (the split operands issue 3 bf16 MMAs per product)
    return GDX_OK;
}

int aggregate(gdx_trainer* t, const Mat& src, uint32_t width, uint32_t rows, const AggEpi& e,
              const uint64_t* row_begin, const uint64_t* row_end, const uint64_t* skip_lo,
              const uint64_t* skip_hi, const Mat* partial, uint64_t nnz_pass) {
    gdx_aggregate_args a{};
    a.row_ptr = row_begin ? row_begin : t->row_ptr;
    a.row_end = row_begin ? row_end : nullptr;
    a.skip_lo = skip_lo; a.skip_hi = skip_hi;
    if (partial) { a.partial = partial->p; a.ld_partial = partial->ld; }
    a.col = t->col;
    a.rows = rows;
    a.width = width;
    a.src = src.p; a.ld_src = src.ld;
    if (src.p24) {  // packed-24 rows: u16 high plane + u8 low plane, both at the 3 ld-byte pitch
        a.src = reinterpret_cast<const float*>(src.hi24());
        a.ld_src = 3 * src.ld / 2;
        a.src_lo8 = src.lo24();
        a.ld_src_lo8 = 3 * src.ld;
    }
    a.self_coef = e.self_coef;
    a.self_base = t->lo;
    a.post_scale = e.post_scale;
    if (e.add.p) { a.add = e.add.p; a.ld_add = e.add.ld; }
    a.relu = e.relu;
    if (e.has_out) { a.out = e.out.p; a.ld_out = e.out.ld; }
    if (e.has_split) { a.out_hi = e.out_split.hi; a.out_lo = e.out_split.lo; a.ld_split = e.out_split.ld; }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (t->profile) {
        TR_CUDA(cudaEventCreate(&e0));
        TR_CUDA(cudaEventCreate(&e1));
        TR_CUDA(cudaEventRecord(e0, t->stream));
    }
    int variant = agg_variant(width, t->nnz, t->nloc);
    // 48-wide packed-24 rows live on a 64-column pitch: gathered whole by the 8-lane kernel
    if (src.p24 && width == 48 && src.ld >= 64 && variant == GDX_AGG_ROWS && t->nloc &&
        static_cast<double>(t->nnz) / static_cast<double>(t->nloc) >= 20.0 && p24_wide())
        variant = GDX_AGG_P24_WIDE;
    TR_OK(gdx_aggregate_balanced(&a, variant, t->bins,
                                 reinterpret_cast<gdx_stream>(t->stream)));
    if (t->profile) {
        TR_CUDA(cudaEventRecord(e1, t->stream));
        t->prof_events.push_back({e0, e1});
        // 4 nnz + 8 (rows+1) + 4 F nnz + 4 F rows per launch
        // (a packed-24 source moves 3 bytes per gathered value instead of 4)
        const double eb = src.p24 ? 3.0 : 4.0;
        t->prof_bytes.push_back(4.0 * nnz_pass + 8.0 * (rows + 1.0) + eb * width * nnz_pass + 4.0 * width * rows);
    }
    return GDX_OK;
}

// Make this rank's rows [lo, lo+nloc) of a gathered buffer visible to the peers:
// SM push (16-byte NVLink stores into every peer's copy) on the side stream, forked
// from the producer and joined before the next wait.
const int64_t* deltas_for(gdx_trainer* t, const void* p) {
    for (size_t k = 0; k < t->regions.size(); ++k) {
        const char* b = t->regions[k];
        if (static_cast<const char*>(p) >= b && static_cast<const char*>(p) < b + t->region_bytes[k])
            return t->region_delta[k].data();
    }
    return nullptr;
}

int push_now(gdx_trainer* t, const float* own, uint64_t bytes);

int publish(gdx_trainer* t, const float* own, uint64_t bytes) {
    if (t->world == 1 || t->subgraph) return GDX_OK;
    if (t->cfg.fused_exchange) {  // pushed by the consuming exchange_aggregate's kernel
        t->pending = own;
        t->pending_bytes = bytes;
        return GDX_OK;
    }
    return push_now(t, own, bytes);
}

int push_now(gdx_trainer* t, const float* own, uint64_t bytes) {
    const int64_t* deltas = deltas_for(t, own);
    if (!deltas) return err(GDX_INTERNAL, "publish: buffer outside the shared regions");
    TR_CUDA(cudaEventRecord(t->ev_fork, t->stream));
    TR_CUDA(cudaStreamWaitEvent(t->side, t->ev_fork, 0));
    TR_OK(gdx_push_peers(own, bytes, deltas, t->world - 1, t->peer_slots_dev, t->push_done,
                         t->cfg.push_ctas ? t->cfg.push_ctas : 32, reinterpret_cast<gdx_stream>(t->side)));
    TR_CUDA(cudaEventRecord(t->ev_join, t->side));
    return GDX_OK;
}

int wait_peers(gdx_trainer* t) {
    TR_CUDA(cudaStreamWaitEvent(t->stream, t->ev_join, 0));
    const uint64_t timeout = t->cfg.peer_timeout_s > 0 ? static_cast<uint64_t>(t->cfg.peer_timeout_s * 1e9)
                                                        : 20000000000ull;
    return gdx_peer_wait(t->slots, t->expected, t->world, t->rank, timeout,
                         reinterpret_cast<gdx_stream>(t->stream));
}

// All-gather `full` (own rows already published) and aggregate the owned rows: the
// local sources while the push is in flight, then the remote ones + epilogue.
int exchange_aggregate(gdx_trainer* t, const Mat& full, uint32_t width, uint32_t rows, const AggEpi& e) {
    if (t->world == 1 || t->subgraph)
        return aggregate(t, full, width, rows, e, nullptr, nullptr, nullptr, nullptr, nullptr, t->nnz);
    if (t->cfg.fused_exchange) {
        const float* own = t->pending;
        const uint64_t bytes = t->pending_bytes;
        t->pending = nullptr;
        const uint32_t c4 = width / 4;
        const bool ok = width % 4 == 0 && (c4 == 8 || c4 == 12 || c4 == 16 || c4 == 32) && !t->bins && !t->profile &&
                        own && rows == t->nloc;
        if (!ok) {  // not fusable here: the two-pass path with the deferred push
            if (own) TR_OK(push_now(t, own, bytes));
        } else {
            gdx_aggregate_args a{};
            a.row_ptr = t->row_ptr;
            a.col = t->col;
            a.rows = rows;
            a.width = width;
            a.src = full.p;
            a.ld_src = full.ld;
            a.self_coef = e.self_coef;
            a.self_base = t->lo;
            a.post_scale = e.post_scale;
            if (e.add.p) { a.add = e.add.p; a.ld_add = e.add.ld; }
            a.relu = e.relu;
            if (e.has_out) { a.out = e.out.p; a.ld_out = e.out.ld; }
            if (e.has_split) { a.out_hi = e.out_split.hi; a.out_lo = e.out_split.lo; a.ld_split = e.out_split.ld; }
            const uint64_t timeout = t->cfg.peer_timeout_s > 0 ? static_cast<uint64_t>(t->cfg.peer_timeout_s * 1e9)
                                                                : 20000000000ull;
            return gdx_aggregate_exchange(&a, t->seg_lo, t->seg_hi, t->partial.p, t->partial.ld, own, bytes,
                                          deltas_for(t, own), t->world - 1, t->peer_slots_dev, t->slots, t->expected,
                                          t->world, t->rank, t->xcounters, timeout,
                                          reinterpret_cast<gdx_stream>(t->stream));
        }
    }
    Mat P = t->partial;  // first pad4(width) columns, pitch of the widest layer
    AggEpi pe;
    pe.out = P;
    pe.has_out = true;
    TR_OK(aggregate(t, full, width, rows, pe, t->seg_lo, t->seg_hi, nullptr, nullptr, nullptr, t->nnz_src));
    TR_OK(wait_peers(t));
    return aggregate(t, full, width, rows, e, nullptr, nullptr, t->seg_lo, t->seg_hi, &P, t->nnz - t->nnz_src);
}

Mat act(gdx_trainer* t, uint32_t l) {  // fp32 output rows of layer l (ReLU mask)
    if (l + 1 < t->L && t->layers[l + 1].agg_first) {
        Mat v = t->layers[l + 1].Xin_full;
        v.p = v.row(t->lo);
        return v;
    }
    return t->layers[l].Hout;
}

// ---- one epoch ---------------------------------------------------------------------
int forward(gdx_trainer* t) {
    const int kind = t->cfg.kind;
    Spl A = t->Xsp;
    for (uint32_t l = 0; l < t->L; ++l) {
        Layer& Ly = t->layers[l];
        const bool relu = l + 1 < t->L;
        const uint32_t m_in = t->rows_in[l], r_out = t->rows_out[l];
        if (Ly.agg_first) {
            Mat own = Ly.Xin_full;
            own.p = own.row(t->lo);
            TR_OK(publish(t, own.p, t->nloc * Ly.Xin_full.ld * 4));
            AggEpi e;
            e.out_split = Ly.C.col_view(Ly.w, Ly.w);
            e.has_split = true;
            e.post_scale = t->inv_deg;
            TR_OK(exchange_aggregate(t, Ly.Xin_full, Ly.w, r_out, e));
            TR_OK(gemm(t, Ly.C, Ly.Wsp, false, false, r_out, Ly.Hout, Mat{}, 0, nullptr, false, nullptr, 1,
                       nullptr, false));
            continue;
        }
        Mat own = Ly.Zfull.rows_from(t->lo);
        if (kind == GDX_MODEL_SAGE)
            TR_OK(gemm(t, A, Ly.Wsp, false, false, m_in, Ly.S, own, Ly.w, nullptr, false, nullptr, 1, nullptr, false));
        else
            TR_OK(gemm(t, A, Ly.Wsp, false, false, m_in, own, Mat{}, 0, kind == GDX_MODEL_GCN ? t->gcn_s : nullptr,
                       false, nullptr, 1, nullptr, false));
        TR_OK(publish(t, own.p, t->nloc * Ly.Zfull.row_bytes()));
        AggEpi e;
        e.has_out = e.has_split = true;
        if (l + 1 < t->L && t->layers[l + 1].agg_first) {
            Layer& nx = t->layers[l + 1];
            e.out = nx.Xin_full;
            e.out.p = e.out.row(t->lo);
            e.out_split = nx.C.col_view(0, nx.w);
        } else {
            e.out = Ly.Hout;
            e.out_split = Ly.Hsp;
        }
        e.relu = relu;
        if (kind == GDX_MODEL_SAGE) {
            e.post_scale = t->inv_deg;
            e.add = Ly.S;
        } else {
            e.self_coef = 1.f;
            if (kind == GDX_MODEL_GCN) e.post_scale = t->gcn_s;
        }
        TR_OK(exchange_aggregate(t, Ly.Zfull, Ly.w, r_out, e));
        A = Ly.Hsp;
    }
    return GDX_OK;
}

// Where layer l's output gradient goes: gs = g * dst_scale into the gathered buffer's
// own rows; for SAGE also the unscaled split copy into G[:, :w].
struct GradTargets {
    Mat own;
    const float* scale = nullptr;
    const Spl* split = nullptr;
};
GradTargets grad_targets(gdx_trainer* t, uint32_t l) {
    Layer& Ly = t->layers[l];
    GradTargets g;
    g.own = Ly.dfull.rows_from(t->lo);
    if (t->cfg.kind == GDX_MODEL_SAGE) {
        g.scale = t->inv_deg;
        g.split = &Ly.G;
    } else if (t->cfg.kind == GDX_MODEL_GCN) {
        g.scale = t->gcn_s;
    }
    return g;
}

int sgd_or_reduce(gdx_trainer* t, Layer& Ly, uint32_t sk) {
    if (t->world == 1)
        return gdx_splitk_reduce(Ly.ws, sk, uint64_t(Ly.nz) * Ly.fin_ld, Ly.nz, Ly.upd_cols, Ly.fin_ld, Ly.dW, Ly.W,
                                 t->cfg.lr, Ly.Wsp.hi, Ly.Wsp.lo, reinterpret_cast<gdx_stream>(t->stream));
    return gdx_splitk_reduce(Ly.ws, sk, uint64_t(Ly.nz) * Ly.fin_ld, Ly.nz, Ly.upd_cols, Ly.fin_ld, Ly.dW, nullptr,
                             0.f, nullptr, nullptr, reinterpret_cast<gdx_stream>(t->stream));
}

int backward_agg_first(gdx_trainer* t, uint32_t l) {
    Layer& Ly = t->layers[l];
    const uint32_t r = t->rows_out[l];
    const Spl w0 = Ly.Wsp.col_view(0, Ly.w), w1 = Ly.Wsp.col_view(Ly.w, Ly.w);
    TR_OK(gemm(t, Ly.Gl, w0, false, true, r, Ly.dself, Mat{}, 0, nullptr, false, nullptr, 1, nullptr, false));
    Mat own = Ly.dAfull;
    own.p = own.row(t->lo);
    TR_OK(gemm(t, Ly.Gl, w1, false, true, r, own, Mat{}, 0, t->inv_deg, false, nullptr, 1, nullptr, false));
    TR_OK(publish(t, own.p, t->nloc * Ly.dAfull.ld * 4));
    const uint32_t sk = splitk_eff(Ly.split_k, r);
    Mat wsm{Ly.ws, Ly.fin_ld};
    TR_OK(gemm(t, Ly.Gl.rows_view(r), Ly.C.rows_view(r), true, true, Ly.nz, wsm, Mat{}, 0, nullptr, false, nullptr,
               sk, nullptr, false));
    TR_OK(sgd_or_reduce(t, Ly, sk));
    AggEpi e;
    e.out = Ly.dtmp;
    e.has_out = true;
    e.add = Ly.dself;
    TR_OK(exchange_aggregate(t, Ly.dAfull, Ly.w, t->rows_in[l], e));
    GradTargets gt = grad_targets(t, l - 1);
    if (gt.own.p24) return err(GDX_INTERNAL, "grad_prepare: packed-24 gradient rows");
    const Mat a = act(t, l - 1);
    TR_OK(gdx_grad_prepare(Ly.dtmp.p, Ly.dtmp.ld, a.p, a.ld, t->rows_out[l - 1], Ly.w, gt.scale, nullptr, 0, gt.own.p,
                           gt.own.ld, gt.split ? gt.split->hi : nullptr, gt.split ? gt.split->lo : nullptr,
                           gt.split ? gt.split->ld : 0, reinterpret_cast<gdx_stream>(t->stream)));
    return publish(t, gt.own.p, t->nloc * t->layers[l - 1].dfull.row_bytes());
}

int backward_and_step(gdx_trainer* t) {
    const int kind = t->cfg.kind;
    for (int li = static_cast<int>(t->L) - 1; li >= 0; --li) {
        const uint32_t l = static_cast<uint32_t>(li);
        Layer& Ly = t->layers[l];
        if (Ly.agg_first) {
            TR_OK(backward_agg_first(t, l));
            continue;
        }
        const uint32_t r_in = t->rows_in[l];
        AggEpi e;
        e.has_split = true;
        if (kind == GDX_MODEL_SAGE) {
            e.out_split = Ly.G.col_view(Ly.w, Ly.w);
        } else {
            e.out_split = Ly.G;
            e.self_coef = 1.f;
            if (kind == GDX_MODEL_GCN) e.post_scale = t->gcn_s;
        }
        TR_OK(exchange_aggregate(t, Ly.dfull, Ly.w, r_in, e));
        if (l > 0) {  // dH_{l-1} = G W_cat, ReLU mask + scale + split fused in the epilogue
            GradTargets gt = grad_targets(t, l - 1);
            const Mat a = act(t, l - 1);
            TR_OK(gemm(t, Ly.G, Ly.Wsp, false, true, t->rows_out[l - 1], gt.own, Mat{}, 0, gt.scale, false,
                       gt.split, 1, &a, true));
            TR_OK(publish(t, gt.own.p, t->nloc * t->layers[l - 1].dfull.row_bytes()));
        }
        const Spl A_in = l == 0 ? t->Xsp : t->layers[l - 1].Hsp;
        const uint32_t sk = splitk_eff(Ly.split_k, r_in);
        Mat wsm{Ly.ws, Ly.fin_ld};
        TR_OK(gemm(t, Ly.G.rows_view(r_in), A_in.rows_view(r_in), true, true, Ly.nz, wsm, Mat{}, 0, nullptr, false,
                   nullptr, sk, nullptr, false));
        TR_OK(sgd_or_reduce(t, Ly, sk));
    }
    if (t->world > 1) {  // one all-reduce of every dW + the loss, then SGD on every rank
        float* mine = t->grad_slots + uint64_t(t->rank) * t->gstride;
        loss_to_slot<<<1, 1, 0, t->stream>>>(t->loss_acc, mine + t->gstride - 4);
        note_launch();
        TR_CUDA(cudaEventRecord(t->ev_fork, t->stream));
        TR_CUDA(cudaStreamWaitEvent(t->side, t->ev_fork, 0));
        TR_OK(gdx_push_peers(mine, t->gstride * 4, t->region_delta[0].data(), t->world - 1, t->peer_slots_dev,
                             t->push_done, 8,
                             reinterpret_cast<gdx_stream>(t->side)));
        TR_CUDA(cudaEventRecord(t->ev_join, t->side));
        TR_OK(wait_peers(t));
        for (Layer& Ly : t->layers)
            TR_OK(gdx_splitk_reduce(t->grad_slots + Ly.grad_off, t->world, t->gstride, Ly.nz, Ly.upd_cols, Ly.fin_ld,
                                    Ly.dWsum, Ly.W, t->cfg.lr, Ly.Wsp.hi, Ly.Wsp.lo,
                                    reinterpret_cast<gdx_stream>(t->stream)));
        TR_OK(gdx_splitk_reduce(t->grad_slots + t->gstride - 4, t->world, t->gstride, 1, 1, 1,
                                t->grad_slots + t->gstride - 3 + uint64_t(t->rank) * t->gstride, nullptr, 0.f,
                                nullptr, nullptr, reinterpret_cast<gdx_stream>(t->stream)));
        slot_to_loss<<<1, 1, 0, t->stream>>>(t->grad_slots + t->gstride - 3 + uint64_t(t->rank) * t->gstride,
                                             t->loss_acc);
        note_launch();
    }
    return GDX_OK;
}

int epoch_body(gdx_trainer* t) {
    zero_f64<<<1, 1, 0, t->stream>>>(t->loss_acc);
    note_launch();
    TR_OK(forward(t));
    Layer& last = t->layers.back();
    const gdx_stream s = reinterpret_cast<gdx_stream>(t->stream);
    const float inv = static_cast<float>(1.0 / t->loss_count);
    if (last.agg_first) {
        TR_OK(gdx_softmax_xent_fused(last.Hout.p, last.Hout.ld, t->loss_rows, t->classes, t->labels, inv, nullptr, 0,
                                     nullptr, nullptr, 0, last.Gl.hi, last.Gl.lo, last.Gl.ld, t->loss_acc, s));
    } else {
        GradTargets gt = grad_targets(t, t->L - 1);
        if (gt.own.p24)
            TR_OK(gdx_softmax_xent_fused_p24(last.Hout.p, last.Hout.ld, t->loss_rows, t->classes, t->labels, inv,
                                             gt.scale, gt.own.hi24(), 3 * gt.own.ld / 2, gt.own.lo24(), 3 * gt.own.ld,
                                             gt.split ? gt.split->hi : nullptr, gt.split ? gt.split->lo : nullptr,
                                             gt.split ? gt.split->ld : 0, t->loss_acc, s));
        else
            TR_OK(gdx_softmax_xent_fused(last.Hout.p, last.Hout.ld, t->loss_rows, t->classes, t->labels, inv,
                                         nullptr, 0, gt.scale, gt.own.p, gt.own.ld,
                                         gt.split ? gt.split->hi : nullptr, gt.split ? gt.split->lo : nullptr,
                                         gt.split ? gt.split->ld : 0, t->loss_acc, s));
        TR_OK(publish(t, gt.own.p, t->nloc * last.dfull.row_bytes()));
    }
    return backward_and_step(t);
}

int setup_model(gdx_trainer* t) {
    const int sms = device_sms();
    const int kind = t->cfg.kind;
    // shared arena layout: grad slots first (same offset on every rank), arrival slots,
    // then (full-graph mode) the exchanged buffers
    std::vector<uint64_t> gsize(t->L);
    t->layers.resize(t->L);
    for (uint32_t l = 0; l < t->L; ++l) {
        Layer& Ly = t->layers[l];
        Ly.fin = t->dims[l];
        Ly.fout = t->dims[l + 1];
        const uint32_t prev_w = l ? t->layers[l - 1].w : 0;
        Ly.agg_first = l == t->L - 1 && l > 0 && kind == GDX_MODEL_SAGE && !t->cfg.no_agg_first &&
                       agg_width(Ly.fout, t->nfull) > prev_w;
        if (Ly.agg_first) {
            Ly.w = prev_w;
            Ly.k = 2 * prev_w;
            Ly.fin_ld = Ly.k;
            Ly.upd_cols = Ly.k;
            Ly.nz = static_cast<uint32_t>(pad8(Ly.fout));
        } else {
            Ly.k = l == 0 ? Ly.fin : prev_w;
            Ly.w = agg_width(Ly.fout, t->nfull);
            Ly.nz = kind == GDX_MODEL_SAGE ? 2 * Ly.w : Ly.w;
            Ly.fin_ld = static_cast<uint32_t>(pad8(Ly.k));
            Ly.upd_cols = Ly.fin;
        }
        Ly.split_k = splitk_for(t->nloc, Ly.agg_first ? Ly.k : Ly.fin, sms);
        gsize[l] = uint64_t(Ly.nz) * Ly.fin_ld;
    }
    uint64_t g = 0;
    for (uint32_t l = 0; l < t->L; ++l) {
        t->layers[l].grad_off = g;
        g += gsize[l];
    }
    t->gstride = pad64(g + 4);  // + loss slot (2 floats used), 256-byte aligned slots
    uint64_t off = t->gstride * 4 * t->world;
    const uint64_t slots_off = off;
    off += 256 + pad64(8 * t->world);
    std::vector<uint64_t> xoff;
    if (!t->subgraph && t->world > 1) {
        for (uint32_t l = 0; l < t->L; ++l) {
            const Layer& Ly = t->layers[l];
            const uint64_t bytes = t->nfull * pad4(Ly.w) * 4;
            xoff.push_back(off);
            off += (bytes + 255) / 256 * 256;
            xoff.push_back(off);
            off += (bytes + 255) / 256 * 256;
        }
    }
    // region 0: grad slots + arrival slots; one region per gathered buffer
    t->arena_bytes = slots_off + 256 + pad64(8 * t->world);
    std::vector<uint64_t> sizes{t->arena_bytes};
    for (size_t j = 0; j < xoff.size(); ++j) {
        const uint64_t end = j + 1 < xoff.size() ? xoff[j + 1] : off;
        sizes.push_back(end - xoff[j]);
    }
    for (uint64_t b : sizes) {
        char* r = nullptr;
        TR_CUDA(cudaMalloc(&r, b));
        TR_CUDA(cudaMemset(r, 0, b));
        t->regions.push_back(r);
        t->region_bytes.push_back(b);
    }
    t->arena = t->regions[0];
    t->grad_slots = reinterpret_cast<float*>(t->arena);
    t->slots = reinterpret_cast<unsigned long long*>(t->arena + slots_off + 256);
    TR_OK(dalloc(t, &t->expected, 1));
    TR_OK(dalloc(t, &t->push_done, 1));
    TR_OK(dalloc(t, &t->xcounters, 2));
    TR_OK(dalloc(t, &t->peer_slots_dev, 8));
    for (uint32_t l = 0; l < t->L; ++l) {
        Layer& Ly = t->layers[l];
        Ly.dW = t->grad_slots + uint64_t(t->rank) * t->gstride + Ly.grad_off;
        if (t->world > 1) TR_OK(dalloc(t, &Ly.dWsum, gsize[l]));
        TR_OK(dalloc(t, &Ly.W, gsize[l]));
        TR_OK(dspl(t, &Ly.Wsp, Ly.nz, Ly.k, Ly.fin_ld));
        TR_OK(dalloc(t, &Ly.ws, uint64_t(Ly.split_k) * gsize[l]));
        auto shared = [&](Mat* m, uint32_t width, int which) -> int {
            if (xoff.empty()) return dmat(t, m, t->nfull, width);
            m->ld = pad4(width);
            m->p = reinterpret_cast<float*>(t->regions[1 + 2 * l + which]);
            return GDX_OK;
        };
        if (Ly.agg_first) {
            TR_OK(shared(&Ly.Xin_full, Ly.w, 0));
            TR_OK(shared(&Ly.dAfull, Ly.w, 1));
            TR_OK(dspl(t, &Ly.C, t->nloc, Ly.k));
            TR_OK(dmat(t, &Ly.Hout, t->nloc, Ly.nz));
            TR_OK(dspl(t, &Ly.Gl, t->nloc, Ly.nz));
            TR_OK(dmat(t, &Ly.dself, t->nloc, Ly.w));
            TR_OK(dmat(t, &Ly.dtmp, t->nloc, Ly.w));
        } else {
            if (kind == GDX_MODEL_SAGE) TR_OK(dmat(t, &Ly.S, t->nloc, Ly.w));
            TR_OK(shared(&Ly.Zfull, Ly.w, 0));
            TR_OK(shared(&Ly.dfull, Ly.w, 1));
            TR_OK(dmat(t, &Ly.Hout, t->nloc, Ly.w));
            TR_OK(dspl(t, &Ly.Hsp, t->nloc, Ly.w));
            TR_OK(dspl(t, &Ly.G, t->nloc, Ly.nz));
        }
    }
    // packed-24 gathered rows (cfg.packed24) for 64k-wide transform-first layers: Z from
    // the forward GEMM's epilogue, dZ from the dH GEMM's (not from the softmax or
    // grad_prepare kernels, which write fp32)
    // grad_prepare kernels, which write fp32).  A 64k+48-wide layer (the 41-class output
    // layer) keeps a 64k+64 plane pitch -- the same bytes as its fp32 rows -- so a gathered
    // row is 3 + 2 aligned sectors instead of 6 (GDX_P24_48=0 keeps those layers fp32);
    // its dZ comes out of the softmax kernel (gdx_softmax_xent_fused_p24).
    const bool p24_ok = t->cfg.packed24 && !t->cfg.fused_exchange && (!t->bins || t->bins->n_heavy == 0);
    static const bool p24_48 = [] {
        const char* e = std::getenv("GDX_P24_48");
        return !e || std::atoi(e) != 0;
    }();
    for (uint32_t l = 0; l < t->L && p24_ok; ++l) {
        Layer& Ly = t->layers[l];
        const bool w48 = Ly.w % 64 == 48 && p24_48;
        if (Ly.agg_first || (Ly.w % 64 != 0 && !w48)) continue;
        const uint64_t ld24 = w48 ? Ly.w + 16 : Ly.Zfull.ld;
        Ly.Zfull.p24 = 1;
        Ly.Zfull.ld = ld24;
        const bool last = l + 1 == t->L;
        Ly.dfull.p24 = last ? t->classes <= 128 && t->classes <= Ly.w : !t->layers[l + 1].agg_first;
        if (Ly.dfull.p24) Ly.dfull.ld = ld24;
    }
    if (!t->subgraph && t->world > 1) {
        uint32_t wmax = 0;
        for (const Layer& Ly : t->layers) wmax = std::max(wmax, Ly.w);
        TR_OK(dmat(t, &t->partial, t->nloc, wmax));
    }
    TR_OK(dalloc(t, &t->loss_acc, 1));
    return GDX_OK;
}

int upload_weights(gdx_trainer* t, const double* w, uint64_t count) {
    uint64_t need = 0;
    for (uint32_t l = 0; l < t->L; ++l)
        need += uint64_t(t->dims[l + 1]) * t->dims[l] * (t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1);
    if (count != need)
        return err(GDX_INPUT, "set_weights: expected " + std::to_string(need) + " values, got " + std::to_string(count));
    for (Layer& Ly : t->layers) {
        std::vector<float> h(uint64_t(Ly.nz) * Ly.fin_ld, 0.f);
        const uint32_t nm = t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1;
        for (uint32_t m = 0; m < nm; ++m) {
            // W_self (m = 0) / W_neigh (m = 1) placement of train.py _Layer / _AggFirstLayer
            const uint64_t r0 = Ly.agg_first ? 0 : uint64_t(m) * Ly.w;
            const uint64_t c0 = Ly.agg_first ? uint64_t(m) * Ly.w : 0;
            for (uint32_t r = 0; r < Ly.fout; ++r)
                for (uint32_t c = 0; c < Ly.fin; ++c) h[(r0 + r) * Ly.fin_ld + c0 + c] = static_cast<float>(w[uint64_t(r) * Ly.fin + c]);
            w += uint64_t(Ly.fout) * Ly.fin;
        }
        TR_CUDA(cudaMemcpy(Ly.W, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        TR_OK(gdx_split_bf16(Ly.W, Ly.fin_ld, Ly.nz, Ly.k, Ly.Wsp.hi, Ly.Wsp.lo, Ly.fin_ld, 0, nullptr));
    }
    TR_CUDA(cudaDeviceSynchronize());
    return GDX_OK;
}

int read_weights(gdx_trainer* t, double* out, uint64_t count, bool grads) {
    TR_CUDA(cudaStreamSynchronize(t->stream));
    uint64_t need = 0;
    for (uint32_t l = 0; l < t->L; ++l)
        need += uint64_t(t->dims[l + 1]) * t->dims[l] * (t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1);
    if (count != need) return err(GDX_INPUT, "get_weights: expected a buffer of " + std::to_string(need));
    for (Layer& Ly : t->layers) {
        std::vector<float> h(uint64_t(Ly.nz) * Ly.fin_ld);
        const float* src = grads ? (t->world > 1 ? Ly.dWsum : Ly.dW) : Ly.W;
        TR_CUDA(cudaMemcpy(h.data(), src, h.size() * 4, cudaMemcpyDeviceToHost));
        const uint32_t nm = t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1;
        for (uint32_t m = 0; m < nm; ++m) {
            const uint64_t r0 = Ly.agg_first ? 0 : uint64_t(m) * Ly.w;
            const uint64_t c0 = Ly.agg_first ? uint64_t(m) * Ly.w : 0;
            for (uint32_t r = 0; r < Ly.fout; ++r)
                for (uint32_t c = 0; c < Ly.fin; ++c) out[uint64_t(r) * Ly.fin + c] = h[(r0 + r) * Ly.fin_ld + c0 + c];
            out += uint64_t(Ly.fout) * Ly.fin;
        }
    }
    return GDX_OK;
}

int run_epoch(gdx_trainer* t) {
    if (t->world > 1 && !t->connected) return err(GDX_CONTRACT, "world > 1: gdx_trainer_connect first");
    if (t->exec) {
        TR_CUDA(cudaGraphLaunch(t->exec, t->stream));
        note_launch();
        return GDX_OK;
    }
    if (t->cfg.use_graph && !t->profile && t->eager_epochs >= 2) {
        // capture one epoch (every launch is on t->stream or forked from it)
        TR_CUDA(cudaStreamBeginCapture(t->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = epoch_body(t);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(t->stream, &g);
        if (rc != GDX_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        TR_CUDA(e);
        t->graph = g;
        TR_CUDA(cudaGraphInstantiate(&t->exec, g, 0));
        TR_CUDA(cudaGraphLaunch(t->exec, t->stream));
        note_launch();
        return GDX_OK;
    }
    TR_OK(epoch_body(t));
    t->eager_epochs++;
    return GDX_OK;
}

}  // namespace

gdx_trainer::~gdx_trainer() {
    if (stream) cudaStreamSynchronize(stream);
    if (bins) gdx_row_bins_free(bins);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto& e : prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto& e : gemm_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    for (void* p : owned) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        if (stage[i]) cudaFree(stage[i]);
        if (stage_labels[i]) cudaFree(stage_labels[i]);
        if (ready[i]) cudaEventDestroy(ready[i]);
        if (freed[i]) cudaEventDestroy(freed[i]);
    }
    if (loss_host) cudaFreeHost(loss_host);
    for (char* r : regions) cudaFree(r);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (copy) cudaStreamDestroy(copy);
    if (stream) cudaStreamDestroy(stream);
}

// ======================= C ABI =============================================
extern "C" int gdx_trainer_create(const gdx_trainer_config* cfg, const gdx_trainer_graph* gr, gdx_trainer** out) {
    GDX_REQUIRE(cfg && gr && out, GDX_INPUT, "gdx_trainer_create: null pointer");
    *out = nullptr;
    GDX_REQUIRE(cfg->kind == GDX_MODEL_SUM || cfg->kind == GDX_MODEL_GCN || cfg->kind == GDX_MODEL_SAGE, GDX_INPUT,
                "gdx_trainer_create: unknown model kind");
    GDX_REQUIRE(cfg->layers >= 1 && cfg->dims, GDX_INPUT, "gdx_trainer_create: need >= 1 layer and dims");
    GDX_REQUIRE(cfg->world >= 1 && cfg->world <= 8 && cfg->rank < cfg->world, GDX_INPUT,
                "gdx_trainer_create: world must be 1..8 (<= 7 peers), rank < world");
    for (uint32_t l = 0; l <= cfg->layers; ++l)
        GDX_REQUIRE(cfg->dims[l] >= 1, GDX_INPUT, "gdx_trainer_create: dims must be >= 1");
    GDX_REQUIRE(cfg->dims[cfg->layers] <= 256, GDX_INPUT, "gdx_trainer_create: classes must be <= 256");
    GDX_REQUIRE(gr->row_offsets && (gr->cols || gr->nnz == 0), GDX_INPUT, "gdx_trainer_create: null CSR");
    std::unique_ptr<gdx_trainer> t(new gdx_trainer());
    t->cfg = *cfg;
    t->dims.assign(cfg->dims, cfg->dims + cfg->layers + 1);
    t->cfg.dims = t->dims.data();
    t->dev = cfg->device;
    t->rank = cfg->rank;
    t->world = cfg->world;
    t->L = cfg->layers;
    t->F = t->dims[0];
    t->classes = t->dims[t->L];
    GDX_CUDA(cudaSetDevice(t->dev));
    GDX_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    {   // the NVLink push stream; GDX_TR_PUSH_PRIO=high gives it the highest priority
        int least = 0, greatest = 0;
        GDX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        const char* pr = std::getenv("GDX_TR_PUSH_PRIO");
        const int prio = (pr && std::string(pr) == "high") ? greatest : least;
        GDX_CUDA(cudaStreamCreateWithPriority(&t->side, cudaStreamNonBlocking, prio));
    }
    GDX_CUDA(cudaStreamCreateWithFlags(&t->copy, cudaStreamNonBlocking));
    GDX_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
    GDX_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
    GDX_CUDA(cudaMallocHost(&t->loss_host, sizeof(double)));
    const uint64_t* ro = gr->row_offsets;
    std::vector<uint64_t> lro;
    std::vector<uint32_t> gid;  // feature / label stream row of every local row
    if (gr->local_rows == 0) {  // full graph, row partitioned
        t->subgraph = false;
        t->n = gr->num_vertices;
        t->B = (uint64_t(t->n) + t->world - 1) / t->world;
        t->lo = std::min<uint64_t>(uint64_t(t->rank) * t->B, t->n);
        const uint64_t hi = std::min<uint64_t>(t->lo + t->B, t->n);
        t->nloc = hi - t->lo;
        t->nfull = t->B * t->world;
        const uint64_t base = ro[t->lo];
        lro.resize(t->nloc + 1);
        for (uint64_t i = 0; i <= t->nloc; ++i) lro[i] = ro[t->lo + i] - base;
        t->nnz = lro[t->nloc];
        GDX_REQUIRE(ro[t->n] == gr->nnz, GDX_INPUT, "gdx_trainer_create: row_offsets[n] != nnz");
        t->loss_rows = static_cast<uint32_t>(t->nloc);
        t->loss_count = static_cast<double>(t->n);
        t->rows_in.assign(t->L, static_cast<uint32_t>(t->nloc));
        t->rows_out.assign(t->L, static_cast<uint32_t>(t->nloc));
        if (int rc = dalloc(t.get(), &t->row_ptr, t->nloc + 1)) return rc;
        if (int rc = dalloc(t.get(), &t->col, std::max<uint64_t>(t->nnz, 1))) return rc;
        GDX_CUDA(cudaMemcpy(t->row_ptr, lro.data(), (t->nloc + 1) * 8, cudaMemcpyHostToDevice));
        if (t->nnz)
            GDX_CUDA(cudaMemcpy(t->col, gr->cols + base, t->nnz * 4, cudaMemcpyHostToDevice));
    } else {  // local subgraph: rows are local ids, prefixes given per layer
        t->subgraph = true;
        GDX_REQUIRE(gr->rows_out && gr->loss_count > 0, GDX_INPUT,
                    "gdx_trainer_create: a local subgraph needs rows_out[layers] and loss_count");
        t->n = gr->num_vertices;
        t->nloc = gr->local_rows;
        t->lo = 0;
        t->B = t->nloc;
        t->nfull = t->nloc;
        lro.assign(ro, ro + t->nloc + 1);
        t->nnz = lro[t->nloc] - lro[0];
        for (auto& x : lro) x -= ro[0];
        t->loss_rows = gr->loss_rows;
        t->loss_count = gr->loss_count;
        t->rows_out.assign(gr->rows_out, gr->rows_out + t->L);
        t->rows_in.resize(t->L);
        for (uint32_t l = 0; l < t->L; ++l) t->rows_in[l] = gr->rows_in ? gr->rows_in[l] : static_cast<uint32_t>(t->nloc);
        if (int rc = dalloc(t.get(), &t->row_ptr, t->nloc + 1)) return rc;
        if (int rc = dalloc(t.get(), &t->col, std::max<uint64_t>(t->nnz, 1))) return rc;
        GDX_CUDA(cudaMemcpy(t->row_ptr, lro.data(), (t->nloc + 1) * 8, cudaMemcpyHostToDevice));
        if (t->nnz) GDX_CUDA(cudaMemcpy(t->col, gr->cols + ro[0], t->nnz * 4, cudaMemcpyHostToDevice));
    }
    // degree bins for skewed graphs: hub rows are chunked across warps
    {
        uint64_t maxd = 0;
        for (uint64_t i = 0; i < t->nloc; ++i) maxd = std::max<uint64_t>(maxd, lro[i + 1] - lro[i]);
        const double mean = t->nloc ? static_cast<double>(t->nnz) / static_cast<double>(t->nloc) : 0.0;
        const uint64_t thr = cfg->heavy_degree ? cfg->heavy_degree
                                               : std::max<uint64_t>(4096, static_cast<uint64_t>(32.0 * mean));
        if (cfg->heavy_degree != 0xFFFFFFFFu && maxd > thr) {
            uint32_t wmax = 8;
            for (uint32_t l = 1; l <= t->L; ++l) wmax = std::max<uint32_t>(wmax, static_cast<uint32_t>(pad8(t->dims[l])));
            if (int rc = gdx_row_bins_build(lro.data(), static_cast<uint32_t>(t->nloc), static_cast<uint32_t>(thr), 1024,
                                            (wmax + 31) / 32 * 32, &t->bins))
                return rc;
        }
    }
    // degree scales, fp64 then rounded (train.py: 1/deg, (deg+1)^-1/2)
    std::vector<float> inv(std::max<uint64_t>(t->nloc, 1), 0.f), gs(std::max<uint64_t>(t->nloc, 1), 0.f);
    for (uint64_t i = 0; i < t->nloc; ++i) {
        const double d = static_cast<double>(lro[i + 1] - lro[i]);
        inv[i] = d > 0 ? static_cast<float>(1.0 / d) : 0.f;
        gs[i] = static_cast<float>(1.0 / std::sqrt(d + 1.0));
    }
    if (int rc = dalloc(t.get(), &t->inv_deg, inv.size())) return rc;
    if (int rc = dalloc(t.get(), &t->gcn_s, gs.size())) return rc;
    GDX_CUDA(cudaMemcpy(t->inv_deg, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
    GDX_CUDA(cudaMemcpy(t->gcn_s, gs.data(), gs.size() * 4, cudaMemcpyHostToDevice));
    if (!t->subgraph && t->world > 1) {
        if (int rc = dalloc(t.get(), &t->seg_lo, std::max<uint64_t>(t->nloc, 1))) return rc;
        if (int rc = dalloc(t.get(), &t->seg_hi, std::max<uint64_t>(t->nloc, 1))) return rc;
        if (int rc = gdx_row_split(t->row_ptr, t->col, static_cast<uint32_t>(t->nloc), static_cast<uint32_t>(t->lo),
                                   static_cast<uint32_t>(t->lo + t->nloc), t->seg_lo, t->seg_hi, nullptr))
            return rc;
        // local-source edge count (per-launch bytes of the profiled split passes)
        std::vector<uint64_t> a(t->nloc), b(t->nloc);
        GDX_CUDA(cudaMemcpy(a.data(), t->seg_lo, t->nloc * 8, cudaMemcpyDeviceToHost));
        GDX_CUDA(cudaMemcpy(b.data(), t->seg_hi, t->nloc * 8, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < t->nloc; ++i) t->nnz_src += b[i] - a[i];
    }
    // inputs: the keyed feature / label streams of the rows' global ids
    if (int rc = dmat(t.get(), &t->X, t->nloc, t->F)) return rc;
    if (int rc = dspl(t.get(), &t->Xsp, t->nloc, t->F)) return rc;
    if (int rc = dalloc(t.get(), &t->labels, std::max<uint64_t>(t->nloc, 1))) return rc;
    if (!t->subgraph) {
        if (t->nloc) {
            if (int rc = gdx_init_uniform(cfg->feature_seed, kFeatTag, 0, t->lo * t->F, static_cast<uint32_t>(t->nloc),
                                          t->F, -0.5, 0.5, t->X.p, t->X.ld, nullptr))
                return rc;
            if (int rc = gdx_init_labels(cfg->label_seed, t->lo, static_cast<uint32_t>(t->nloc), t->classes, t->labels,
                                         nullptr))
                return rc;
        }
    } else if (gr->global_ids && t->nloc) {
        // preloaded rows: the streams' rows at the local vertices' global ids (one
        // generation over all V, then a row gather); inputs beyond L hops (rows >=
        // rows_in[0]) stay zero (reference_gnn.cpp:129-131)
        const uint32_t avail = t->rows_in[0];
        uint32_t* dids = nullptr;
        float* all = nullptr;
        int32_t* lab_all = nullptr;
        if (int rc = dalloc(t.get(), &dids, t->nloc)) return rc;
        GDX_CUDA(cudaMemcpy(dids, gr->global_ids, t->nloc * 4, cudaMemcpyHostToDevice));
        GDX_CUDA(cudaMalloc(&all, uint64_t(t->n) * t->F * 4));
        GDX_CUDA(cudaMalloc(&lab_all, uint64_t(t->n) * 4));
        int rc = gdx_init_uniform(cfg->feature_seed, kFeatTag, 0, 0, t->n, t->F, -0.5, 0.5, all, t->F, nullptr);
        if (!rc) rc = gdx_init_labels(cfg->label_seed, 0, t->n, t->classes, lab_all, nullptr);
        if (!rc && avail) rc = gdx_gather_rows(all, t->F, dids, avail, t->F, t->X.p, t->X.ld, nullptr);
        // labels: 4-byte rows moved bit for bit
        if (!rc) rc = gdx_gather_rows(reinterpret_cast<const float*>(lab_all), 1, dids, static_cast<uint32_t>(t->nloc),
                                      1, reinterpret_cast<float*>(t->labels), 1, nullptr);
        cudaDeviceSynchronize();
        cudaFree(all);
        cudaFree(lab_all);
        if (rc) return rc;
    }
    if (t->nloc)
        if (int rc = gdx_split_bf16(t->X.p, t->X.ld, static_cast<uint32_t>(t->nloc), t->F, t->Xsp.hi, t->Xsp.lo,
                                    t->Xsp.ld, 0, nullptr))
            return rc;
    if (int rc = setup_model(t.get())) return rc;
    GDX_CUDA(cudaDeviceSynchronize());
    *out = t.release();
    return GDX_OK;
}

extern "C" int gdx_trainer_destroy(gdx_trainer* t) {
    if (!t) return GDX_OK;
    cudaSetDevice(t->dev);
    delete t;
    return GDX_OK;
}

extern "C" int gdx_trainer_init_weights(gdx_trainer* t, uint64_t seed, int he_init) {
    GDX_REQUIRE(t, GDX_INPUT, "gdx_trainer_init_weights: null trainer");
    GDX_CUDA(cudaSetDevice(t->dev));
    // consecutive U(-.5,.5) draws of (seed, "weig") in reference order (train.py init_weights)
    uint64_t total = 0;
    const uint32_t nm = t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1;
    for (uint32_t l = 0; l < t->L; ++l) total += uint64_t(nm) * t->dims[l + 1] * t->dims[l];
    double* d = nullptr;
    GDX_CUDA(cudaMalloc(&d, total * 8));
    std::vector<double> h(total);
    uint64_t first = 0;
    for (uint32_t l = 0; l < t->L; ++l)
        for (uint32_t m = 0; m < nm; ++m) {
            const int rc = gdx_init_uniform_f64(seed, kWeigTag, 0, first, t->dims[l + 1], t->dims[l], -0.5, 0.5,
                                                d + first, t->dims[l], nullptr);
            if (rc) {
                cudaFree(d);
                return rc;
            }
            first += uint64_t(t->dims[l + 1]) * t->dims[l];
        }
    cudaError_t e = cudaMemcpy(h.data(), d, total * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    GDX_CUDA(e);
    if (he_init) {  // ModelConfig.init == 'he': times 2 sqrt(6 / fan_in)
        uint64_t o = 0;
        for (uint32_t l = 0; l < t->L; ++l)
            for (uint32_t m = 0; m < nm; ++m) {
                const double s = 2.0 * std::sqrt(6.0 / t->dims[l]);
                for (uint64_t i = 0; i < uint64_t(t->dims[l + 1]) * t->dims[l]; ++i) h[o + i] *= s;
                o += uint64_t(t->dims[l + 1]) * t->dims[l];
            }
    }
    return upload_weights(t, h.data(), total);
}

extern "C" int gdx_trainer_set_weights(gdx_trainer* t, const double* w, uint64_t count) {
    GDX_REQUIRE(t && w, GDX_INPUT, "gdx_trainer_set_weights: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    return upload_weights(t, w, count);
}

extern "C" int gdx_trainer_get_weights(gdx_trainer* t, double* w, uint64_t count) {
    GDX_REQUIRE(t && w, GDX_INPUT, "gdx_trainer_get_weights: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    return read_weights(t, w, count, false);
}

extern "C" int gdx_trainer_get_grads(gdx_trainer* t, double* g, uint64_t count) {
    GDX_REQUIRE(t && g, GDX_INPUT, "gdx_trainer_get_grads: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    return read_weights(t, g, count, true);
}

extern "C" uint64_t gdx_trainer_weight_count(const gdx_trainer* t) {
    if (!t) return 0;
    uint64_t need = 0;
    for (uint32_t l = 0; l < t->L; ++l)
        need += uint64_t(t->dims[l + 1]) * t->dims[l] * (t->cfg.kind == GDX_MODEL_SAGE ? 2 : 1);
    return need;
}

extern "C" uint64_t gdx_trainer_ipc_blob_bytes(const gdx_trainer* t) {
    return t ? 64ull * t->regions.size() : 0;
}

extern "C" int gdx_trainer_ipc_export(gdx_trainer* t, void* blob) {
    GDX_REQUIRE(t && blob, GDX_INPUT, "gdx_trainer_ipc_export: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    for (size_t k = 0; k < t->regions.size(); ++k)
        TR_OK(gdx_ipc_get_handle(t->regions[k], static_cast<char*>(blob) + 64 * k));
    return GDX_OK;
}

extern "C" int gdx_trainer_connect(gdx_trainer* t, const void* blobs) {
    GDX_REQUIRE(t && blobs, GDX_INPUT, "gdx_trainer_connect: null pointer");
    GDX_REQUIRE(!t->connected, GDX_CONTRACT, "gdx_trainer_connect: already connected");
    GDX_CUDA(cudaSetDevice(t->dev));
    if (t->world == 1) {
        t->connected = true;
        return GDX_OK;
    }
    std::vector<unsigned long long*> peer_slot(t->world - 1);
    const uint64_t slot_off = reinterpret_cast<char*>(t->slots) - t->arena;
    const uint64_t blob = 64ull * t->regions.size();
    t->region_delta.assign(t->regions.size(), std::vector<int64_t>(7, 0));
    uint32_t i = 0;
    for (uint32_t r = 0; r < t->world; ++r) {
        if (r == t->rank) continue;
        for (size_t k = 0; k < t->regions.size(); ++k) {
            void* base = nullptr;
            TR_OK(gdx_ipc_open(static_cast<const char*>(blobs) + blob * r + 64 * k, &base));
            t->opened.push_back(base);
            t->region_delta[k][i] = static_cast<char*>(base) - t->regions[k];
            // our arrival slot inside peer r's array
            if (k == 0) peer_slot[i] = reinterpret_cast<unsigned long long*>(static_cast<char*>(base) + slot_off) + t->rank;
        }
        ++i;
    }
    GDX_CUDA(cudaMemcpy(t->peer_slots_dev, peer_slot.data(), peer_slot.size() * sizeof(void*), cudaMemcpyHostToDevice));
    t->connected = true;
    return GDX_OK;
}

extern "C" int gdx_trainer_epoch(gdx_trainer* t, double* loss_out) {
    GDX_REQUIRE(t, GDX_INPUT, "gdx_trainer_epoch: null trainer");
    GDX_CUDA(cudaSetDevice(t->dev));
    TR_OK(run_epoch(t));
    if (loss_out) {
        GDX_CUDA(cudaMemcpyAsync(t->loss_host, t->loss_acc, 8, cudaMemcpyDeviceToHost, t->stream));
        GDX_CUDA(cudaStreamSynchronize(t->stream));
        *loss_out = *t->loss_host / t->loss_count;
    }
    return GDX_OK;
}

extern "C" int gdx_trainer_stage_inputs(gdx_trainer* t, const float* x_host, const int32_t* labels_host) {
    GDX_REQUIRE(t && x_host, GDX_INPUT, "gdx_trainer_stage_inputs: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    const int i = static_cast<int>(t->issued % 2);
    if (!t->stage[0]) {  // both halves of the double buffer at once, before any copy is queued
        for (int j = 0; j < 2; ++j) {
            GDX_CUDA(cudaMalloc(&t->stage[j], std::max<uint64_t>(t->nloc, 1) * t->F * 4));
            GDX_CUDA(cudaMalloc(&t->stage_labels[j], std::max<uint64_t>(t->nloc, 1) * 4));
            GDX_CUDA(cudaEventCreateWithFlags(&t->ready[j], cudaEventDisableTiming));
            GDX_CUDA(cudaEventCreateWithFlags(&t->freed[j], cudaEventDisableTiming));
        }
    }
    if (t->issued >= 2) GDX_CUDA(cudaStreamWaitEvent(t->copy, t->freed[i], 0));
    // ONE contiguous DMA of the host block [nloc, F] (the PCIe rate from pinned memory)
    GDX_CUDA(cudaMemcpyAsync(t->stage[i], x_host, t->nloc * t->F * 4, cudaMemcpyHostToDevice, t->copy));
    if (labels_host)
        GDX_CUDA(cudaMemcpyAsync(t->stage_labels[i], labels_host, t->nloc * 4, cudaMemcpyHostToDevice, t->copy));
    t->staged_labels[i] = labels_host != nullptr;
    GDX_CUDA(cudaEventRecord(t->ready[i], t->copy));
    t->issued++;
    return GDX_OK;
}

extern "C" int gdx_trainer_step_staged(gdx_trainer* t, int with_labels, double* loss_out) {
    GDX_REQUIRE(t, GDX_INPUT, "gdx_trainer_step_staged: null trainer");
    GDX_REQUIRE(t->consumed < t->issued, GDX_CONTRACT, "gdx_trainer_step_staged: nothing staged");
    GDX_CUDA(cudaSetDevice(t->dev));
    const int i = static_cast<int>(t->consumed % 2);
    GDX_REQUIRE(!with_labels || t->staged_labels[i], GDX_CONTRACT,
                "gdx_trainer_step_staged: labels requested but none were staged");
    GDX_CUDA(cudaStreamWaitEvent(t->stream, t->ready[i], 0));
    if (t->nloc)
        TR_OK(gdx_split_bf16(t->stage[i], t->F, static_cast<uint32_t>(t->nloc), t->F, t->Xsp.hi, t->Xsp.lo, t->Xsp.ld, 0,
                             reinterpret_cast<gdx_stream>(t->stream)));
    if (with_labels)
        GDX_CUDA(cudaMemcpyAsync(t->labels, t->stage_labels[i], t->nloc * 4, cudaMemcpyDeviceToDevice, t->stream));
    GDX_CUDA(cudaEventRecord(t->freed[i], t->stream));
    t->consumed++;
    return gdx_trainer_epoch(t, loss_out);
}

extern "C" void* gdx_trainer_stream(gdx_trainer* t) { return t ? static_cast<void*>(t->stream) : nullptr; }

extern "C" int gdx_trainer_info(const gdx_trainer* t, uint64_t* out, uint32_t count) {
    GDX_REQUIRE(t && out, GDX_INPUT, "gdx_trainer_info: null pointer");
    const uint64_t v[] = {t->nloc, t->nnz, t->lo, t->nfull, t->loss_rows, static_cast<uint64_t>(t->loss_count),
                          t->exec ? 1ull : 0ull, (!t->layers.empty() && t->layers.back().agg_first) ? 1ull : 0ull,
                          t->nnz_src, t->bins ? t->bins->n_heavy : 0ull};
    for (uint32_t i = 0; i < count && i < sizeof(v) / sizeof(v[0]); ++i) out[i] = v[i];
    return GDX_OK;
}

extern "C" int gdx_trainer_profile_gemm(gdx_trainer* t, double* ms, uint64_t* launches, double* flops) {
    GDX_REQUIRE(t && ms && launches && flops, GDX_INPUT, "gdx_trainer_profile_gemm: null pointer");
    GDX_CUDA(cudaSetDevice(t->dev));
    GDX_CUDA(cudaStreamSynchronize(t->stream));
    double tot = 0, fl = 0;
    for (size_t i = 0; i < t->gemm_events.size(); ++i) {
        float x = 0;
        GDX_CUDA(cudaEventElapsedTime(&x, t->gemm_events[i].first, t->gemm_events[i].second));
        tot += x;
        fl += t->gemm_flops[i];
    }
    *ms = tot;
    *launches = t->gemm_events.size();
    *flops = fl;
    return GDX_OK;
}

extern "C" int gdx_trainer_profile(gdx_trainer* t, int on, double* ms, uint64_t* launches, double* bytes) {
    GDX_REQUIRE(t, GDX_INPUT, "gdx_trainer_profile: null trainer");
    GDX_CUDA(cudaSetDevice(t->dev));
    if (ms || launches || bytes) {
        GDX_CUDA(cudaStreamSynchronize(t->stream));
        double tot = 0, by = 0;
        for (size_t i = 0; i < t->prof_events.size(); ++i) {
            float x = 0;
            GDX_CUDA(cudaEventElapsedTime(&x, t->prof_events[i].first, t->prof_events[i].second));
            tot += x;
            by += t->prof_bytes[i];
        }
        if (ms) *ms = tot;
        if (launches) *launches = t->prof_events.size();
        if (bytes) *bytes = by;
    }
    for (auto& e : t->prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    t->prof_events.clear();
    t->prof_bytes.clear();
    for (auto& e : t->gemm_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    t->gemm_events.clear();
    t->gemm_flops.clear();
    t->profile = on != 0;
    return GDX_OK;
}
