// duhl.cu -- host runtime and C ABI of the B200-native DuHL hot path.
//
// Unit A (PAPER.md Assumption 1) = pinned host DRAM holding all of A,
// mapped into the device address space; unit B = HBM holding the working set
// A_[P] in a slot pool sized by cfg.hbm_budget_bytes.  Selected columns are
// staged with cudaMemcpyAsync on a copy stream (Alg. 2 l.4); the compute stream
// waits on an event before the SCD epoch.  See include/duhl.h for the contract.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library dlopen()s libnccl.so.2 at duhl_comm_init

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/duhl.h"
#include "device.cuh"
#include "unit_a_host.h"
#include "kernels.h"

using namespace duhl;

namespace {
constexpr int kGapTileRows = 4096;
constexpr int kStageCtas = 16;  // k_stage_gather CTAs (2 per SM the SCD grid leaves): 51.4 GB/s alone (stage2.cu)
constexpr unsigned kCeToken = 0x80000000u;  // wait token of a column the copy engine stages
constexpr int kCeCounter = 16;              // its progress counter (sequence numbers)
constexpr double kStageCeShare = 0.3;       // share of a gather round's columns on the copy engine
constexpr size_t kProgressBytes = 17 * 128;  // staging counters, one 128-byte line each (kProgressStride):
                                             // 16 gather CTAs + the copy-engine share (kCeCounter)
inline int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }
}  // namespace

// ---- NCCL, resolved at run time (shares torch's already-loaded libnccl.so.2 if present)
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};
static NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
            api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
            api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
            api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
            api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
            api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy;
        }
    }
    return api.ok ? &api : nullptr;
}

// In-process group (duhl_group_create): contexts driven by threads of one process
// reduce through host memory in rank order (deterministic; no NCCL).
struct duhl_group {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<std::vector<double>> slot;  // [n] one buffer per rank
    // generation barrier; false after timeout_s seconds without all ranks
    bool barrier(double timeout_s) {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g; });
        if (!ok) --arrived;
        return ok;
    }
};

struct duhl_ctx {
    // ---- problem (this rank's shard: columns [col_offset, col_offset + n) of n_glob)
    int model = 0;
    int64_t d = 0, d4 = 0, n = 0, n_glob = 0, col_offset = 0;
    // ---- multi-GPU (CoCoA-style aggregation)
    ncclComm_t comm = nullptr;
    duhl_group* group = nullptr;  // in-process group instead of NCCL (duhl_comm_init_group)
    duhl_trace_cb trace_cb = nullptr;  // duhl_solve per-round callback
    void* trace_user = nullptr;
    int nranks = 1, rank = 0;
    double *d_dv = nullptr, *d_aold = nullptr, *d_ls = nullptr;  // dv, alpha_P at round start, line search
    double lambda = 0, B = 0;
    duhl_config cfg{};
    std::string err;
    int dev = 0, nsm = 0, unit_a_ctas = 0;
    bool pipe = false;  // SCD epoch runs k_scd_pipe (else k_scd_gram / k_scd_ser); see choose_scd_shape
    bool ser = false;   // k_scd_ser instead of k_scd_gram (cfg.scd_kernel 0 / 3; 1 = k_scd_gram)
    bool tpa = false;   // cfg.scd_async: asynchronous k_scd_tpa epoch (W clusters of tpa_C CTAs)
    int tpa_C = 1;
    int64_t tpa_Rc = 0;
    bool tpa_v0s = false;
    float* d_vf = nullptr;          // fp32 shadow of the shared vector (asynchronous epoch)
    double *d_v0t = nullptr, *d_a0t = nullptr;  // v~ and alpha_P at epoch start (exact resync)
    double* d_u0 = nullptr;                     // [n] a_j^T v~0 for j in P (asynchronous epoch)
    cudaStream_t st = nullptr, cst = nullptr, rst = nullptr;  // compute, copy (H2D), unit-A refresh
    cudaStream_t cst2 = nullptr;     // copy-engine share of a gather round's staging
    cudaEvent_t ev_copy2 = nullptr;
    cudaEvent_t ev_copy = nullptr, ev_snap = nullptr, ev_ref = nullptr;
    // ---- unit A: pinned host store
    float* h_store = nullptr;
    bool own_store = false, registered = false;
    // sparse (CSC) problems: the matrix lives in HBM; no slot pool, no staging
    bool csc = false;
    int64_t nnz = 0;
    int64_t* d_colptr = nullptr;
    int* d_rows = nullptr;
    float* d_vals = nullptr;
    std::vector<int64_t> h_colptr;  // host copy of col_ptr (algorithmic byte counts)
    double csc_pass_bytes = 0.0;    // algorithmic bytes of one SCD pass over the current order
    int csc_warps = 0;              // concurrent coordinates of the asynchronous CSC epoch
    void* d_topm_work = nullptr;    // scratch of the multi-CTA top-m
    // resident problems (no slot pool) keep P on the device: the host copy and inP are
    // refreshed only when an ABI call needs them
    int* d_stamp = nullptr;         // [n] id of the select that last took column j
    unsigned long long* d_rsel = nullptr;  // [2] swaps, nnz over P
    double* d_rho = nullptr;               // [2] sum of z over P, over all columns (round record rho)
    double* d_est = nullptr;               // [4] gap estimate: sum z over P, over the sample, counts
    int64_t* d_smp = nullptr;              // [n] this round's refreshed columns outside P (the sample)
    int sel_id = 0;
    int64_t m_cur = 0;              // |P|
    bool P_host_valid = true;
    int64_t ld_host = 0;
    const float* h_alias = nullptr;  // device address of h_store
    // ---- unit B: HBM slot pool
    float* pool = nullptr;
    int64_t S = 0, ld_dev = 0, m_cfg = 0;
    std::vector<int> col_slot, slot_col;
    int* d_col_slot = nullptr;
    // ---- state
    double *d_alpha = nullptr, *d_vt = nullptr, *d_b = nullptr, *d_y = nullptr;
    double *d_norms = nullptr, *d_z = nullptr;
    // ---- working set
    std::vector<int64_t> P;      // current working set, ascending
    std::vector<char> inP;       // [n]
    int64_t *d_P = nullptr, *d_order_j = nullptr, *d_cols = nullptr, *d_chg_cols = nullptr;
    int *d_P_slot = nullptr, *d_order_slot = nullptr, *d_chg_slots = nullptr;
    double* d_vsnap = nullptr;   // round-start snapshot of the shared vector (unit-A refresh)
    // ---- gap scratch
    double *d_s_acc = nullptr, *d_gap_out = nullptr, *d_s_out = nullptr, *d_sums = nullptr;
    int* d_flag = nullptr;
    // ---- SCD
    double* d_red = nullptr;
    unsigned* d_bar = nullptr;
    int W = 0, R = 0, G = 0, NB = 2;
    // ---- misc
    int64_t launches = 0, h2d_bytes = 0, zc_bytes = 0, updates = 0, cursor = 0, d2h_bytes = 0;
    // ---- profiling (cfg.profile): CUDA-event pairs per launch, harvested at sync points
    struct Timed { cudaEvent_t a, b; int kind; double bytes; };
    std::vector<Timed> pending;
    std::vector<cudaEvent_t> event_pool;
    int64_t st_launch[7] = {0, 0, 0, 0, 0, 0, 0};
    double st_ms[7] = {0, 0, 0, 0, 0, 0, 0}, st_bytes[7] = {0, 0, 0, 0, 0, 0, 0};
    double* d_s_acc2 = nullptr;  // partial-dot accumulator of the concurrent refresh pass
    // ---- unit A on host threads (cfg.unit_a_host_threads): a_i^T v~ for part of the refresh
    HostUnitA* hua = nullptr;
    double* h_vt = nullptr;        // pinned [d4]: round-start v~ for the host threads
    double* h_hs = nullptr;        // pinned [n]: their dots
    double* h_hnorm = nullptr;     // pinned [n]: column norms of create's host ingest share
    int64_t* h_ref_idx = nullptr;  // a round's refresh columns (async upload, no realloc): pinned [n],
    int64_t* h_ref_smp = nullptr;  // and the gap-estimate sample, allocated at the first large refresh
    std::vector<int64_t> ref_idx_v, ref_smp_v;  // small refreshes: plain heap buffers
    int64_t* h_hcols = nullptr;    // pinned [n]: their columns
    double* d_hs = nullptr;        // [n] dots uploaded for k_gap_finalize
    int64_t* d_hcols = nullptr;    // [n]
    cudaEvent_t ev_hvt = nullptr, ev_g0 = nullptr, ev_g1 = nullptr, ev_c1 = nullptr;  // v~ on the host;
                                   // GPU refresh span; end of the round's staging copies
    double cert_share = 0.4;       // share of a certificate's non-resident columns on the host
    double hua_share = 0.7;        // current share of the non-resident refresh columns on the host
    int64_t hua_cols = 0;          // host-refreshed columns (all rounds)
    // ---- staging overlapped with the SCD epoch
    typedef int (*WriteValue32)(cudaStream_t, unsigned long long, unsigned, unsigned);
    WriteValue32 write_value = nullptr;  // cuStreamWriteValue32 via cudaGetDriverEntryPoint
    bool overlap = false;  // this round's copies overlap the epoch (progress counter); else copies first
    int stage_ctas = 0;    // > 0: this round's copies are a k_stage_gather launch of that many CTAs
    int64_t* h_plan_cols = nullptr;  // pinned gather plan (columns, slots), uploaded on the copy stream
    int* h_plan_slots = nullptr;
    int64_t* d_plan_cols = nullptr;
    int* d_plan_slots = nullptr;
    cudaEvent_t ev_plan = nullptr;   // the last plan upload has read the pinned plan
    unsigned* d_progress = nullptr;      // last landed staging copy (sequence number)
    unsigned batch_seq = 0;
    std::vector<unsigned> slot_batch;    // [S] sequence number of the copy that filled a slot
    unsigned *d_P_batch = nullptr, *d_order_batch = nullptr;
    double *d_order_a = nullptr, *d_order_inv = nullptr, *d_order_y = nullptr;
    std::vector<int64_t> pend_cols;      // staged columns not yet in the device table
    std::vector<int> pend_slots;
    struct Copy { int64_t col; int slot; unsigned seq; };  // gather rounds: seq = wait token
    std::vector<Copy> copy_plan;         // planned, not yet enqueued staging copies
};

// ------------------------------------------------------------------------- profiling
static cudaEvent_t pool_event(duhl_ctx* ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
struct ProfScope {  // brackets one launch (or copy batch) with events on `st`
    duhl_ctx* ctx;
    cudaStream_t st;
    int kind;
    double bytes;
    cudaEvent_t a = nullptr;
    ProfScope(duhl_ctx* c, cudaStream_t s, int k, double by) : ctx(c), st(s), kind(k), bytes(by) {
        if (ctx->cfg.profile) {
            a = pool_event(ctx);
            cudaEventRecord(a, st);
        }
    }
    void end() {
        if (a) {
            cudaEvent_t b = pool_event(ctx);
            cudaEventRecord(b, st);
            ctx->pending.push_back({a, b, kind, bytes});
            a = nullptr;
        }
    }
    ~ProfScope() { end(); }
};
static void harvest(duhl_ctx* ctx) {  // call after the streams are synchronized
    for (auto& t : ctx->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
            ctx->st_launch[t.kind] += 1;
            ctx->st_ms[t.kind] += ms;
            ctx->st_bytes[t.kind] += t.bytes;
        }
        ctx->event_pool.push_back(t.a);
        ctx->event_pool.push_back(t.b);
    }
    ctx->pending.clear();
    cudaGetLastError();
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
            return DUHL_E_CUDA;                                                       \
        }                                                                             \
    } while (0)

#define TRY(call)                          \
    do {                                   \
        duhl_status s_ = (call);           \
        if (s_ != DUHL_OK) return s_;      \
    } while (0)

// Device -> host read-back on stream st, counted (duhl_get_counters: d2h_bytes).
static cudaError_t d2h_copy(duhl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);

static duhl_status fail(duhl_ctx* ctx, duhl_status s, const std::string& msg) {
    ctx->err = msg;
    return s;
}

static cudaError_t d2h_copy(duhl_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    ctx->d2h_bytes += (int64_t)bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
}

// ------------------------------------------------------------------------- helpers
static ColSrc colsrc(const duhl_ctx* ctx) {
    ColSrc s;
    s.pool = ctx->pool;
    s.ld_dev = ctx->ld_dev;
    s.host = ctx->h_alias;
    s.ld_host = ctx->ld_host;
    s.col_slot = ctx->d_col_slot;
    return s;
}

static CscMat cscmat(const duhl_ctx* ctx) { return CscMat{ctx->d_colptr, ctx->d_rows, ctx->d_vals}; }

// ridge: the SCD kernels take 1/(||a_j||^2 + lambda d) per position (k_perm_order)
// (elastic net: 1/(||a_j||^2 + lambda eta d))
static double ridge_ld(const duhl_ctx* ctx) {
    return ctx->model == DUHL_RIDGE ? ctx->lambda * (double)ctx->d
         : ctx->model == DUHL_ELASTIC_NET ? ctx->lambda * ctx->cfg.eta * (double)ctx->d : 0.0;
}

static double wscale(const duhl_ctx* ctx) {
    return ctx->model != DUHL_SVM_DUAL ? 1.0 : 1.0 / (ctx->lambda * (double)ctx->n_glob);
}

// In-process group: copy out, barrier, every rank sums the slots in rank order (so
// all ranks hold bit-identical results, as the oracle's shard-order sum), barrier,
// copy back.  Bounded waits: a rank that never arrives fails the call.
static duhl_status group_allreduce(duhl_ctx* ctx, double* buf, size_t count, bool is_max) {
    duhl_group* g = ctx->group;
    std::vector<double>& mine = g->slot[ctx->rank];
    mine.resize(count);
    if (d2h_copy(ctx, mine.data(), buf, count * sizeof(double), ctx->st) != cudaSuccess ||
        cudaStreamSynchronize(ctx->st) != cudaSuccess)
        return fail(ctx, DUHL_E_CUDA, "group allreduce: device -> host copy failed");
    if (!g->barrier(600.0)) return fail(ctx, DUHL_E_NCCL, "group allreduce: a rank did not arrive");
    std::vector<double> out(g->slot[0]);
    for (int r = 1; r < g->n; ++r) {
        const std::vector<double>& x = g->slot[r];
        if (x.size() != count) return fail(ctx, DUHL_E_NCCL, "group allreduce: ranks disagree on the count");
        for (size_t i = 0; i < count; ++i) out[i] = is_max ? std::max(out[i], x[i]) : out[i] + x[i];
    }
    if (!g->barrier(600.0)) return fail(ctx, DUHL_E_NCCL, "group allreduce: a rank did not arrive");
    if (cudaMemcpyAsync(buf, out.data(), count * sizeof(double), cudaMemcpyHostToDevice, ctx->st) != cudaSuccess ||
        cudaStreamSynchronize(ctx->st) != cudaSuccess)
        return fail(ctx, DUHL_E_CUDA, "group allreduce: host -> device copy failed");
    return DUHL_OK;
}

// In-place sum (or max) allreduce over the group on the compute stream; no-op without a
// communicator (a 1-rank NCCL communicator still runs the collective).
static duhl_status allreduce(duhl_ctx* ctx, double* buf, size_t count, ncclRedOp_t op = ncclSum) {
    if (ctx->group) return group_allreduce(ctx, buf, count, op == ncclMax);
    if (!ctx->comm) return DUHL_OK;
    ncclResult_t r = nccl_api()->allReduce(buf, buf, count, ncclDouble, op, ctx->comm, ctx->st);
    if (r != ncclSuccess) return fail(ctx, DUHL_E_NCCL, std::string("ncclAllReduce: ") + nccl_api()->getErrorString(r));
    return DUHL_OK;
}

static GapParams gap_params(duhl_ctx* ctx, const int64_t* d_cols, int64_t k) {
    GapParams p{};
    p.model = ctx->model;
    p.d = ctx->d;
    p.d4 = ctx->d4;
    p.n = ctx->n_glob;  // gap formulas use the global n (SVM 1/n, w = v/(lambda n))
    p.src = colsrc(ctx);
    p.cols = d_cols;
    p.k = k;
    p.vt = ctx->d_vt;
    p.wscale = wscale(ctx);
    p.alpha = ctx->d_alpha;
    p.y = ctx->d_y;
    p.lambda = ctx->lambda;
    p.B = ctx->B;
    p.eta = ctx->cfg.eta;
    p.s_acc = ctx->d_s_acc;
    p.z = ctx->d_z;
    p.flag = ctx->d_flag;
    return p;
}

static duhl_status check_flag(duhl_ctx* ctx, const char* where) {
    int fl[2] = {0, 0};
    CK(d2h_copy(ctx, fl, ctx->d_flag, 2 * sizeof(int), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    const int flag = fl[0];
    if (fl[1]) {
        CK(cudaMemsetAsync(ctx->d_flag + 1, 0, sizeof(int), ctx->st));
        // bits: 1 staging copy, 2 grid barrier, 4 stage-free, 8 stage-data, 16 delta (SCD kernel waits)
        std::string what;
        const char* nm[5] = {"staging copy", "grid barrier", "stage-free", "stage-data", "delta"};
        for (int k = 0; k < 5; ++k)
            if (fl[1] & (1 << k)) what += std::string(what.empty() ? "" : ", ") + nm[k];
        return fail(ctx, DUHL_E_CUDA, std::string(where) + ": " + what + " wait timed out");
    }
    if (flag) {
        CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->st));
        return fail(ctx, DUHL_E_NUMERIC,
                    std::string(where) + (flag & 2 ? ": non-finite gap/state" : ": negative duality gap"));
    }
    return DUHL_OK;
}

// gap pass over d_cols[0..k) (nullptr = all n), writing z; optional device outputs
static duhl_status run_gaps(duhl_ctx* ctx, const int64_t* d_cols, int64_t k, double* gap_out,
                            double* s_out, double* sums, bool write_z = true,
                            const double* vt_override = nullptr, cudaStream_t stream = nullptr,
                            double* s_acc = nullptr, int tile_rows = kGapTileRows, int max_ctas = 0) {
    cudaStream_t sx = stream ? stream : ctx->st;
    GapParams p = gap_params(ctx, d_cols, d_cols ? k : ctx->n);
    if (vt_override) p.vt = vt_override;
    p.gap_out = gap_out;
    p.s_out = s_out;
    p.sums = sums;
    if (!write_z) p.z = nullptr;
    if (s_acc) p.s_acc = s_acc;
    const int64_t tiles = (ctx->d4 + tile_rows - 1) / tile_rows;
    // algorithmic bytes: dense 4 d4 + 24 per column (+ w tiles); CSC 8 per nonzero + 24 per column
    const double by = !ctx->csc ? (double)p.k * (4.0 * ctx->d4 + 24.0) + 8.0 * ctx->d4 * tiles
                      : !d_cols ? 8.0 * (double)ctx->nnz + 24.0 * (double)ctx->n
                      : d_cols == ctx->d_P ? ctx->csc_pass_bytes
                      : (double)p.k * (8.0 * (double)ctx->nnz / (double)ctx->n + 24.0);
    ProfScope ps(ctx, sx, stream ? 4 : 1, by);
    if (ctx->csc) CK(launch_csc_gap(p, cscmat(ctx), max_ctas, sx, &ctx->launches));
    else CK(launch_gap_pass(p, tile_rows, sx, &ctx->launches, max_ctas));
    return DUHL_OK;
}

static duhl_status upload_slots_changes(duhl_ctx* ctx, const std::vector<int64_t>& cols,
                                        const std::vector<int>& slots) {
    if (cols.empty()) return DUHL_OK;
    CK(cudaMemcpyAsync(ctx->d_chg_cols, cols.data(), cols.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_chg_slots, slots.data(), slots.size() * sizeof(int),
                       cudaMemcpyHostToDevice, ctx->st));
    CK(launch_set_slots(ctx->d_col_slot, ctx->d_chg_cols, ctx->d_chg_slots, (int64_t)cols.size(),
                        ctx->st, &ctx->launches));
    // the uploads read pageable host vectors: make them complete before they go away
    CK(cudaStreamSynchronize(ctx->st));
    return DUHL_OK;
}

// Host copy of the device pass permutation (kernels.cu feistel_index): the
// position map of pass 0 orders the H2D staging so columns land in the order
// the SCD kernel consumes them.
static int64_t feistel_host(uint64_t key, int h, int64_t m, int64_t t) {
    const uint64_t mask = (1ull << h) - 1;
    uint64_t x = (uint64_t)t;
    do {
        uint64_t L = x >> h, R = x & mask;
        for (int r = 0; r < 8; ++r) {
            uint64_t F = mix64(key ^ ((uint64_t)r << 56) ^ R) & mask;
            uint64_t nl = R;
            R = L ^ F;
            L = nl;
        }
        x = (L << h) | R;
    } while (x >= (uint64_t)m);
    return (int64_t)x;
}

// Make the device column table point at the columns staged by the last
// stage_working_set (their copies must have landed: the compute stream waits
// on the copy stream first).
static duhl_status issue_staging(duhl_ctx* ctx);
static duhl_status finalize_staging(duhl_ctx* ctx) {
    TRY(issue_staging(ctx));
    if (ctx->pend_cols.empty()) return DUHL_OK;
    CK(cudaStreamWaitEvent(ctx->st, ctx->ev_copy, 0));
    std::vector<int64_t> cols;
    std::vector<int> slots;
    cols.swap(ctx->pend_cols);
    slots.swap(ctx->pend_slots);
    return upload_slots_changes(ctx, cols, slots);
}

// Enqueue the planned host -> HBM copies on the copy stream, each followed by a
// stream write of its sequence number to d_progress (the SCD kernel waits on
// it).  Called right after the SCD launch so the host-side enqueue overlaps the
// epoch.  On a failure the counter is forced to its final value so a waiting
// kernel can drain, and the error is reported.
static duhl_status issue_staging(duhl_ctx* ctx) {
    if (ctx->copy_plan.empty()) return DUHL_OK;
    duhl_status rc = DUHL_OK;
    if (ctx->stage_ctas > 0) {  // light round: one gather launch (k_stage_gather), entries in plan order
        const size_t np = ctx->copy_plan.size();
        const size_t col_bytes = (size_t)ctx->ld_dev * sizeof(float);
        ProfScope ps(ctx, ctx->cst, 3, (double)(np * col_bytes));
        cudaEventSynchronize(ctx->ev_plan);  // the previous upload has read the pinned plan
        size_t ng = 0;
        bool any_ce = false;
        for (size_t q = 0; q < np; ++q) {
            const auto& c = ctx->copy_plan[q];
            if (c.seq & kCeToken) {  // the copy engine's share, on its own stream: one copy + one
                                     // progress write per column (the PCIe link takes both paths)
                any_ce = true;
                if (cudaMemcpyAsync(ctx->pool + (int64_t)c.slot * ctx->ld_dev, ctx->h_store + c.col * ctx->ld_host,
                                    col_bytes, cudaMemcpyHostToDevice, ctx->cst2) != cudaSuccess ||
                    ctx->write_value(ctx->cst2,
                                     (unsigned long long)(uintptr_t)(ctx->d_progress + (size_t)kCeCounter * kProgressStride),
                                     c.seq & ~kCeToken, 0) != 0) {
                    rc = fail(ctx, DUHL_E_CUDA, "staging copy (copy-engine share) failed");
                    break;
                }
                continue;
            }
            ctx->h_plan_cols[ng] = c.col;
            ctx->h_plan_slots[ng] = c.slot;
            ++ng;
        }
        if (rc == DUHL_OK &&
            (cudaMemcpyAsync(ctx->d_plan_cols, ctx->h_plan_cols, ng * sizeof(int64_t), cudaMemcpyHostToDevice,
                             ctx->cst) != cudaSuccess ||
             cudaMemcpyAsync(ctx->d_plan_slots, ctx->h_plan_slots, ng * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->cst) != cudaSuccess ||
             cudaEventRecord(ctx->ev_plan, ctx->cst) != cudaSuccess ||
             launch_stage_gather(ctx->h_alias, ctx->ld_host, ctx->pool, ctx->ld_dev, ctx->ld_dev, ctx->d_plan_cols,
                                 ctx->d_plan_slots, (int64_t)ng, ctx->d_progress, ctx->stage_ctas, ctx->cst,
                                 &ctx->launches) != cudaSuccess))
            rc = fail(ctx, DUHL_E_CUDA, "staging gather launch failed");
        if (rc != DUHL_OK) {  // let a waiting epoch drain: every token reads as landed
            std::vector<unsigned> big(kProgressBytes / sizeof(unsigned), 0x7fffffffu);
            cudaMemcpy(ctx->d_progress, big.data(), kProgressBytes, cudaMemcpyHostToDevice);
        }
        if (any_ce) {
            cudaEventRecord(ctx->ev_copy2, ctx->cst2);
            cudaStreamWaitEvent(ctx->cst, ctx->ev_copy2, 0);
        }
        ps.end();
        ctx->h2d_bytes += (int64_t)(np * col_bytes);
        ctx->copy_plan.clear();
        cudaEventRecord(ctx->ev_copy, ctx->cst);
        if (!ctx->overlap) cudaStreamWaitEvent(ctx->st, ctx->ev_copy, 0);
        return rc;
    }
    {
        ProfScope ps(ctx, ctx->cst, 3, 0.0);
        const size_t col_bytes = (size_t)ctx->ld_dev * sizeof(float);
        const size_t np = ctx->copy_plan.size();
        for (size_t q = 0; q < np;) {
            // maximal run of consecutive columns into consecutive slots with one sequence number
            const auto& c0 = ctx->copy_plan[q];
            size_t e = q + 1;
            while (e < np && ctx->copy_plan[e].seq == c0.seq && ctx->copy_plan[e].col == c0.col + (int64_t)(e - q) &&
                   ctx->copy_plan[e].slot == c0.slot + (int)(e - q) && ctx->ld_host == ctx->ld_dev)
                ++e;
            const size_t bytes = (e - q) * col_bytes;
            if (cudaMemcpyAsync(ctx->pool + (int64_t)c0.slot * ctx->ld_dev, ctx->h_store + c0.col * ctx->ld_host,
                                bytes, cudaMemcpyHostToDevice, ctx->cst) != cudaSuccess) {
                rc = fail(ctx, DUHL_E_CUDA, "staging cudaMemcpyAsync failed");
                break;
            }
            ctx->h2d_bytes += (int64_t)bytes;
            ps.bytes += (double)bytes;
            const bool last_of_seq = e == np || ctx->copy_plan[e].seq != c0.seq;
            if (ctx->overlap && last_of_seq &&
                ctx->write_value(ctx->cst, (unsigned long long)(uintptr_t)ctx->d_progress, c0.seq, 0) != 0) {
                rc = fail(ctx, DUHL_E_CUDA, "cuStreamWriteValue32 failed");
                break;
            }
            q = e;
        }
    }
    if (std::getenv("DUHL_STAGE_TRACE"))
        std::fprintf(stderr, "issue_staging: %zu copies, seq %u..%u, batch_seq %u\n", ctx->copy_plan.size(),
                     ctx->copy_plan.empty() ? 0u : ctx->copy_plan.front().seq,
                     ctx->copy_plan.empty() ? 0u : ctx->copy_plan.back().seq, ctx->batch_seq);
    if (rc != DUHL_OK) {
        unsigned last = ctx->batch_seq;
        cudaMemcpy(ctx->d_progress, &last, sizeof(unsigned), cudaMemcpyHostToDevice);
    }
    ctx->copy_plan.clear();
    cudaEventRecord(ctx->ev_copy, ctx->cst);
    if (!ctx->overlap) cudaStreamWaitEvent(ctx->st, ctx->ev_copy, 0);
    return rc;
}

// Stage P (ascending) into the slot pool (Alg. 2 l.4): evict non-members (the
// device table drops them at once, so concurrent gap passes read them from
// host memory), then plan one host -> HBM copy per new column in the order
// pass 0 of round `round` visits it (issue_staging enqueues them after the SCD
// launch; the kernel waits on the copy-progress counter per block, so staging
// overlaps the epoch).  New columns enter the device table after the epoch
// (finalize_staging).
// Resident problem: d_P holds the new working set (m entries); slots/batches,
// swap count and the CSC pass bytes come from one device pass (no O(n) host work).
static duhl_status resident_commit(duhl_ctx* ctx, int64_t m, int64_t* swaps) {
    ++ctx->sel_id;
    CK(launch_resident_select(ctx->d_P, m, ctx->d_stamp, ctx->sel_id, ctx->d_P_slot, ctx->d_P_batch,
                              ctx->csc ? ctx->d_colptr : nullptr, ctx->d_rsel, ctx->st, &ctx->launches));
    unsigned long long h[2] = {0, 0};
    CK(d2h_copy(ctx, h, ctx->d_rsel, sizeof(h), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->m_cur = m;
    if (ctx->csc) ctx->csc_pass_bytes = 8.0 * (double)h[1] + 24.0 * (double)m;
    if (swaps) *swaps = (int64_t)h[0];
    return DUHL_OK;
}

// The host copy of P (and inP) for the calls that need it (explicit-order epochs, P_out).
static duhl_status ensure_host_P(duhl_ctx* ctx) {
    if (ctx->P_host_valid) return DUHL_OK;
    ctx->P.resize(ctx->m_cur);
    CK(d2h_copy(ctx, ctx->P.data(), ctx->d_P, ctx->m_cur * sizeof(int64_t), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    std::fill(ctx->inP.begin(), ctx->inP.end(), 0);
    for (int64_t j : ctx->P) ctx->inP[j] = 1;
    ctx->P_host_valid = true;
    return DUHL_OK;
}

constexpr int64_t kPinnedRefreshCols = 65536;  // refresh lists at least this long live in pinned memory
constexpr int64_t kHeavyRunCols = 16;  // mean index-run length that sends a heavy round to the copy engine
constexpr size_t kStageCeMinBytes = 512 * 1024;  // shorter columns: no copy-engine share in gather rounds

static duhl_status stage_working_set(duhl_ctx* ctx, const std::vector<int64_t>& P, int64_t round,
                                     int64_t* swaps) {
    TRY(finalize_staging(ctx));
    const int64_t m = (int64_t)P.size();
    std::vector<char> in_new(ctx->n, 0);
    for (int64_t j : P) in_new[j] = 1;
    int64_t nsw = 0;
    std::vector<int64_t> chg_cols;
    std::vector<int> chg_slots;
    if (ctx->cfg.hbm_budget_bytes != 0) {
        std::vector<int> free_slots;
        for (int64_t s = 0; s < ctx->S; ++s) {
            int c = ctx->slot_col[s];
            if (c < 0 || !in_new[c]) {
                if (c >= 0) {
                    ctx->col_slot[c] = -1;
                    chg_cols.push_back(c);
                    chg_slots.push_back(-1);
                }
                ctx->slot_col[s] = -1;
                free_slots.push_back((int)s);
            }
        }
        // new columns in pass-0 visiting order when the epoch consumes them as they land
        // (overlap); otherwise the copies complete before the epoch and index order will do
        // (saves m host Feistel evaluations per round: 1.5 ms at C3's m = 50,176)
        std::vector<int64_t> news;
        news.reserve(m);
        if (ctx->overlap) {
            int h = 1;
            while ((1ll << (2 * h)) < m) ++h;
            const uint64_t key = mix64(mix64(mix64(ctx->cfg.seed) ^ (uint64_t)round) ^ 0ull);
            for (int64_t t = 0; t < m; ++t) {
                const int64_t j = P[feistel_host(key, h, m, t)];
                if (ctx->col_slot[j] < 0) news.push_back(j);
            }
        } else {
            for (int64_t j : P)
                if (ctx->col_slot[j] < 0) news.push_back(j);
        }
        if ((int64_t)news.size() > (int64_t)free_slots.size())
            return fail(ctx, DUHL_E_INVALID, "working set exceeds the HBM slot pool");
        // plan the copies now (slot, sequence number); issue_staging enqueues them.
        // Light rounds: one copy per column in pass-0 order, a progress write every
        // 4 columns, so the epoch starts at once.  Heavy rounds (more than half of P
        // new): columns in index order with consecutive slots, so runs coalesce into
        // large copies at full PCIe rate, and one progress write at the end.
        const bool heavy = (int64_t)news.size() * 2 > m;
        // A heavy round goes to the copy engine in coalesced runs only when its new columns form
        // long index runs (C4's first rounds: whole index blocks, ~51 GB/s).  Scattered columns
        // (C3's Lasso selections: one 160-KB copy each, ~22 GB/s) take the gather kernel like a
        // light round.
        bool heavy_ce = false;
        if (heavy) {
            std::vector<int64_t> srt(news);
            std::sort(srt.begin(), srt.end());
            int64_t runs = srt.empty() ? 0 : 1;
            for (size_t q = 1; q < srt.size(); ++q) runs += srt[q] != srt[q - 1] + 1;
            static const int64_t run_cols = std::getenv("DUHL_HEAVY_RUN_COLS")  // developer A/B
                                                ? std::atoll(std::getenv("DUHL_HEAVY_RUN_COLS")) : kHeavyRunCols;
            heavy_ce = runs == 0 || (int64_t)srt.size() >= run_cols * runs || ctx->unit_a_ctas <= 0;
            if (heavy_ce) news.swap(srt);
        }
        // every earlier copy has landed before this round's epoch (the compute stream waited on
        // ev_copy): kept slots need no wait
        std::fill(ctx->slot_batch.begin(), ctx->slot_batch.end(), 0u);
        // light rounds: zero-copy gather by kStageCtas CTAs on the SMs the
        // SCD grid leaves to unit A (faster than per-column copies); entry q + 1 is the
        // column's wait token.  The counters are zeroed on the compute stream before this round's
        // epoch can poll them.
        static const bool force_ce = std::getenv("DUHL_STAGE_CE") != nullptr;
        static const int nstage = std::getenv("DUHL_STAGE_CTAS") ? std::max(1, std::min(16, std::atoi(std::getenv("DUHL_STAGE_CTAS"))))
                                                               : kStageCtas;  // developer override (<= 16 counters)
        // (also when the copies complete before the epoch: the gather is the faster path either way)
        ctx->stage_ctas = (!heavy_ce && ctx->unit_a_ctas > 0 && !force_ce) ? nstage : 0;
        // every round that overlaps (or gathers) starts from zeroed counters: gather CTA 0's counter
        // is the copy engine's sequence counter progress[0], so a heavy (copy-engine) round after
        // a gather round would otherwise see the gather's final count as landed copies
#ifndef DUHL_EXP_OLD_PROGRESS_RESET  // developer: the round-2 bug, kept reproducible for the regression test
        if (ctx->stage_ctas > 0 || ctx->overlap) CK(cudaMemsetAsync(ctx->d_progress, 0, kProgressBytes, ctx->st));
#else
        if (ctx->stage_ctas > 0) CK(cudaMemsetAsync(ctx->d_progress, 0, kProgressBytes, ctx->st));
#endif
        // share of a gather round's columns copied by the copy engine beside the gather kernel:
        // only for long columns -- a per-column copy costs a fixed setup, so 160-KB columns (C3)
        // move at ~22 GB/s on the copy engine against ~50 for the gather (C3 time to 1e-5 2.30 s
        // with a 0.3 share, 1.88 s without)
        static const char* ce_env = std::getenv("DUHL_STAGE_CE_SHARE");
        const double ce_share_cfg = ce_env ? std::atof(ce_env)
                                           : ((size_t)ctx->ld_dev * sizeof(float) >= kStageCeMinBytes ? kStageCeShare : 0.0);
        const double ce_share = ctx->write_value ? std::max(0.0, std::min(0.9, ce_share_cfg)) : 0.0;
        unsigned nce = 0, ngath = 0;
        size_t fi = 0;
        const unsigned heavy_seq = ctx->overlap && heavy_ce ? ctx->batch_seq + 1 : 0u;
        for (size_t q = 0; q < news.size(); ++q) {
            const int64_t j = news[q];
            const int s = free_slots[fi++];
            ctx->col_slot[j] = s;
            ctx->slot_col[s] = (int)j;
            ctx->pend_cols.push_back(j);
            ctx->pend_slots.push_back(s);
            unsigned seq = 0;
            if (ctx->stage_ctas > 0) {  // every k-th column (Bresenham on the share) to the copy engine
                const bool ce = std::floor((double)(q + 1) * ce_share) > std::floor((double)q * ce_share);
                seq = ce ? (kCeToken | (unsigned)++nce) : (unsigned)++ngath;
            }
            else if (ctx->overlap) seq = heavy_ce ? heavy_seq : ctx->batch_seq + 1 + (unsigned)(q / 4);
            ctx->slot_batch[s] = seq;
            ctx->copy_plan.push_back({j, s, seq});
        }
        // swaps = |P_t \ P_{t-1}| (Fig. 4b's count; P_{-1} = {}): the columns copied, except that
        // round 0 may find some of them left in the pool by duhl_create's ingest pass
        for (int64_t j : P) nsw += ctx->inP[j] ? 0 : 1;
        if (ctx->overlap && ctx->stage_ctas == 0 && !news.empty())
            ctx->batch_seq = heavy_ce ? heavy_seq : ctx->batch_seq + (unsigned)((news.size() + 3) / 4);
        // the compute stream may still read evicted slots (previous epoch): order copies after it
        CK(cudaEventRecord(ctx->ev_copy, ctx->st));
        CK(cudaStreamWaitEvent(ctx->cst, ctx->ev_copy, 0));
        CK(cudaStreamWaitEvent(ctx->cst2, ctx->ev_copy, 0));
    } else {  // everything resident: bookkeeping on the device
        CK(cudaMemcpyAsync(ctx->d_P, P.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        TRY(resident_commit(ctx, m, swaps));
        ctx->P = P;
        std::fill(ctx->inP.begin(), ctx->inP.end(), 0);
        for (int64_t j : P) ctx->inP[j] = 1;
        ctx->P_host_valid = true;
        return DUHL_OK;
    }
    TRY(upload_slots_changes(ctx, chg_cols, chg_slots));
    std::vector<int> Ps(m);
    std::vector<unsigned> Pb(m);
    for (int64_t q = 0; q < m; ++q) {
        Ps[q] = ctx->col_slot[P[q]];
        Pb[q] = ctx->slot_batch.empty() ? 0u : ctx->slot_batch[Ps[q]];
    }
    CK(cudaMemcpyAsync(ctx->d_P, P.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_P_slot, Ps.data(), m * sizeof(int), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_P_batch, Pb.data(), m * sizeof(unsigned), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->P = P;
    ctx->m_cur = m;
    ctx->P_host_valid = true;
    std::fill(ctx->inP.begin(), ctx->inP.end(), 0);
    for (int64_t j : P) ctx->inP[j] = 1;
    if (swaps) *swaps = nsw;
    return DUHL_OK;
}

// (Device memory comes from plain cudaMalloc: the stream-ordered pool allocator would avoid the
// driver's occasional 0.1-1 s cudaFree / cudaMalloc stalls seen in repeated create / close loops
// (tools/create_timing.py), but cuStreamWriteValue32 -- the staging progress counters -- rejects
// pool memory, and creates still stalled now and then with it.)
static void free_all(duhl_ctx* ctx) {
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->cst) cudaStreamSynchronize(ctx->cst);
    if (ctx->cst2) cudaStreamSynchronize(ctx->cst2);
    if (ctx->rst) cudaStreamSynchronize(ctx->rst);
    void* dev_ptrs[] = {ctx->pool, ctx->d_col_slot, ctx->d_alpha, ctx->d_vt, ctx->d_b, ctx->d_y,
                        ctx->d_norms, ctx->d_z, ctx->d_P, ctx->d_order_j, ctx->d_cols,
                        ctx->d_chg_cols, ctx->d_P_slot, ctx->d_order_slot, ctx->d_chg_slots,
                        ctx->d_vsnap, ctx->d_s_acc2, ctx->d_progress, ctx->d_P_batch,
                        ctx->d_dv, ctx->d_aold, ctx->d_ls,
                        ctx->d_order_batch, ctx->d_order_a, ctx->d_order_inv, ctx->d_order_y,
                        ctx->d_s_acc, ctx->d_gap_out, ctx->d_s_out, ctx->d_sums, ctx->d_flag,
                        ctx->d_red, ctx->d_bar, ctx->d_colptr, ctx->d_rows, ctx->d_vals, ctx->d_topm_work,
                        ctx->d_stamp, ctx->d_rsel, ctx->d_rho, ctx->d_hs, ctx->d_hcols,
                        ctx->d_plan_cols, ctx->d_plan_slots, ctx->d_vf, ctx->d_v0t, ctx->d_a0t, ctx->d_u0, ctx->d_est,
                        ctx->d_smp};
    for (void* p : dev_ptrs)
        if (p) cudaFree(p);
    if (ctx->comm && nccl_api()) nccl_api()->commDestroy(ctx->comm);
    hua_destroy(ctx->hua);
    ctx->hua = nullptr;
    for (void* p : {(void*)ctx->h_vt, (void*)ctx->h_hs, (void*)ctx->h_hnorm, (void*)ctx->h_hcols,
                    (void*)ctx->h_ref_idx, (void*)ctx->h_ref_smp, (void*)ctx->h_plan_cols,
                    (void*)ctx->h_plan_slots})
        if (p) cudaFreeHost(p);
    for (cudaEvent_t e : {ctx->ev_hvt, ctx->ev_g0, ctx->ev_g1, ctx->ev_c1})
        if (e) cudaEventDestroy(e);
    if (ctx->registered) cudaHostUnregister(ctx->h_store);
    if (ctx->own_store && ctx->h_store) cudaFreeHost(ctx->h_store);
    for (auto& t : ctx->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
    if (ctx->ev_snap) cudaEventDestroy(ctx->ev_snap);
    if (ctx->ev_ref) cudaEventDestroy(ctx->ev_ref);
    if (ctx->ev_plan) cudaEventDestroy(ctx->ev_plan);
    if (ctx->rst) cudaStreamDestroy(ctx->rst);

    if (ctx->st) cudaStreamDestroy(ctx->st);
    if (ctx->cst) cudaStreamDestroy(ctx->cst);
    if (ctx->cst2) cudaStreamDestroy(ctx->cst2);
    if (ctx->ev_copy2) cudaEventDestroy(ctx->ev_copy2);
}

static size_t scd_red_bytes(const duhl_ctx* ctx) {
    return (ctx->pipe ? pipe_red_doubles(ctx->W) : scd_red_doubles(ctx->W)) * sizeof(double);
}

// SCD launch shape: G CTAs own contiguous row ranges of R rows (R % 4 == 0);
// W = coordinates per Gram block, largest multiple of 4 (<= 32) whose
// double-buffered stage fits in shared memory.
static void choose_scd_shape(duhl_ctx* ctx) {
    // the unit-A refresh grid keeps its SMs while the epoch runs
    const int64_t sms = std::max<int64_t>(1, ctx->nsm - std::max(0, ctx->unit_a_ctas));
    if (ctx->cfg.scd_async && !ctx->csc) {
        // asynchronous epoch: W coordinates in flight, each on a cluster of C CTAs whose row
        // slices of the column fit in shared memory (<= 200 KB: C4's 803-KB columns take C = 4)
        int W = ctx->cfg.scd_block > 0 ? ctx->cfg.scd_block : 16;
        int C = 1;  // two slices (double buffer) of <= 200 KB together
        while (C < 8 && round4((ctx->d4 + C - 1) / C) * 8 > 200 * 1024) C *= 2;
        if (const char* e = std::getenv("DUHL_TPA_CLUSTER"))  // developer override (power of 2, <= 8)
            C = std::max(C, std::min(8, std::atoi(e)));
        ctx->tpa_v0s = false;
        W = (int)std::max<int64_t>(1, std::min<int64_t>(W, sms / C));
        ctx->tpa = true;
        ctx->tpa_C = C;
        ctx->tpa_Rc = round4((ctx->d4 + C - 1) / C);
        ctx->W = W;
        ctx->G = W * C;
        ctx->R = (int)ctx->tpa_Rc;
        return;
    }
    // pipelined kernel (scd_pipe.cuh): G compute CTAs + 1 control CTA; W <= 32 with 3 (else 4)
    // TMA stages.  Auto (scd_kernel 0) takes it where shared memory allows W >= 24 (short row
    // slices, e.g. C3: 2x fewer blocks than W = 16, measured 14.7 vs 25 ms per pass); at W <= 16
    // the warp-specialised kernel is as fast or faster (C4, W = 12: 6.6 vs 7.3 ms).
    if (ctx->cfg.scd_kernel != 1 && ctx->cfg.scd_kernel != 3) {
        const int64_t smax = std::max<int64_t>(1, sms - 1);
        int64_t G = ctx->cfg.scd_ctas > 0 ? std::min<int64_t>(ctx->cfg.scd_ctas, smax)
                                          : std::min<int64_t>(smax, std::max<int64_t>(1, (ctx->d4 + 127) / 128));
        int64_t R = round4((ctx->d4 + G - 1) / G);
        G = (ctx->d4 + R - 1) / R;
        const size_t cap = 225 * 1024;
        int W = ctx->cfg.scd_block > 0 ? ctx->cfg.scd_block : 32;
        W = std::max(4, std::min(32, W / 4 * 4));
        while (W > 4 && pipe_smem_bytes(W, (int)R, 3) > cap) W -= 4;
        if (ctx->cfg.scd_kernel == 2 || W >= 24) {
            ctx->pipe = true;
            ctx->NB = pipe_smem_bytes(W, (int)R, 4) <= cap ? 4 : 3;
            if (const char* e = std::getenv("DUHL_SCD_STAGES")) ctx->NB = std::max(3, std::min(4, std::atoi(e)));
            ctx->W = W;
            ctx->R = (int)R;
            ctx->G = (int)G;
            return;
        }
    }
    ctx->pipe = false;
    // k_scd_ser (no cross Gram, u assembled by the compute warps) unless k_scd_gram is asked
    // for: C4 fast mode 4.65 vs 6.87 ms per pass, exact 6.4 vs 7.2
    ctx->ser = ctx->cfg.scd_kernel != 1;
    if (const char* e = std::getenv("DUHL_SCD_SER")) ctx->ser = std::atoi(e) != 0;  // developer A/B
    int64_t G = ctx->cfg.scd_ctas > 0 ? std::min<int64_t>(ctx->cfg.scd_ctas, sms)
                                      : std::min<int64_t>(sms, std::max<int64_t>(1, (ctx->d4 + 127) / 128));
    int64_t R = round4((ctx->d4 + G - 1) / G);
    G = (ctx->d4 + R - 1) / R;
    // W <= 16 coordinates per block; 3 TMA stages of W column slices must fit in
    // shared memory together with the fp64 v slice and per-warp partials
    int W = ctx->cfg.scd_block > 0 ? ctx->cfg.scd_block : 16;
    W = std::max(4, std::min(16, W / 4 * 4));
    const size_t cap = 225 * 1024;
    while (W > 4 && scd_smem_bytes(W, (int)R, 3) > cap) W -= 4;
    ctx->NB = 3;
    ctx->W = W;
    ctx->R = (int)R;
    ctx->G = (int)G;
}

// ============================================================================ C ABI
extern "C" {

void duhl_default_config(duhl_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->refresh_fraction = 0.05;
    cfg->cert_every = 10;
    cfg->seed = 170805357ull;
    cfg->cert_adaptive = 1;
    cfg->scd_exact = 1;
    cfg->unit_a_host_share = -1.0;
}

const char* duhl_last_error(const duhl_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// Dense (A) or sparse (C) ingest; exactly one is non-null.
static duhl_status create_impl(const duhl_matrix* A, const duhl_csc* C, const double* b_or_y, double lambda,
                               duhl_model model, const duhl_config* cfg_in, duhl_ctx** out) {
    if (!out) return DUHL_E_INVALID;
    *out = nullptr;
    if (A && (!A->values || A->d < 1 || A->n < 1 || A->ld < A->d)) return DUHL_E_INVALID;
    if (C && (!C->col_ptr || !C->row_idx || !C->values || C->d < 1 || C->n < 1 || C->d > (int64_t)INT32_MAX))
        return DUHL_E_INVALID;
    if (!A == !C || !b_or_y) return DUHL_E_INVALID;
    if (!(lambda > 0.0) || !std::isfinite(lambda)) return DUHL_E_INVALID;
    if (model != DUHL_LASSO && model != DUHL_SVM_DUAL && model != DUHL_RIDGE && model != DUHL_ELASTIC_NET)
        return DUHL_E_INVALID;
    if (model == DUHL_ELASTIC_NET && !(cfg_in && cfg_in->eta > 0.0 && cfg_in->eta < 1.0)) return DUHL_E_INVALID;
    const int64_t nin = A ? A->n : C->n, din = A ? A->d : C->d;
    if (nin > (int64_t)INT32_MAX - 1) return DUHL_E_INVALID;
    duhl_ctx* ctx = new duhl_ctx();
    if (cfg_in) ctx->cfg = *cfg_in; else duhl_default_config(&ctx->cfg);
    if (ctx->cfg.cert_every < 1) ctx->cfg.cert_every = 1;
    ctx->model = model;
    ctx->d = din;
    ctx->n = nin;
    ctx->csc = C != nullptr;
    if (ctx->csc) {  // validate the structure once on the host
        const int64_t* cp = C->col_ptr;
        if (cp[0] != 0) { delete ctx; return DUHL_E_INVALID; }
        for (int64_t i = 0; i < nin; ++i)
            if (cp[i + 1] < cp[i]) { delete ctx; return DUHL_E_INVALID; }
        ctx->nnz = cp[nin];
        for (int64_t i = 0; i < nin; ++i)
            for (int64_t k = cp[i]; k < cp[i + 1]; ++k) {
                const int32_t r = C->row_idx[k];
                if (r < 0 || r >= din || (k > cp[i] && r <= C->row_idx[k - 1]) || !std::isfinite(C->values[k])) {
                    delete ctx;
                    return DUHL_E_INVALID;
                }
            }
        if (ctx->cfg.hbm_budget_bytes != 0) {  // a sparse matrix is held resident
            const size_t need = (size_t)ctx->nnz * 8 + (size_t)(nin + 1) * 8;
            if (ctx->cfg.hbm_budget_bytes < need) { delete ctx; return DUHL_E_INVALID; }
            ctx->cfg.hbm_budget_bytes = 0;
        }
        ctx->h_colptr.assign(cp, cp + nin + 1);
        // concurrency of the asynchronous epoch (warps): scd_ctas if given, else d/16.  Concurrent
        // steps are Jacobi-like: a step ignores the others' updates, whose summed effect on it is
        // ~ sqrt(C/d) of its own for C concurrent random columns, so C = d/16 keeps it ~1/4.  The
        // exact line search on the round's step keeps every round monotone; it is
        // always on for the asynchronous sparse epoch (sparse path)
        ctx->csc_warps = ctx->cfg.scd_ctas > 0 ? ctx->cfg.scd_ctas : (int)std::max<int64_t>(32, din / 16);
        if (!ctx->cfg.scd_exact) ctx->cfg.linesearch = 1;
    }
    ctx->n_glob = ctx->cfg.n_global > 0 ? ctx->cfg.n_global : nin;
    ctx->col_offset = ctx->cfg.col_offset;
    if (ctx->col_offset < 0 || ctx->col_offset + nin > ctx->n_glob) { delete ctx; return DUHL_E_INVALID; }
    ctx->d4 = round4(din);
    ctx->lambda = lambda;
    const int64_t d = ctx->d, n = ctx->n, d4 = ctx->d4;
    // labels
    if (model == DUHL_SVM_DUAL) {
        for (int64_t i = 0; i < n; ++i)
            if (b_or_y[i] != 1.0 && b_or_y[i] != -1.0) { delete ctx; return DUHL_E_INVALID; }
    } else {
        for (int64_t k = 0; k < d; ++k)
            if (!std::isfinite(b_or_y[k])) { delete ctx; return DUHL_E_INVALID; }
    }
    auto bail = [&](duhl_status s) { free_all(ctx); delete ctx; return s; };
    // device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= ctx->cfg.device) return bail(DUHL_E_CUDA);
    ctx->dev = ctx->cfg.device;
    if (cudaSetDevice(ctx->dev) != cudaSuccess) return bail(DUHL_E_CUDA);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, ctx->dev) != cudaSuccess || prop.major != 10) return bail(DUHL_E_CUDA);
    ctx->nsm = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->cst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->cst2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_copy2, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->rst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_snap, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_ref, cudaEventDisableTiming) != cudaSuccess)
        return bail(DUHL_E_CUDA);
    if (preload_kernels() != cudaSuccess || preload_tpa_kernels() != cudaSuccess)
        return bail(DUHL_E_CUDA);  // no lazy loads mid-epoch
    if (ctx->csc) {  // ---- sparse: the CSC arrays go to HBM once
        auto dm = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes > 0 ? bytes : 16) == cudaSuccess; };
        if (!dm((void**)&ctx->d_colptr, (n + 1) * sizeof(int64_t)) || !dm((void**)&ctx->d_rows, ctx->nnz * sizeof(int)) ||
            !dm((void**)&ctx->d_vals, ctx->nnz * sizeof(float))) {
            cudaGetLastError();
            return bail(DUHL_E_NOMEM);
        }
        if (cudaMemcpy(ctx->d_colptr, C->col_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(ctx->d_rows, C->row_idx, ctx->nnz * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(ctx->d_vals, C->values, ctx->nnz * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(DUHL_E_CUDA);
        ctx->h2d_bytes += (int64_t)((n + 1) * 8 + ctx->nnz * 8);
    } else {
    // ---- unit A: pinned host store (column i at h_store + i*ld_host, rows d..d4 zero)
    const bool can_borrow = ctx->cfg.borrow_host && d % 4 == 0 && A->ld % 4 == 0 &&
                            ((uintptr_t)A->values % 16 == 0);
    if (can_borrow) {
        ctx->h_store = const_cast<float*>(A->values);
        ctx->ld_host = A->ld;
        // memory the caller already pinned (cudaHostAlloc / cudaHostRegister, e.g. a pinned
        // torch tensor) is used as is -- pinning 32 GB costs ~3.3 s on this box (tools/micro/stage.cu)
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, ctx->h_store) == cudaSuccess &&
                            pa.type == cudaMemoryTypeHost && pa.devicePointer != nullptr;
        cudaGetLastError();
        if (!pinned) {
            if (cudaHostRegister(ctx->h_store, (size_t)n * A->ld * sizeof(float),
                                 cudaHostRegisterMapped | cudaHostRegisterReadOnly) != cudaSuccess) {
                cudaGetLastError();
                if (cudaHostRegister(ctx->h_store, (size_t)n * A->ld * sizeof(float), cudaHostRegisterMapped) !=
                    cudaSuccess)
                    return bail(DUHL_E_CUDA);
            }
            ctx->registered = true;
        }
    } else {
        ctx->ld_host = d4;
        if (cudaHostAlloc((void**)&ctx->h_store, (size_t)n * d4 * sizeof(float), cudaHostAllocMapped) !=
            cudaSuccess)
            return bail(DUHL_E_NOMEM);
        ctx->own_store = true;
        const float* src = A->values;
        const int64_t ld = A->ld;
        float* dst = ctx->h_store;
        unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([=]() {
                for (int64_t i = t; i < n; i += nt) {
                    std::memcpy(dst + i * d4, src + i * ld, (size_t)d * sizeof(float));
                    for (int64_t k = d; k < d4; ++k) dst[i * d4 + k] = 0.0f;
                }
            });
        for (auto& x : th) x.join();
    }
    // data validity (finite values) is checked by the device ingest pass below: a non-finite
    // element makes ||a_i||^2 non-finite
    void* alias = nullptr;
    if (cudaHostGetDevicePointer(&alias, ctx->h_store, 0) != cudaSuccess) return bail(DUHL_E_CUDA);
    ctx->h_alias = (const float*)alias;
    }
    // ---- unit B: slot pool
    ctx->ld_dev = d4;
    const size_t col_bytes = (size_t)d4 * sizeof(float);
    if (ctx->cfg.hbm_budget_bytes == 0) {
        ctx->S = n;
    } else {
        ctx->S = std::min<int64_t>(n, (int64_t)(ctx->cfg.hbm_budget_bytes / col_bytes));
        if (ctx->S < 1) { ctx->err = "HBM budget smaller than one column"; return bail(DUHL_E_INVALID); }
    }
    ctx->m_cfg = ctx->cfg.m > 0 ? ctx->cfg.m : ctx->S;
    if (ctx->m_cfg > n || ctx->m_cfg > ctx->S) return bail(DUHL_E_INVALID);
    auto dmal = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes > 0 ? bytes : 16) == cudaSuccess; };
    bool ok = dmal((void**)&ctx->pool, ctx->csc ? 0 : (size_t)ctx->S * col_bytes) &&
              dmal((void**)&ctx->d_col_slot, n * sizeof(int)) &&
              dmal((void**)&ctx->d_alpha, n * sizeof(double)) &&
              dmal((void**)&ctx->d_vt, d4 * sizeof(double)) &&
              dmal((void**)&ctx->d_b, d4 * sizeof(double)) &&
              dmal((void**)&ctx->d_y, n * sizeof(double)) &&
              dmal((void**)&ctx->d_norms, n * sizeof(double)) &&
              dmal((void**)&ctx->d_z, n * sizeof(double)) &&
              dmal((void**)&ctx->d_P, n * sizeof(int64_t)) &&
              dmal((void**)&ctx->d_order_j, n * sizeof(int64_t)) &&
              dmal((void**)&ctx->d_cols, n * sizeof(int64_t)) &&
              dmal((void**)&ctx->d_chg_cols, 2 * n * sizeof(int64_t)) &&
              dmal((void**)&ctx->d_P_slot, n * sizeof(int)) &&
              dmal((void**)&ctx->d_order_slot, n * sizeof(int)) &&
              dmal((void**)&ctx->d_chg_slots, 2 * n * sizeof(int)) &&
              dmal((void**)&ctx->d_vsnap, d4 * sizeof(double)) &&
              dmal((void**)&ctx->d_dv, d4 * sizeof(double)) &&
              dmal((void**)&ctx->d_aold, n * sizeof(double)) &&
              dmal((void**)&ctx->d_ls, 256 * sizeof(double)) &&
              dmal((void**)&ctx->d_s_acc2, n * sizeof(double)) &&
              dmal((void**)&ctx->d_progress, kProgressBytes) &&
              dmal((void**)&ctx->d_P_batch, n * sizeof(unsigned)) &&
              dmal((void**)&ctx->d_order_batch, n * sizeof(unsigned)) &&
              dmal((void**)&ctx->d_order_a, n * sizeof(double)) &&
              dmal((void**)&ctx->d_order_inv, n * sizeof(double)) &&
              dmal((void**)&ctx->d_order_y, n * sizeof(double)) &&
              dmal((void**)&ctx->d_s_acc, n * sizeof(double)) &&
              dmal((void**)&ctx->d_gap_out, n * sizeof(double)) &&
              dmal((void**)&ctx->d_s_out, n * sizeof(double)) &&
              dmal((void**)&ctx->d_sums, 8 * sizeof(double)) &&
              dmal((void**)&ctx->d_flag, 4 * sizeof(int)) &&
              dmal((void**)&ctx->d_plan_cols, n * sizeof(int64_t)) &&
              dmal((void**)&ctx->d_plan_slots, n * sizeof(int));
    if (!ok) { cudaGetLastError(); ctx->err = "cudaMalloc failed"; return bail(DUHL_E_NOMEM); }
    // SMs the SCD grid leaves to unit A's refresh and the staging gather of budgeted problems:
    // 8 (measured: C4 step 85 vs 90 ms with 16 refresh CTAs)
    ctx->unit_a_ctas = ctx->cfg.unit_a_ctas > 0 ? std::min(ctx->cfg.unit_a_ctas, ctx->nsm / 2)
                       : (ctx->cfg.unit_a_ctas == 0 && ctx->cfg.hbm_budget_bytes != 0 && !ctx->csc) ? 8 : 0;
    choose_scd_shape(ctx);
    if (ctx->tpa) {
        if (ctx->tpa_Rc * 8 > 200 * 1024) { ctx->err = "column too long for the asynchronous epoch"; return bail(DUHL_E_INVALID); }
        if (!dmal((void**)&ctx->d_vf, d4 * sizeof(float)) || !dmal((void**)&ctx->d_v0t, d4 * sizeof(double)) ||
            !dmal((void**)&ctx->d_a0t, n * sizeof(double)) || !dmal((void**)&ctx->d_u0, n * sizeof(double)))
            return bail(DUHL_E_NOMEM);
        ctx->cfg.linesearch = 1;  // asynchronous rounds take the exact gamma line search
    }
    if (!dmal((void**)&ctx->d_topm_work, launch_topm_work_bytes()) || !dmal((void**)&ctx->d_stamp, n * sizeof(int)) ||
        !dmal((void**)&ctx->d_rsel, 2 * sizeof(unsigned long long)) || !dmal((void**)&ctx->d_rho, 2 * sizeof(double)) ||
        !dmal((void**)&ctx->d_est, 4 * sizeof(double)) || !dmal((void**)&ctx->d_smp, n * sizeof(int64_t)) ||
        cudaMemset(ctx->d_est, 0, 4 * sizeof(double)) != cudaSuccess)
        return bail(DUHL_E_NOMEM);
    if (cudaMemset(ctx->d_stamp, 0xff, n * sizeof(int)) != cudaSuccess) return bail(DUHL_E_CUDA);  // -1: never
    if (!ctx->csc && ctx->cfg.unit_a_host_threads > 0) {  // unit A on host threads (duhl.h)
        if (ctx->cfg.unit_a_host_threads > 1024 || ctx->cfg.unit_a_host_share > 1.0) return bail(DUHL_E_INVALID);
        if (!dmal((void**)&ctx->d_hs, n * sizeof(double)) || !dmal((void**)&ctx->d_hcols, n * sizeof(int64_t)) ||
            cudaMemset(ctx->d_hs, 0, n * sizeof(double)) != cudaSuccess)
            return bail(DUHL_E_NOMEM);
        if (cudaHostAlloc((void**)&ctx->h_vt, ctx->d4 * sizeof(double), 0) != cudaSuccess ||
            cudaHostAlloc((void**)&ctx->h_hs, n * sizeof(double), 0) != cudaSuccess ||
            cudaHostAlloc((void**)&ctx->h_hnorm, n * sizeof(double), 0) != cudaSuccess ||
            cudaHostAlloc((void**)&ctx->h_hcols, n * sizeof(int64_t), 0) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_hvt, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreate(&ctx->ev_g0) != cudaSuccess || cudaEventCreate(&ctx->ev_g1) != cudaSuccess ||
            cudaEventCreate(&ctx->ev_c1) != cudaSuccess)
            return bail(DUHL_E_NOMEM);
        if (ctx->cfg.unit_a_host_share >= 0.0) ctx->hua_share = ctx->cfg.unit_a_host_share;
        ctx->hua = hua_create(ctx->cfg.unit_a_host_threads, ctx->dev);
    }
    if (!dmal((void**)&ctx->d_red, scd_red_bytes(ctx)) ||
        !dmal((void**)&ctx->d_bar, 64))
        return bail(DUHL_E_NOMEM);
    if (!ctx->csc && ctx->cfg.hbm_budget_bytes != 0 &&
        (cudaHostAlloc((void**)&ctx->h_plan_cols, n * sizeof(int64_t), 0) != cudaSuccess ||
         cudaHostAlloc((void**)&ctx->h_plan_slots, n * sizeof(int), 0) != cudaSuccess ||
         cudaEventCreateWithFlags(&ctx->ev_plan, cudaEventDisableTiming) != cudaSuccess))
        return bail(DUHL_E_NOMEM);
    ctx->col_slot.assign(n, -1);
    ctx->slot_col.assign(ctx->S, -1);
    ctx->slot_batch.assign(ctx->S, 0u);
    {   // stream memory ops (copy-progress counter) if the driver offers them
        int memops = 0;
        cudaDeviceGetAttribute(&memops, (cudaDeviceAttr)120 /* CAN_USE_STREAM_MEM_OPS_V1 */, ctx->dev);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess && fn && !std::getenv("DUHL_NO_STAGING_OVERLAP"))
            ctx->write_value = (duhl_ctx::WriteValue32)fn;
        (void)memops;
        cudaGetLastError();
    }
    ctx->inP.assign(n, 0);
    cudaStream_t st = ctx->st;
    bool ok2 = true;
    auto ck = [&](cudaError_t e) { if (e != cudaSuccess) ok2 = false; };
    ck(cudaMemsetAsync(ctx->d_s_acc, 0, n * sizeof(double), st));
    ck(cudaMemsetAsync(ctx->d_s_acc2, 0, n * sizeof(double), st));
    ck(cudaMemsetAsync(ctx->d_progress, 0, kProgressBytes, st));
    ck(cudaMemsetAsync(ctx->d_flag, 0, 4 * sizeof(int), st));
    ck(cudaMemsetAsync(ctx->d_alpha, 0, n * sizeof(double), st));
    ck(cudaMemsetAsync(ctx->d_b, 0, d4 * sizeof(double), st));
    ck(cudaMemsetAsync(ctx->d_y, 0, n * sizeof(double), st));
    if (ctx->cfg.hbm_budget_bytes == 0) {  // everything resident: slot i = column i
        for (int64_t i = 0; i < n; ++i) { ctx->col_slot[i] = (int)i; ctx->slot_col[i] = (int)i; }
        if (!ctx->csc) {
            ck(cudaMemcpy2DAsync(ctx->pool, col_bytes, ctx->h_store, ctx->ld_host * sizeof(float), col_bytes,
                                 (size_t)n, cudaMemcpyHostToDevice, st));
            ctx->h2d_bytes += (int64_t)(n * col_bytes);
        }
    }
    ck(cudaMemcpyAsync(ctx->d_col_slot, ctx->col_slot.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    if (model == DUHL_SVM_DUAL)
        ck(cudaMemcpyAsync(ctx->d_y, b_or_y, n * sizeof(double), cudaMemcpyHostToDevice, st));
    else
        ck(cudaMemcpyAsync(ctx->d_b, b_or_y, d * sizeof(double), cudaMemcpyHostToDevice, st));
    ck(cudaStreamSynchronize(st));
    if (!ok2) { cudaGetLastError(); ctx->err = "device setup failed"; return bail(DUHL_E_CUDA); }
    // ---- precompute (a1): B, initial shared vector, then ONE pass over A for ||a_i||^2 and
    // z = the exact gaps at alpha = 0 (SVM: 1/n; regression: from a_i^T (-b))
    if (ctx->csc) ck(launch_csc_norms(cscmat(ctx), n, ctx->d_norms, st, &ctx->launches));
    if (model == DUHL_LASSO) {
        double h[2] = {0, 0};
        ck(cudaMemsetAsync(ctx->d_sums, 0, 8 * sizeof(double), st));
        ck(launch_vec_sums(ctx->d_b, nullptr, d4, ctx->d_sums, st, &ctx->launches));
        ck(d2h_copy(ctx, h, ctx->d_sums, 2 * sizeof(double), st));
        ck(cudaStreamSynchronize(st));
        ctx->B = h[0] / (2.0 * lambda * (double)d);  // P:848, reading R1
    }
    ck(launch_matvec(colsrc(ctx), ctx->d_alpha, 0, d, d4, model != DUHL_SVM_DUAL ? ctx->d_b : nullptr,
                     ctx->d_vt, st, &ctx->launches));  // alpha = 0: v~ = -b, v^ = 0
    ck(cudaStreamSynchronize(st));
    if (!ok2) { cudaGetLastError(); ctx->err = "precompute failed"; return bail(DUHL_E_CUDA); }
    if (!ctx->csc) {  // ingest: norms + gaps at alpha = 0 in one pass (k_gap_tile<INGEST>)
        ck(cudaMemsetAsync(ctx->d_norms, 0, n * sizeof(double), st));
        // unit A on host threads takes a share of the pass (as of the refresh): columns
        // [ng, n) -- norms and a_i^T v~ at alpha = 0 straight from host DRAM, while the GPU reads
        // [0, ng) over PCIe; the GPU keeps at least the S columns it leaves in the pool.  C4 (14
        // threads): create 0.84 s with the GPU alone, 0.40 / 0.31 / 0.24 s at host shares 0.5 /
        // 0.6 / 0.7 (both sides then read host DRAM at ~95 + ~45 GB/s)
        static const double host_share = std::getenv("DUHL_INGEST_HOST_SHARE")
                                             ? std::atof(std::getenv("DUHL_INGEST_HOST_SHARE")) : 0.7;
        int64_t ng = n;
        if (ctx->hua && ctx->cfg.hbm_budget_bytes != 0 && host_share > 0.0)
            ng = std::max<int64_t>(std::min<int64_t>(ctx->S, n),
                                   n - (int64_t)std::llround(std::min(1.0, host_share) * (double)n));
        const int64_t kh = n - ng;
        if (kh > 0) {  // v~ at alpha = 0: -b (Lasso, ridge, elastic net) or 0 (SVM dual)
            for (int64_t r = 0; r < ctx->d4; ++r)
                ctx->h_vt[r] = (model != DUHL_SVM_DUAL && r < d) ? -b_or_y[r] : 0.0;
            for (int64_t t = 0; t < kh; ++t) ctx->h_hcols[t] = ng + t;
            ck(cudaEventRecord(ctx->ev_hvt, st));
            hua_post(ctx->hua, ctx->h_store, ctx->ld_host, ctx->d4, ctx->h_hcols, kh, ctx->h_vt, wscale(ctx),
                     ctx->ev_hvt, ctx->h_hs, ctx->h_hnorm);
        }
        GapParams p = gap_params(ctx, nullptr, ng);
        p.norms_out = ctx->d_norms;
        // budgeted: the pass also leaves columns 0..S-1 in slots 0..S-1 (it reads them anyway);
        // the first selection keeps those of them it picks and evicts the rest (stage_working_set)
        const bool prefill = ctx->cfg.hbm_budget_bytes != 0 && !std::getenv("DUHL_NO_PREFILL");
        if (prefill) {
            p.fill_pool = ctx->pool;
            p.fill_ld = ctx->ld_dev;
            p.fill_cols = std::min<int64_t>(ctx->S, n);
        }
        ProfScope ps(ctx, st, 1, (double)n * (4.0 * ctx->d4 + 24.0));
        if (kh > 0) ck(cudaEventRecord(ctx->ev_g0, st));
        ck(launch_gap_pass(p, kGapTileRows, st, &ctx->launches));
        if (kh > 0) ck(cudaEventRecord(ctx->ev_g1, st));
        ps.end();
        if (ctx->cfg.hbm_budget_bytes != 0)  // the GPU's share read the pinned store over PCIe
            ctx->zc_bytes += ng * ctx->ld_dev * (int64_t)sizeof(float);
        if (prefill) {
            for (int64_t i = 0; i < p.fill_cols; ++i) { ctx->col_slot[i] = (int)i; ctx->slot_col[i] = (int)i; }
            ck(cudaMemcpyAsync(ctx->d_col_slot, ctx->col_slot.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
        }
        if (kh > 0) {  // the host share: norms to their place, dots -> gap_i at alpha = 0 (k_gap_finalize)
            const double host_s = hua_wait(ctx->hua);
            float gms = 0.0f;  // both units' column rates seed the certificates' split (same regime:
                               // host threads and PCIe reads drawing on host DRAM together)
            if (cudaEventSynchronize(ctx->ev_g1) == cudaSuccess && host_s > 0.0 &&
                cudaEventElapsedTime(&gms, ctx->ev_g0, ctx->ev_g1) == cudaSuccess && gms > 0.0f) {
                const double rh = (double)kh / host_s, rg = (double)ng / (1e-3 * gms);
                ctx->cert_share = std::min(0.95, std::max(0.05, rh / (rh + rg)));
            }
            ck(cudaMemcpyAsync(ctx->d_norms + ng, ctx->h_hnorm, kh * sizeof(double), cudaMemcpyHostToDevice, st));
            ck(cudaMemcpyAsync(ctx->d_hs, ctx->h_hs, kh * sizeof(double), cudaMemcpyHostToDevice, st));
            ck(cudaMemcpyAsync(ctx->d_hcols, ctx->h_hcols, kh * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            GapParams hp = gap_params(ctx, ctx->d_hcols, kh);
            hp.s_acc = ctx->d_hs;
            ck(launch_gap_finalize(hp, st, &ctx->launches));
        }
        double h = 0.0;
        ck(cudaMemsetAsync(ctx->d_sums + 7, 0, sizeof(double), st));
        ck(launch_sum(ctx->d_norms, n, ctx->d_sums + 7, st, &ctx->launches));
        ck(cudaMemcpyAsync(&h, ctx->d_sums + 7, sizeof(double), cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        if (!ok2) { cudaGetLastError(); ctx->err = "ingest pass failed"; return bail(DUHL_E_CUDA); }
        if (!std::isfinite(h)) { ctx->err = "non-finite matrix entries"; return bail(DUHL_E_INVALID); }
    } else if (run_gaps(ctx, nullptr, n, nullptr, nullptr, nullptr) != DUHL_OK) {
        return bail(DUHL_E_CUDA);
    }
    if (check_flag(ctx, "initial gaps") != DUHL_OK) return bail(DUHL_E_NUMERIC);
    *out = ctx;
    return DUHL_OK;
}

duhl_status duhl_create(const duhl_matrix* A, const double* b_or_y, double lambda, duhl_model model,
                        const duhl_config* cfg, duhl_ctx** out) {
    if (!A) return DUHL_E_INVALID;
    return create_impl(A, nullptr, b_or_y, lambda, model, cfg, out);
}

duhl_status duhl_create_csc(const duhl_csc* A, const double* b_or_y, double lambda, duhl_model model,
                            const duhl_config* cfg, duhl_ctx** out) {
    if (!A) return DUHL_E_INVALID;
    return create_impl(nullptr, A, b_or_y, lambda, model, cfg, out);
}

duhl_status duhl_destroy(duhl_ctx* ctx) {
    if (!ctx) return DUHL_E_INVALID;
    cudaSetDevice(ctx->dev);
    free_all(ctx);
    delete ctx;
    return DUHL_OK;
}

duhl_status duhl_gaps(duhl_ctx* ctx, const int64_t* idx, int64_t k, double* z_out, double* s_out) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    const int64_t* dcols = nullptr;
    if (idx) {
        if (k < 0 || k > ctx->n) return fail(ctx, DUHL_E_INVALID, "k out of range");
        for (int64_t t = 0; t < k; ++t)
            if (idx[t] < 0 || idx[t] >= ctx->n) return fail(ctx, DUHL_E_INVALID, "index out of range");
        if (k == 0) return DUHL_OK;
        CK(cudaMemcpyAsync(ctx->d_cols, idx, k * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        dcols = ctx->d_cols;
    } else {
        k = ctx->n;
    }
    TRY(run_gaps(ctx, dcols, k, z_out ? ctx->d_gap_out : nullptr, s_out ? ctx->d_s_out : nullptr, nullptr));
    if (z_out) CK(d2h_copy(ctx, z_out, ctx->d_gap_out, k * sizeof(double), ctx->st));
    if (s_out) CK(d2h_copy(ctx, s_out, ctx->d_s_out, k * sizeof(double), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return check_flag(ctx, "duhl_gaps");
}

static duhl_status select_impl(duhl_ctx* ctx, duhl_policy policy, int64_t m, int64_t round,
                               int64_t* n_swaps_out) {
    if (m <= 0) m = ctx->m_cfg;
    if (m > ctx->n || m > ctx->S) return fail(ctx, DUHL_E_INVALID, "m exceeds n or the HBM slot pool");
    std::vector<int64_t> P;
    if (policy == DUHL_SEL_SEQUENTIAL) {  // blocks [k m, min((k+1) m, n)), k = round mod ceil(n/m)
        int64_t nblk = (ctx->n + m - 1) / m, kb = round % nblk;
        int64_t lo = kb * m, hi = std::min(ctx->n, lo + m);
        for (int64_t i = lo; i < hi; ++i) P.push_back(i);
    } else if (policy == DUHL_SEL_GAP || policy == DUHL_SEL_UNIFORM || policy == DUHL_SEL_IMPORTANCE) {
        {
            ProfScope ps(ctx, ctx->st, 2, 8.0 * ctx->n * 7);
            const int keymode = policy == DUHL_SEL_GAP ? 0 : (policy == DUHL_SEL_UNIFORM ? 1 : 2);
            CK(launch_topm(policy == DUHL_SEL_IMPORTANCE ? ctx->d_norms : ctx->d_z, ctx->n, m, keymode,
                           ctx->cfg.seed, round, ctx->d_P, ctx->d_flag, ctx->st, &ctx->launches,
                           ctx->d_topm_work));
        }
        if (ctx->cfg.hbm_budget_bytes == 0) {  // resident: P stays on the device
            TRY(finalize_staging(ctx));
            TRY(resident_commit(ctx, m, n_swaps_out));
            ctx->P_host_valid = false;
            return check_flag(ctx, "duhl_select");
        }
        P.resize(m);
        CK(d2h_copy(ctx, P.data(), ctx->d_P, m * sizeof(int64_t), ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        TRY(check_flag(ctx, "duhl_select"));
    } else {
        return fail(ctx, DUHL_E_INVALID, "unknown policy");
    }
    return stage_working_set(ctx, P, round, n_swaps_out);
}

duhl_status duhl_select(duhl_ctx* ctx, duhl_policy policy, int64_t m, int64_t round, int64_t* P_out,
                        int64_t* n_swaps_out) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    TRY(finalize_staging(ctx));
    ctx->overlap = ctx->write_value != nullptr && !ctx->tpa;
    TRY(select_impl(ctx, policy, m, round, n_swaps_out));
    if (P_out) {
        TRY(ensure_host_P(ctx));
        std::memcpy(P_out, ctx->P.data(), ctx->P.size() * sizeof(int64_t));
    }
    return DUHL_OK;
}

static duhl_status scd_launch(duhl_ctx* ctx, int64_t L, bool waits_on_staging = false) {
    if (ctx->csc) {  // asynchronous warp-per-coordinate epoch (exact mode: one warp, in order)
        CscScdParams q{};
        q.model = ctx->model;
        q.d = ctx->d;
        q.n = ctx->n_glob;
        q.lambda = ctx->lambda;
        q.A = cscmat(ctx);
        q.order_j = ctx->d_order_j;
        q.L = L;
        q.norms = ctx->d_norms;
        q.y = ctx->model == DUHL_SVM_DUAL ? ctx->d_y : nullptr;
        q.alpha = ctx->d_alpha;
        q.vt = ctx->d_vt;
        q.eta = ctx->cfg.eta;
        ProfScope ps(ctx, ctx->st, 0, ctx->csc_pass_bytes);
        CK(launch_csc_scd(q, ctx->cfg.scd_exact ? 1 : ctx->csc_warps, ctx->st, &ctx->launches));
        ctx->updates += L;
        return DUHL_OK;
    }
    if (ctx->tpa) {
        TpaParams q{};
        q.model = ctx->model;
        q.d = ctx->d;
        q.d4 = ctx->d4;
        q.n = ctx->n_glob;
        q.lambda = ctx->lambda;
        q.eta = ctx->cfg.eta;
        q.pool = ctx->pool;
        q.ld_dev = ctx->ld_dev;
        q.order_j = ctx->d_order_j;
        q.order_slot = ctx->d_order_slot;
        q.order_a = ctx->d_order_a;
        q.L = L;
        q.norms = ctx->d_norms;
        q.y = ctx->model == DUHL_SVM_DUAL ? ctx->d_y : nullptr;
        q.alpha = ctx->d_alpha;
        q.vf = ctx->d_vf;
        q.v0 = ctx->d_v0t;
        q.v0_smem = 0;
        q.u0 = ctx->d_u0;
        q.C = ctx->tpa_C;
        q.Rc = ctx->tpa_Rc;
        q.progress = nullptr;  // the asynchronous epoch starts after its columns landed
        q.err = ctx->d_flag + 1;
        ProfScope ps(ctx, ctx->st, waits_on_staging ? 5 : 0, (double)L * (4.0 * ctx->d4 + 24.0) + 16.0 * ctx->d4);
        CK(launch_scd_tpa(q, ctx->W, ctx->st, &ctx->launches));
        ctx->updates += L;
        return DUHL_OK;
    }
    ScdParams p{};
    p.model = ctx->model;
    p.d = ctx->d;
    p.d4 = ctx->d4;
    p.n = ctx->n_glob;
    p.lambda = ctx->lambda;
    p.pool = ctx->pool;
    p.ld_dev = ctx->ld_dev;
    p.order_j = ctx->d_order_j;
    p.order_slot = ctx->d_order_slot;
    p.L = L;
    p.norms = ctx->d_norms;
    p.y = ctx->model == DUHL_SVM_DUAL ? ctx->d_y : nullptr;
    p.alpha = ctx->d_alpha;
    p.vt = ctx->d_vt;
    p.W = ctx->W;
    p.R = ctx->R;
    p.G = ctx->G;
    p.NB = ctx->NB;
    p.exact = ctx->cfg.scd_exact;
    {   // DUHL_GRAM_TC=0/1 overrides the default (tensor-core Gram tiles where they apply)
        static const int tc = std::getenv("DUHL_GRAM_TC") ? std::atoi(std::getenv("DUHL_GRAM_TC")) : 1;
        p.gram_tc = tc;
    }
    p.lam_q = ridge_ld(ctx);
    p.lam_l1 = ctx->model == DUHL_ELASTIC_NET ? ctx->lambda * (double)ctx->d * (1.0 - ctx->cfg.eta) : 0.0;
    p.red = ctx->d_red;
    p.order_batch = ctx->overlap ? ctx->d_order_batch : nullptr;
    p.err = ctx->d_flag + 1;
    p.order_a = ctx->d_order_a;
    p.order_inv = ctx->d_order_inv;
    p.order_y = ctx->d_order_y;
    p.progress = ctx->overlap ? ctx->d_progress : nullptr;
    p.stage_ctas = ctx->overlap ? ctx->stage_ctas : 0;
    p.bar = ctx->d_bar;
    CK(cudaMemsetAsync(ctx->d_red, 0, scd_red_bytes(ctx), ctx->st));
    CK(cudaMemsetAsync(ctx->d_bar, 0, 64, ctx->st));
    static const bool trace = std::getenv("DUHL_SCD_TRACE") != nullptr;  // developer phase timing
    unsigned long long* dtr = nullptr;
    if (trace) {
        CK(cudaMalloc((void**)&dtr, 16 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(dtr, 0, 16 * sizeof(unsigned long long), ctx->st));
    }
    p.trace = dtr;
    {
        ProfScope ps(ctx, ctx->st, waits_on_staging ? 5 : 0, (double)L * (4.0 * ctx->d4 + 24.0) + 16.0 * ctx->d4);
        CK(ctx->pipe  ? launch_scd_pipe(p, ctx->st, &ctx->launches)
           : ctx->ser ? launch_scd_ser(p, ctx->st, &ctx->launches)
                      : launch_scd_gram(p, ctx->st, &ctx->launches));
    }
    if (trace) {
        unsigned long long h[16];
        TRY(issue_staging(ctx));  // the synchronize below must not starve a waiting epoch
        CK(d2h_copy(ctx, h, dtr, sizeof(h), ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        cudaFree(dtr);
        const double nb = (double)((L + ctx->W - 1) / ctx->W);
        int clk_khz = 0;
        cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, ctx->dev);
        const double cyc_per_us = clk_khz > 0 ? clk_khz / 1e3 : 1965.0;
        std::fprintf(stderr, "scd trace (us/block at %.0f MHz) W=%d G=%d R=%d: ", cyc_per_us, ctx->W, ctx->G,
                     ctx->R);
        const char* nm0a[8] = {"ctl:other", "-", "ctl:WAIT", "ctl:read", "ctl:seq", "cmp:wait-delta",
                              "cmp:vupdate", "cmp:tiles"};
        const char* const* nm0 = nm0a;
        const char* nm1[8] = {"ctl:poll", "ctl:read", "ctl:steps", "ctl:other", "ctl:publish", "-", "-", "-"};
        const char* nm1c[8] = {"gram:wait-data", "gram:tiles", "gram:sum+arrive", "v:wait-delta", "v:vupd",
                               "v:u+arrive", "v:other", "gram:other"};
        const char* nms[8] = {"ctl:WAIT", "ctl:read", "ctl:steps", "ctl:other", "cmp:data+G+u'", "cmp:wait-delta",
                              "cmp:corr", "cmp:RED+arrive+vupd"};
        const bool pipe = ctx->pipe;
        if (ctx->ser) nm0 = nms;
        for (int c2 = 0; c2 < 2; ++c2) {
            std::fprintf(stderr, "%s", pipe ? (c2 ? " | cta0: " : "control: ") : (c2 ? " | last: " : "cta0: "));
            for (int k = 0; k < 8; ++k)
                std::fprintf(stderr, "%s %.2f ", pipe ? (c2 ? nm1c[k] : nm1[k]) : nm0[k], h[c2 * 8 + k] / nb / cyc_per_us);
        }
        std::fprintf(stderr, "\n");
    }
    ctx->updates += L;
    return DUHL_OK;
}

// Asynchronous epoch (cfg.scd_async): start from v~0, alpha_P0 and a zero fp32 shadow of the
// epoch's updates; end
// with the exact resync v~ = v~0 + A_P (alpha_P - alpha_P0) in fp64, so gaps and
// certificates see the exact shared vector whatever the interleaving was.
static duhl_status tpa_begin(duhl_ctx* ctx, int64_t m) {
    CK(cudaMemcpyAsync(ctx->d_v0t, ctx->d_vt, ctx->d4 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
    CK(launch_gather_f64(ctx->d_alpha, ctx->d_P, m, ctx->d_a0t, ctx->st, &ctx->launches));
    // u0_j = a_j^T v~0 for j in P: one gap-kernel pass over the working set (its columns have
    // landed: the asynchronous epoch runs after its staging; the device table is brought up to
    // date first), s = a_j^T (wscale v~0) -> u0 = s / wscale
    TRY(finalize_staging(ctx));
    {
        GapParams gp = gap_params(ctx, ctx->d_P, m);
        gp.vt = ctx->d_v0t;
        gp.z = nullptr;
        gp.s_out = ctx->d_s_out;
        const int64_t tiles = (ctx->d4 + kGapTileRows - 1) / kGapTileRows;
        ProfScope ps(ctx, ctx->st, 6, (double)m * (4.0 * ctx->d4 + 24.0) + 8.0 * ctx->d4 * tiles);
        CK(launch_gap_pass(gp, kGapTileRows, ctx->st, &ctx->launches));
        CK(launch_scatter_scaled(ctx->d_s_out, ctx->d_P, m, 1.0 / gp.wscale, ctx->d_u0, ctx->st, &ctx->launches));
    }
    CK(cudaMemsetAsync(ctx->d_vf, 0, ctx->d4 * sizeof(float), ctx->st));
    return DUHL_OK;
}
static duhl_status tpa_end(duhl_ctx* ctx, int64_t m) {
    ProfScope ps(ctx, ctx->st, 6, (double)m * (4.0 * ctx->d4 + 24.0) + 24.0 * ctx->d4);
    CK(launch_tpa_resync(ctx->pool, ctx->ld_dev, ctx->d_P_slot, ctx->d_P, ctx->d_alpha, ctx->d_a0t, m, ctx->d_v0t,
                         ctx->d_vt, ctx->d4, ctx->st, &ctx->launches));
    return DUHL_OK;
}

// The epoch on the working set.  Staging copies planned by the last select are
// enqueued after the pass-0 launch when they overlap it (the kernel waits on the
// progress counter per block), else before it (the compute stream waits).
static duhl_status scd_passes(duhl_ctx* ctx, int passes, uint64_t seed, int64_t round) {
    const int64_t m = ctx->m_cur;
    // staging that overlaps the epoch is enqueued after the pass-0 launch: the host enqueue of
    // per-column copies overlaps it, and a gather launch finds the cooperative SCD grid resident
    // on its SMs (one CTA per SM, the whole register file), so its CTAs can only go to the SMs
    // the grid leaves (unit_a_ctas) -- never in the way of the grid it feeds
    if (!ctx->overlap) TRY(issue_staging(ctx));
    const bool staged = ctx->overlap && !ctx->copy_plan.empty();  // pass 0 consumes columns as they land
    if (ctx->tpa) TRY(tpa_begin(ctx, m));
    for (int pass = 0; pass < passes; ++pass) {
        CK(launch_perm_order(ctx->d_P, ctx->d_P_slot, ctx->d_P_batch, m, seed, round, pass,
                             ctx->d_order_j, ctx->d_order_slot, ctx->d_order_batch, ctx->d_order_a,
                             ctx->d_order_inv, ctx->d_order_y, ctx->d_alpha, ctx->d_norms,
                             ctx->model == DUHL_SVM_DUAL ? ctx->d_y : nullptr, ctx->st, &ctx->launches,
                             ridge_ld(ctx)));
        TRY(scd_launch(ctx, m, staged && pass == 0));
        if (pass == 0) TRY(issue_staging(ctx));  // no-op unless overlapping: host enqueue overlaps pass 0
    }
    if (ctx->tpa) TRY(tpa_end(ctx, m));
    return DUHL_OK;
}

duhl_status duhl_scd_epoch(duhl_ctx* ctx, int passes, uint64_t seed, int64_t round, const int64_t* perm,
                           int64_t perm_len) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    if (ctx->m_cur == 0) return fail(ctx, DUHL_E_INVALID, "no working set: call duhl_select first");
    if (perm) {
        TRY(ensure_host_P(ctx));
        if (perm_len < 0 || perm_len > (int64_t)ctx->P.size()) return fail(ctx, DUHL_E_INVALID, "perm_len");
        std::vector<char> seen(ctx->n, 0);
        std::vector<int> slots(perm_len);
        std::vector<unsigned> batches(perm_len);
        for (int64_t t = 0; t < perm_len; ++t) {
            int64_t j = perm[t];
            if (j < 0 || j >= ctx->n || !ctx->inP[j] || seen[j] || ctx->col_slot[j] < 0)
                return fail(ctx, DUHL_E_INVALID, "perm entries must be distinct resident members of P");
            seen[j] = 1;
            slots[t] = ctx->col_slot[j];
            batches[t] = ctx->slot_batch[slots[t]];
        }
        if (!ctx->overlap) TRY(issue_staging(ctx));
        if (ctx->csc) {
            double by = 0.0;
            for (int64_t t = 0; t < perm_len; ++t)
                by += 8.0 * (double)(ctx->h_colptr[perm[t] + 1] - ctx->h_colptr[perm[t]]) + 24.0;
            ctx->csc_pass_bytes = by;
        }
        CK(cudaMemcpyAsync(ctx->d_order_j, perm, perm_len * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_order_slot, slots.data(), perm_len * sizeof(int), cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_order_batch, batches.data(), perm_len * sizeof(unsigned),
                           cudaMemcpyHostToDevice, ctx->st));
        CK(launch_perm_order(nullptr, nullptr, nullptr, perm_len, 0, 0, 0, ctx->d_order_j, ctx->d_order_slot,
                             ctx->d_order_batch, ctx->d_order_a, ctx->d_order_inv, ctx->d_order_y,
                             ctx->d_alpha, ctx->d_norms, ctx->model == DUHL_SVM_DUAL ? ctx->d_y : nullptr,
                             ctx->st, &ctx->launches, ridge_ld(ctx)));
        if (ctx->tpa) TRY(tpa_begin(ctx, ctx->m_cur));
        TRY(scd_launch(ctx, perm_len));
        if (ctx->tpa) TRY(tpa_end(ctx, ctx->m_cur));
        TRY(issue_staging(ctx));
        TRY(finalize_staging(ctx));
        return check_flag(ctx, "duhl_scd_epoch");
    }
    if (passes < 1) return fail(ctx, DUHL_E_INVALID, "passes < 1");
    TRY(scd_passes(ctx, passes, seed, round));
    TRY(finalize_staging(ctx));
    return check_flag(ctx, "duhl_scd_epoch");
}

static duhl_status certificate(duhl_ctx* ctx, double* gap, double* primal, double* dual) {
    CK(cudaMemsetAsync(ctx->d_sums, 0, 8 * sizeof(double), ctx->st));
    int64_t resident = 0;
    for (int64_t s = 0; s < ctx->S; ++s) resident += ctx->slot_col[s] >= 0;
    const int64_t nonres = ctx->csc ? 0 : ctx->n - resident;
    const int64_t kh = ctx->hua ? (int64_t)std::llround(ctx->cert_share * (double)nonres) : 0;
    ctx->zc_bytes += (nonres - kh) * ctx->ld_dev * (int64_t)sizeof(float);
    if (kh > 0) {  // host threads take the last kh non-resident columns (unit A on the host, duhl.h)
        std::vector<int64_t> gcols;
        gcols.reserve(ctx->n - kh);
        int64_t seen = 0, hc = 0;
        for (int64_t i = 0; i < ctx->n; ++i) {
            if (ctx->col_slot[i] < 0 && seen++ >= nonres - kh) ctx->h_hcols[hc++] = i;
            else gcols.push_back(i);
        }
        const int64_t kg = (int64_t)gcols.size();
        CK(d2h_copy(ctx, ctx->h_vt, ctx->d_vt, ctx->d4 * sizeof(double), ctx->st));
        CK(cudaEventRecord(ctx->ev_hvt, ctx->st));
        hua_post(ctx->hua, ctx->h_store, ctx->ld_host, ctx->d4, ctx->h_hcols, kh, ctx->h_vt, wscale(ctx),
                 ctx->ev_hvt, ctx->h_hs);
        CK(cudaMemcpyAsync(ctx->d_hcols, ctx->h_hcols, kh * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        if (kg > 0) {
            CK(cudaMemcpyAsync(ctx->d_cols, gcols.data(), kg * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
            CK(cudaEventRecord(ctx->ev_g0, ctx->st));
            TRY(run_gaps(ctx, ctx->d_cols, kg, nullptr, nullptr, ctx->d_sums, /*write_z=*/true));
            CK(cudaEventRecord(ctx->ev_g1, ctx->st));
        }
        const double host_s = hua_wait(ctx->hua);
        CK(cudaMemcpyAsync(ctx->d_hs, ctx->h_hs, kh * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
        GapParams hp = gap_params(ctx, ctx->d_hcols, kh);
        hp.s_acc = ctx->d_hs;
        hp.sums = ctx->d_sums;
        hp.z = ctx->d_z;  // R25: the certificate's gaps refresh the gap memory
        CK(launch_gap_finalize(hp, ctx->st, &ctx->launches));
        CK(cudaStreamSynchronize(ctx->st));  // gcols is pageable and local
        float gms = 0.0f;  // balance the next certificate: both units end together
        if (kg > 0 && host_s > 0.0 && cudaEventElapsedTime(&gms, ctx->ev_g0, ctx->ev_g1) == cudaSuccess &&
            gms > 0.0f && nonres > kh) {
            const double rh = (double)kh / host_s, rg = (double)(nonres - kh) / (1e-3 * gms);
            ctx->cert_share = std::min(0.95, std::max(0.05, 0.5 * ctx->cert_share + 0.5 * rh / (rh + rg)));
        }
        ctx->hua_cols += kh;
    } else {
        TRY(run_gaps(ctx, nullptr, ctx->n, nullptr, nullptr, ctx->d_sums, /*write_z=*/true));
    }
    TRY(allreduce(ctx, ctx->d_sums, 3));           // per-column sums over the shards
    TRY(allreduce(ctx, ctx->d_sums + 3, 1, ncclMax));
    CK(launch_vec_sums(ctx->d_vt, ctx->model != DUHL_SVM_DUAL ? ctx->d_b : nullptr, ctx->d4, ctx->d_sums + 4,
                       ctx->st, &ctx->launches));     // v is replicated: no reduction
    double h[8];
    CK(d2h_copy(ctx, h, ctx->d_sums, 8 * sizeof(double), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    TRY(check_flag(ctx, "certificate"));
    const double dd = (double)ctx->d, nn = (double)ctx->n_glob, lam = ctx->lambda;
    const double G = h[0], aux = h[1], asum = h[2], vv = h[4], vb = h[5];
    double amax;
    std::memcpy(&amax, &h[3], sizeof(double));
    double O, D;
    if (ctx->model == DUHL_LASSO) {
        // w = v~; O = ||w||^2/(2d) + lambda ||alpha||_1;  D = -(u^T b + (d/2)||u||^2) - sum B[|a^T u| - lambda]_+
        O = vv / (2.0 * dd) + lam * asum;
        D = -(vb / dd + 0.5 * vv / dd) - aux;
    } else if (ctx->model == DUHL_ELASTIC_NET) {
        // O = ||w||^2/(2d) + lambda sum (eta/2 a^2 + (1-eta)|a|);  D = -(u^T b + (d/2)||u||^2) - sum g*(a^T u)
        O = vv / (2.0 * dd) + lam * asum;
        D = -(vb / dd + 0.5 * vv / dd) - aux;
    } else if (ctx->model == DUHL_RIDGE) {
        // O = ||w||^2/(2d) + (lambda/2)||alpha||^2;  D = -(u^T b + (d/2)||u||^2) - sum (a^T u)^2/(2 lambda)
        O = vv / (2.0 * dd) + 0.5 * lam * asum;
        D = -(vb / dd + 0.5 * vv / dd) - aux;
    } else {
        // O = -(1/n) sum y a + ||v||^2/(2 lambda n^2);  D = -[(1/n) sum hinge + (lambda/2)||w||^2]
        O = -asum / nn + vv / (2.0 * lam * nn * nn);
        D = -(aux / nn + 0.5 * vv / (lam * nn * nn));
    }
    if (gap) *gap = G;
    if (primal) *primal = O;
    if (dual) *dual = D;
    if (!std::isfinite(G) || !std::isfinite(O)) return fail(ctx, DUHL_E_NUMERIC, "non-finite certificate");
    if (ctx->model == DUHL_LASSO && amax > ctx->B * (1.0 + 1e-12))
        return fail(ctx, DUHL_E_BOUND, "max |alpha_i| exceeds the Lipschitzing bound B (P:848)");
    return DUHL_OK;
}

duhl_status duhl_duality_gap(duhl_ctx* ctx, double* gap, double* primal, double* dual) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    return certificate(ctx, gap, primal, dual);
}

// CoCoA-style aggregation after the local epoch (R16):
// dv = sum over ranks of (v_local - v0); gamma = exact line search on [0, 1] of
// the global objective along (alpha_old + gamma dalpha, v0 + gamma dv), or 1;
// then v = v0 + gamma dv and alpha_P = alpha_old + gamma dalpha.
//   SVM: closed form from sum y dalpha (allreduced), v0^T dv, ||dv||^2
//   Lasso: the right derivative D(g) = (v~0^T dv + g ||dv||^2)/d
//                  + lambda sum dalpha sgn+(alpha_old + g dalpha) is increasing:
//                  bracket its sign change on 64-point grids (one allreduce each),
//                  then solve the linear piece inside the final bracket.
static duhl_status aggregate(duhl_ctx* ctx, double* gamma_out) {
    const int64_t m = ctx->m_cur;
    const double dd = (double)ctx->d, nn = (double)ctx->n_glob, lam = ctx->lambda;
    CK(launch_delta_v(ctx->d_vt, ctx->d_vsnap, ctx->d4, ctx->d_dv, ctx->d_ls + 64, ctx->st, &ctx->launches));
    TRY(allreduce(ctx, ctx->d_dv, (size_t)ctx->d4));
    CK(cudaMemsetAsync(ctx->d_ls, 0, 8 * sizeof(double), ctx->st));
    CK(launch_vec_sums(ctx->d_dv, ctx->d_vsnap, ctx->d4, ctx->d_ls, ctx->st, &ctx->launches));  // |dv|^2, v0.dv
    double gamma = 1.0;
    if (ctx->cfg.linesearch) {
        if (ctx->model == DUHL_RIDGE) {  // quadratic in gamma: closed form
            CK(launch_ridge_sums(ctx->d_alpha, ctx->d_P, ctx->d_aold, m, ctx->d_ls + 2, ctx->st, &ctx->launches));
            TRY(allreduce(ctx, ctx->d_ls + 2, 2));
            double h[4];
            CK(d2h_copy(ctx, h, ctx->d_ls, 4 * sizeof(double), ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            const double dvdv = h[0], vdv = h[1], ada = h[2], dada = h[3];
            const double den = dvdv / dd + lam * dada;
            if (den > 0.0) {
                gamma = -(vdv / dd + lam * ada) / den;
                gamma = gamma < 0.0 ? 0.0 : (gamma > 1.0 ? 1.0 : gamma);
            }
        } else if (ctx->model == DUHL_SVM_DUAL) {
            CK(launch_ydalpha(ctx->d_alpha, ctx->d_y, ctx->d_P, ctx->d_aold, m, ctx->d_ls + 2, ctx->st,
                              &ctx->launches));
            TRY(allreduce(ctx, ctx->d_ls + 2, 1));
            double h[3];
            CK(d2h_copy(ctx, h, ctx->d_ls, 3 * sizeof(double), ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            const double dvdv = h[0], vdv = h[1], yda = h[2], ln2 = lam * nn * nn;
            if (dvdv > 0.0) {
                gamma = (yda / nn - vdv / ln2) / (dvdv / ln2);
                gamma = gamma < 0.0 ? 0.0 : (gamma > 1.0 ? 1.0 : gamma);
            }
        } else {  // Lasso (l1 = 1, l2 = 0) and elastic net (l1 = 1 - eta, l2 = eta): walk the breakpoints
            const bool en = ctx->model == DUHL_ELASTIC_NET;
            const double l1 = en ? 1.0 - ctx->cfg.eta : 1.0, l2 = en ? ctx->cfg.eta : 0.0;
            if (en) {
                CK(launch_ridge_sums(ctx->d_alpha, ctx->d_P, ctx->d_aold, m, ctx->d_ls + 2, ctx->st, &ctx->launches));
                TRY(allreduce(ctx, ctx->d_ls + 2, 2));
            }
            double h[4];
            CK(d2h_copy(ctx, h, ctx->d_ls, 4 * sizeof(double), ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            const double dvdv = h[0], vdv = h[1], ada = en ? h[2] : 0.0, dada = en ? h[3] : 0.0;
            auto Dfun = [&](double g, double S) { return (vdv + g * dvdv) / dd + lam * (l1 * S + l2 * (ada + g * dada)); };
            double lo = 0.0, hi = 1.0, gam[64], S[64];
            bool done = false;
            for (int it = 0; it < 5 && !done; ++it) {
                const int ng = 64;
                for (int q = 0; q < ng; ++q) gam[q] = it == 0 ? (double)q / (ng - 1) : lo + (hi - lo) * (q + 1) / ng;
                if (it == 4) { gam[0] = 0.5 * (lo + hi); }  // final: the pattern inside the bracket
                const int nq = it == 4 ? 1 : ng;
                CK(cudaMemcpyAsync(ctx->d_ls + 128, gam, nq * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
                CK(cudaMemsetAsync(ctx->d_ls + 192, 0, nq * sizeof(double), ctx->st));
                CK(launch_lasso_dgrid(ctx->d_alpha, ctx->d_P, ctx->d_aold, m, ctx->d_ls + 128, nq, ctx->d_ls + 192,
                                      ctx->st, &ctx->launches));
                TRY(allreduce(ctx, ctx->d_ls + 192, (size_t)nq));
                CK(d2h_copy(ctx, S, ctx->d_ls + 192, nq * sizeof(double), ctx->st));
                CK(cudaStreamSynchronize(ctx->st));
                if (it == 0) {
                    if (Dfun(0.0, S[0]) >= 0.0) { gamma = 0.0; done = true; break; }
                    if (Dfun(1.0, S[ng - 1]) < 0.0) { gamma = 1.0; done = true; break; }
                    int q = 1;
                    while (q < ng && Dfun(gam[q], S[q]) < 0.0) ++q;
                    lo = gam[q - 1];
                    hi = gam[q];
                } else if (it < 4) {
                    int q = 0;
                    while (q < ng && Dfun(gam[q], S[q]) < 0.0) ++q;
                    if (q > 0) lo = gam[q - 1];
                    hi = gam[q < ng ? q : ng - 1];
                } else {
                    const double den = dvdv / dd + lam * l2 * dada;
                    const double x = den > 0.0 ? -(vdv / dd + lam * (l1 * S[0] + l2 * ada)) / den : hi;
                    gamma = x < lo ? lo : (x > hi ? hi : x);
                    done = true;
                }
            }
        }
    }
    CK(launch_apply_gamma(ctx->d_vt, ctx->d_vsnap, ctx->d_dv, ctx->d4, ctx->d_alpha, ctx->d_P, ctx->d_aold, m,
                          gamma, ctx->st, &ctx->launches));
    if (gamma_out) *gamma_out = gamma;
    return DUHL_OK;
}

// Unit-A refresh of the cursor chunk (columns in d_cols) against the v snapshot,
// on its own stream beside the staging copies; PCIe-bound (zero-copy reads) for
// non-resident columns.
// Unit-A refresh of the cursor chunk (columns in d_cols) against the v snapshot,
// on its own stream beside the staging copies; PCIe-bound (zero-copy reads) for
// non-resident columns.
static duhl_status refresh_launch(duhl_ctx* ctx, int64_t kref) {
    if (kref <= 0) return DUHL_OK;
    CK(cudaStreamWaitEvent(ctx->rst, ctx->ev_snap, 0));
    TRY(run_gaps(ctx, ctx->d_cols, kref, nullptr, nullptr, nullptr, true, ctx->d_vsnap, ctx->rst,
                 ctx->d_s_acc2, kGapTileRows, ctx->unit_a_ctas));
    CK(cudaEventRecord(ctx->ev_ref, ctx->rst));
    return DUHL_OK;
}

static duhl_status round_impl(duhl_ctx* ctx, int64_t t, int passes, duhl_policy policy, int certify,
                              duhl_round_record* rec) {
    auto t0 = std::chrono::steady_clock::now();
    const int64_t n = ctx->n;
    int64_t kref = (int64_t)std::ceil(ctx->cfg.refresh_fraction * (double)n - 1e-9);
    kref = std::max<int64_t>(0, std::min(n, kref));
    int64_t swaps = 0;
    static const bool htrace = std::getenv("DUHL_ROUND_TRACE") != nullptr;  // developer timing
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto tsel = now();
    // Copies overlap the epoch only when unit A is idle: with a refresh, PCIe is
    // shared by the staging copies and the zero-copy refresh reads, so both run
    // first, side by side, and the epoch follows at full HBM rate.
    TRY(finalize_staging(ctx));
    // With host threads in unit A, PCIe carries (almost) only the staging: the copies overlap the
    // epoch and the threads take every non-resident refresh column.  DUHL_NO_HOST_OVERLAP=1
    // restores copies-first.
    static const bool no_host_overlap = std::getenv("DUHL_NO_HOST_OVERLAP") != nullptr;
    const bool host_overlap = ctx->hua && !no_host_overlap;
    ctx->overlap = ctx->write_value != nullptr && (kref == 0 || host_overlap) && !ctx->tpa;
    TRY(select_impl(ctx, policy, ctx->m_cfg, t, &swaps));                  // Alg. 2 l.3-4
    {   // rho_{t,P} (Eq. 6) on the gap memory the selection used
        CK(cudaMemsetAsync(ctx->d_rho, 0, 2 * sizeof(double), ctx->st));
        CK(launch_gather_f64(ctx->d_z, ctx->d_P, ctx->m_cur, ctx->d_gap_out, ctx->st, &ctx->launches));
        CK(launch_sum(ctx->d_gap_out, ctx->m_cur, ctx->d_rho, ctx->st, &ctx->launches));
        CK(launch_sum(ctx->d_z, n, ctx->d_rho + 1, ctx->st, &ctx->launches));
    }
    auto tstaged = now();
    // pinned per-context buffers: no per-round allocation, and the uploads are truly asynchronous
    // (C5 refreshes 1 M columns a round: two 8-MB pageable copies and a zero-filled vector cost
    // ~6 ms of host time per 17-ms round before)
    if (kref >= kPinnedRefreshCols && !ctx->h_ref_idx &&
        (cudaHostAlloc((void**)&ctx->h_ref_idx, n * sizeof(int64_t), 0) != cudaSuccess ||
         cudaHostAlloc((void**)&ctx->h_ref_smp, n * sizeof(int64_t), 0) != cudaSuccess))
        return fail(ctx, DUHL_E_NOMEM, "pinned refresh buffers");
    if (kref < kPinnedRefreshCols && (int64_t)ctx->ref_idx_v.size() < kref) {
        ctx->ref_idx_v.resize(kref);
        ctx->ref_smp_v.resize(kref);
    }
    int64_t* idx = kref >= kPinnedRefreshCols ? ctx->h_ref_idx : ctx->ref_idx_v.data();
    int64_t* smp = kref >= kPinnedRefreshCols ? ctx->h_ref_smp : ctx->ref_smp_v.data();
    int64_t nsmp = 0;
    int64_t kg = kref, kh = 0, nonres = 0;  // refresh columns on the GPU / host threads; non-resident
    bool heavy_round = false;             // the threads took every non-resident column (see below)
    const bool agg = ctx->nranks > 1 || ctx->cfg.linesearch;
    if (agg) {  // round-start state for the aggregation: v0 and alpha_P
        CK(cudaMemcpyAsync(ctx->d_vsnap, ctx->d_vt, ctx->d4 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
        CK(launch_gather_f64(ctx->d_alpha, ctx->d_P, ctx->m_cur, ctx->d_aold, ctx->st,
                             &ctx->launches));
    }
    if (kref > 0) {  // unit A (l.7-10): gaps at alpha^(t) on its own stream, beside the
                     // staging copies and (unit_a_ctas > 0) the epoch on the remaining SMs;
                     // otherwise the epoch waits for it (it would hold the SMs the
                     // cooperative launch needs)
        int64_t host_cols = 0;
        {   // the cursor's range (no modulo per entry); non-resident count only with a budget
            int64_t c = ctx->cursor;
            for (int64_t q = 0; q < kref; ++q) {
                idx[q] = c;
                if (++c == n) c = 0;
            }
            if (ctx->cfg.hbm_budget_bytes != 0)
                for (int64_t q = 0; q < kref; ++q) host_cols += ctx->col_slot[idx[q]] < 0;
        }
        if (ctx->P_host_valid) {  // the refreshed columns outside P: a systematic sample of fresh gaps
            nsmp = 0;
            for (int64_t q = 0; q < kref; ++q)
                if (!ctx->inP[idx[q]]) smp[nsmp++] = idx[q];
        }
        ctx->cursor = (ctx->cursor + kref) % n;
        nonres = host_cols;
        // the host threads take the last kh of the non-resident columns; the GPU the rest
        // (a round that stages more than m/2 columns leaves PCIe to the staging: the threads take all)
        static const bool heavy_host = std::getenv("DUHL_NO_HEAVY_HOST_REFRESH") == nullptr;
        heavy_round = heavy_host && swaps * 2 > ctx->m_cur;
        kh = ctx->hua ? ((ctx->overlap || heavy_round) ? host_cols
                                                       : (int64_t)std::llround(ctx->hua_share * (double)host_cols))
                      : 0;
        if (kh > 0) {
            int64_t g = 0, hcount = 0, seen = 0;
            for (int64_t q = 0; q < kref; ++q) {
                const bool nr = ctx->col_slot[idx[q]] < 0;
                if (nr && seen++ >= host_cols - kh) ctx->h_hcols[hcount++] = idx[q];
                else idx[g++] = idx[q];
            }
            kg = g;
        }
        ctx->zc_bytes += (host_cols - kh) * ctx->ld_dev * (int64_t)sizeof(float);
        if (kg > 0)
            CK(cudaMemcpyAsync(ctx->d_cols, idx, kg * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        if (!agg)
            CK(cudaMemcpyAsync(ctx->d_vsnap, ctx->d_vt, ctx->d4 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaEventRecord(ctx->ev_snap, ctx->st));
        if (kh > 0) {  // v~ snapshot to the host threads; their columns to the device for the finalize
            CK(d2h_copy(ctx, ctx->h_vt, ctx->d_vsnap, ctx->d4 * sizeof(double), ctx->st));
            CK(cudaEventRecord(ctx->ev_hvt, ctx->st));
            CK(cudaMemcpyAsync(ctx->d_hcols, ctx->h_hcols, kh * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
            hua_post(ctx->hua, ctx->h_store, ctx->ld_host, ctx->d4, ctx->h_hcols, kh, ctx->h_vt, wscale(ctx),
                     ctx->ev_hvt, ctx->h_hs);
            CK(cudaEventRecord(ctx->ev_g0, ctx->st));
        }
        TRY(refresh_launch(ctx, kg));
        if (kh > 0) {
            if (kg > 0) CK(cudaEventRecord(ctx->ev_g1, ctx->rst));
            else CK(cudaEventRecord(ctx->ev_g1, ctx->st));
        }
        if (ctx->unit_a_ctas <= 0 && kg > 0) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_ref, 0));
    }
    auto tlaunch = now();
    TRY(scd_passes(ctx, passes, ctx->cfg.seed, t));                        // l.6, l.11
    if (kh > 0) CK(cudaEventRecord(ctx->ev_c1, ctx->cst));  // the staging copies are all enqueued
    TRY(finalize_staging(ctx));                                            // staged columns -> table
    auto tscd = now();
    auto tref = tscd;
    if (htrace) {  // developer timing: when the epoch and the unit-A refresh end (host view)
        CK(cudaStreamSynchronize(ctx->st));
        tscd = now();
        CK(cudaStreamSynchronize(ctx->rst));
        tref = now();
    }
    if (kg > 0 && ctx->unit_a_ctas > 0) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_ref, 0));  // join unit A
    double host_s = 0.0;
    if (kh > 0) {  // join the host threads: their dots -> gap_i at the round-start alpha of columns
                   // outside P (columns of P are refreshed after the epoch below, R9)
        host_s = hua_wait(ctx->hua);
        CK(cudaMemcpyAsync(ctx->d_hs, ctx->h_hs, kh * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
        GapParams hp = gap_params(ctx, ctx->d_hcols, kh);
        hp.s_acc = ctx->d_hs;
        CK(launch_gap_finalize(hp, ctx->st, &ctx->launches));
        ctx->hua_cols += kh;
    }
    double gamma = 1.0;
    if (agg) TRY(aggregate(ctx, &gamma));                                   // l.11 across ranks
    const int64_t m = ctx->m_cur;                                          // z_P at alpha^(t+1) (R9)
    TRY(run_gaps(ctx, ctx->d_P, m, nullptr, nullptr, nullptr));
    double cg = -1.0;
    if (certify) TRY(certificate(ctx, &cg, nullptr, nullptr));
    CK(cudaMemsetAsync(ctx->d_sums + 6, 0, sizeof(double), ctx->st));
    CK(launch_sum(ctx->d_z, n, ctx->d_sums + 6, ctx->st, &ctx->launches));
    TRY(allreduce(ctx, ctx->d_sums + 6, 1));
    // Gap estimate for the adaptive certificates: z_P is fresh (R9) and the refreshed columns
    // outside P are a systematic sample of fresh gaps of the other n - m columns, so
    //   est = sum_P z + (n - m) mean_sample z   (every term at most one round old),
    // where the plain sum of z mixes in gaps up to 1/f rounds stale.
    double est[4] = {0.0, 0.0, 0.0, 0.0};
    const bool have_est = nsmp > 0;
    if (have_est) {
        CK(cudaMemsetAsync(ctx->d_est, 0, 4 * sizeof(double), ctx->st));
        CK(launch_gather_f64(ctx->d_z, ctx->d_P, m, ctx->d_gap_out, ctx->st, &ctx->launches));
        CK(launch_sum(ctx->d_gap_out, m, ctx->d_est, ctx->st, &ctx->launches));
        CK(cudaMemcpyAsync(ctx->d_smp, smp, nsmp * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
        CK(launch_gather_f64(ctx->d_z, ctx->d_smp, nsmp, ctx->d_s_out, ctx->st, &ctx->launches));
        CK(launch_sum(ctx->d_s_out, nsmp, ctx->d_est + 1, ctx->st, &ctx->launches));
        const double cnt[2] = {(double)nsmp, (double)(n - m)};
        CK(cudaMemcpyAsync(ctx->d_est + 2, cnt, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
    }
    if (ctx->group || ctx->comm) {  // every rank takes part (a rank without a sample adds zeros)
        if (!have_est) CK(cudaMemsetAsync(ctx->d_est, 0, 4 * sizeof(double), ctx->st));
        TRY(allreduce(ctx, ctx->d_est, 4));
    }
    if (have_est || ctx->group || ctx->comm) CK(d2h_copy(ctx, est, ctx->d_est, 4 * sizeof(double), ctx->st));
    double zs = 0.0, rs[2] = {0.0, 0.0};
    CK(d2h_copy(ctx, &zs, ctx->d_sums + 6, sizeof(double), ctx->st));
    CK(d2h_copy(ctx, rs, ctx->d_rho, 2 * sizeof(double), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    TRY(check_flag(ctx, "duhl_round"));
    harvest(ctx);
    if (htrace) {
        auto tend = now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "round %lld: select+stage %.2f ms, refresh-launch %.2f, epoch end %.2f, refresh end "
                     "%.2f, tail %.2f, total %.2f\n", (long long)t, ms(tsel, tstaged), ms(tstaged, tlaunch),
                     ms(tsel, tscd), ms(tsel, tref), ms(tref, tend), ms(tsel, tend));
    }
    if (rec) {
        rec->round = t;
        rec->swaps = swaps;
        rec->refreshed = kref;
        rec->cert_gap = cg;
        rec->z_sum = zs;
        rec->gamma = gamma;
        rec->time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        rec->rho = (rs[1] > 0.0 && m > 0) ? (rs[0] / (double)m) / (rs[1] / (double)n) : 1.0;
        rec->gap_est = est[2] > 0.0 ? est[0] + est[3] * est[1] / est[2] : -1.0;
    }
    if (kh > 0 && ctx->cfg.unit_a_host_share < 0.0 && !heavy_round) {  // (a forced share measures no balance)
        // balance: the host's columns take as long as what PCIe carries this round (staging
        // copies + the GPU's zero-copy columns): kh = (swaps + nonres) r_h / (r_h + r_p)
        float gms = 0.0f, cms = 0.0f;
        const int64_t kgn = nonres - kh;  // non-resident columns the GPU read over PCIe
        if (kgn == 0 || cudaEventElapsedTime(&gms, ctx->ev_g0, ctx->ev_g1) != cudaSuccess) gms = 0.0f;
        if (swaps == 0 || cudaEventElapsedTime(&cms, ctx->ev_g0, ctx->ev_c1) != cudaSuccess) cms = 0.0f;
        const double tp = 1e-3 * std::max(gms, cms);
        if (host_s > 0.0 && tp > 0.0 && swaps + kgn > 0) {
            const double rh = (double)kh / host_s, rp = (double)(swaps + kgn) / tp;
            const double target = std::min(1.0, (double)(swaps + nonres) * rh / (rh + rp) / (double)nonres);
            ctx->hua_share = std::min(1.0, std::max(0.05, 0.75 * ctx->hua_share + 0.25 * target));
        }
    }
    return DUHL_OK;
}

duhl_status duhl_round(duhl_ctx* ctx, int64_t round, int passes, duhl_policy policy, int certify,
                       duhl_round_record* rec) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    if (passes < 1 || round < 0) return fail(ctx, DUHL_E_INVALID, "passes/round");
    return round_impl(ctx, round, passes, policy, certify, rec);
}

duhl_status duhl_solve(duhl_ctx* ctx, double eps, int64_t max_rounds, int passes, duhl_policy policy,
                       duhl_round_record* trace, int64_t trace_cap, int64_t* rounds_out, double* gap_out) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    if (passes < 1 || max_rounds < 0) return fail(ctx, DUHL_E_INVALID, "passes/max_rounds");
    auto t0 = std::chrono::steady_clock::now();
    double gap = INFINITY;
    duhl_status st = DUHL_E_NOT_CONVERGED;
    int64_t t = 0, last_cert = -1, backoff = 1;
    double zs = INFINITY;
    // Adaptive certificates: the gap memory's sum z_s is a time-delayed estimate of the gap
    // (P:307-313); a failed certificate calibrates it -- the next one waits until
    // z_s * ratio <= eps, ratio = the largest certified gap / z_s seen (>= 1), and at least
    // `backoff` rounds (doubling after each failure).
    double ratio = 1.0;
    auto want = [&](double z) { return ctx->cfg.cert_adaptive && z * ratio <= eps && (t - last_cert) >= backoff; };
    auto failed = [&](double g, double z) {
        if (z > 0.0 && g / z > ratio) ratio = g / z;
        backoff *= 2;
    };
    for (t = 0; t < max_rounds; ++t) {
        // certify on the fixed schedule, or (adaptive) when the calibrated estimate says we may be done
        bool sched = (t + 1) % ctx->cfg.cert_every == 0;
        bool adapt = want(zs);
        duhl_round_record r{};
        TRY(round_impl(ctx, t, passes, policy, (sched || adapt) ? 1 : 0, &r));
        zs = r.gap_est >= 0.0 ? r.gap_est : r.z_sum;  // the sampled estimate where a refresh ran
        if (r.cert_gap >= 0.0) {
            gap = r.cert_gap;
            if (adapt && !sched && gap > eps) failed(gap, zs);  // both at the end of round t
            last_cert = t;
        } else if (want(zs)) {
            // the estimate crossed eps during this round: certify now rather than next round
            TRY(certificate(ctx, &gap, nullptr, nullptr));
            r.cert_gap = gap;
            if (gap > eps) failed(gap, zs);
            last_cert = t;
        }
        r.time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (trace && t < trace_cap) trace[t] = r;
        if (ctx->trace_cb) ctx->trace_cb(&r, ctx->trace_user);
        if (r.cert_gap >= 0.0 && gap <= eps) { st = DUHL_OK; ++t; break; }
    }
    if (rounds_out) *rounds_out = t;
    if (gap_out) *gap_out = gap;
    if (st == DUHL_E_NOT_CONVERGED) ctx->err = "max_rounds reached before the certified gap <= eps";
    return st;
}

duhl_status duhl_get_state(duhl_ctx* ctx, double* alpha_out, double* v_out, double* z_out) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    if (alpha_out) CK(d2h_copy(ctx, alpha_out, ctx->d_alpha, ctx->n * sizeof(double), ctx->st));
    if (v_out) CK(d2h_copy(ctx, v_out, ctx->d_vt, ctx->d * sizeof(double), ctx->st));
    if (z_out) CK(d2h_copy(ctx, z_out, ctx->d_z, ctx->n * sizeof(double), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return DUHL_OK;
}

duhl_status duhl_set_state(duhl_ctx* ctx, const double* alpha) {
    if (!ctx || !alpha) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    std::vector<double> y;
    if (ctx->model == DUHL_SVM_DUAL) {
        y.resize(ctx->n);
        CK(cudaMemcpy(y.data(), ctx->d_y, ctx->n * sizeof(double), cudaMemcpyDeviceToHost));
    }
    for (int64_t i = 0; i < ctx->n; ++i) {
        if (!std::isfinite(alpha[i])) return fail(ctx, DUHL_E_INVALID, "non-finite alpha");
        if (ctx->model == DUHL_SVM_DUAL && (y[i] * alpha[i] < 0.0 || y[i] * alpha[i] > 1.0))
            return fail(ctx, DUHL_E_INVALID, "SVM alpha outside the box y_i alpha_i in [0,1]");
    }
    CK(cudaMemcpyAsync(ctx->d_alpha, alpha, ctx->n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
    // sharded (collective): v = sum_k A_k alpha_k - b, i.e. each rank its own columns, b
    // subtracted on rank 0 only, then summed over the ranks
    const bool sub_b = ctx->model != DUHL_SVM_DUAL && ctx->rank == 0;
    CK(launch_matvec(colsrc(ctx), ctx->d_alpha, ctx->csc ? 0 : ctx->n, ctx->d, ctx->d4,
                     sub_b ? ctx->d_b : nullptr, ctx->d_vt, ctx->st, &ctx->launches));
    if (ctx->csc) CK(launch_csc_matvec(cscmat(ctx), ctx->d_alpha, ctx->n, ctx->d_vt, ctx->st, &ctx->launches));
    TRY(allreduce(ctx, ctx->d_vt, (size_t)ctx->d4));
    TRY(run_gaps(ctx, nullptr, ctx->n, nullptr, nullptr, nullptr));
    CK(cudaStreamSynchronize(ctx->st));
    return check_flag(ctx, "duhl_set_state");
}

duhl_status duhl_comm_unique_id(void* id_out) {
    if (!id_out) return DUHL_E_INVALID;
    NcclApi* api = nccl_api();
    if (!api) return DUHL_E_NCCL;
    ncclUniqueId id;
    if (api->getUniqueId(&id) != ncclSuccess) return DUHL_E_NCCL;
    std::memcpy(id_out, &id, sizeof(id));
    return DUHL_OK;
}

duhl_status duhl_comm_init(duhl_ctx* ctx, const void* id, int nranks, int rank) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    NcclApi* api = nccl_api();
    if (!api) return fail(ctx, DUHL_E_NCCL, "libnccl.so.2 not found");
    if (ctx->comm || ctx->group) return fail(ctx, DUHL_E_INVALID, "communicator already initialised");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = api->commInitRank(&ctx->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        ctx->comm = nullptr;
        return fail(ctx, DUHL_E_NCCL, std::string("ncclCommInitRank: ") + api->getErrorString(r));
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    // sigma' = 1 local subproblems summed with weight 1 can diverge; the exact line search on
    // gamma keeps every round monotone (R16), so it is on for K > 1
    if (nranks > 1) ctx->cfg.linesearch = 1;
    return DUHL_OK;
}

duhl_status duhl_group_create(int nranks, duhl_group** out) {
    if (!out) return DUHL_E_INVALID;
    *out = nullptr;
    if (nranks < 1 || nranks > 1024) return DUHL_E_INVALID;
    duhl_group* g = new duhl_group();
    g->n = nranks;
    g->slot.resize(nranks);
    *out = g;
    return DUHL_OK;
}

duhl_status duhl_group_destroy(duhl_group* g) {
    if (!g) return DUHL_E_INVALID;
    delete g;
    return DUHL_OK;
}

duhl_status duhl_comm_init_group(duhl_ctx* ctx, duhl_group* g, int rank) {
    if (!ctx || !g || rank < 0 || rank >= g->n) return DUHL_E_INVALID;
    if (ctx->comm || ctx->group) return fail(ctx, DUHL_E_INVALID, "communicator already initialised");
    ctx->group = g;
    ctx->nranks = g->n;
    ctx->rank = rank;
    if (g->n > 1) ctx->cfg.linesearch = 1;
    return DUHL_OK;
}

duhl_status duhl_set_trace_callback(duhl_ctx* ctx, duhl_trace_cb cb, void* user) {
    if (!ctx) return DUHL_E_INVALID;
    ctx->trace_cb = cb;
    ctx->trace_user = user;
    return DUHL_OK;
}

duhl_status duhl_get_working_set(duhl_ctx* ctx, int64_t* P_out, int64_t cap, int64_t* m_out) {
    if (!ctx) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    TRY(ensure_host_P(ctx));
    const int64_t m = (int64_t)ctx->P.size();
    if (m_out) *m_out = m;
    if (P_out) {
        if (cap < m) return fail(ctx, DUHL_E_INVALID, "P_out capacity smaller than |P|");
        std::memcpy(P_out, ctx->P.data(), m * sizeof(int64_t));
    }
    return DUHL_OK;
}

duhl_status duhl_get_stream(duhl_ctx* ctx, void** stream_out) {
    if (!ctx || !stream_out) return DUHL_E_INVALID;
    *stream_out = (void*)ctx->st;
    return DUHL_OK;
}

duhl_status duhl_get_kernel_stats(duhl_ctx* ctx, int kind, int64_t* launches, double* ms,
                                  double* bytes) {
    if (!ctx || kind < 0 || kind > 6) return DUHL_E_INVALID;
    CK(cudaSetDevice(ctx->dev));
    CK(cudaStreamSynchronize(ctx->st));
    CK(cudaStreamSynchronize(ctx->cst));
    CK(cudaStreamSynchronize(ctx->rst));
    harvest(ctx);
    if (launches) *launches = ctx->st_launch[kind];
    if (ms) *ms = ctx->st_ms[kind];
    if (bytes) *bytes = ctx->st_bytes[kind];
    return DUHL_OK;
}

duhl_status duhl_get_scd_shape(duhl_ctx* ctx, int* kernel, int* W, int* G, int* R) {
    if (!ctx) return DUHL_E_INVALID;
    if (kernel) *kernel = ctx->csc ? 0 : (ctx->tpa ? 3 : (ctx->pipe ? 2 : (ctx->ser ? 4 : 1)));
    if (W) *W = ctx->W;
    if (G) *G = ctx->G;
    if (R) *R = ctx->R;
    return DUHL_OK;
}

duhl_status duhl_get_counters(duhl_ctx* ctx, int64_t* launches, int64_t* h2d_bytes, int64_t* zc_bytes,
                              int64_t* updates, int64_t* d2h_bytes) {
    if (!ctx) return DUHL_E_INVALID;
    if (d2h_bytes) *d2h_bytes = ctx->d2h_bytes;
    if (launches) *launches = ctx->launches;
    if (h2d_bytes) *h2d_bytes = ctx->h2d_bytes;
    if (zc_bytes) *zc_bytes = ctx->zc_bytes;
    if (updates) *updates = ctx->updates;
    return DUHL_OK;
}

duhl_status duhl_get_unit_a_host(duhl_ctx* ctx, int64_t* cols, double* share) {
    if (!ctx) return DUHL_E_INVALID;
    if (cols) *cols = ctx->hua ? ctx->hua_cols : 0;
    if (share) *share = ctx->hua ? ctx->hua_share : 0.0;
    return DUHL_OK;
}

}  // extern "C"
