/*
 * duhl.h -- C ABI of the B200-native DuHL hot path (arXiv 1708.05357).
 *
 * DuHL ("Duality-gap based Heterogeneous Learning", Alg. 2)
 * trains a generalized linear model  min_alpha  f(A alpha) + sum_i g_i(alpha_i)
 * (Eq. 1) when A (d x n, columns a_i) is larger than accelerator memory:
 *   - unit A = pinned host DRAM holding all of A,
 *   - unit B = B200 HBM holding the working set A_[P] (|P| = m) under a budget.
 * Each round selects the m coordinates with the largest (time-delayed) duality
 * gaps z (Eq. 11), swaps their columns into HBM, runs randomized
 * coordinate-descent passes on them (App. D) and refreshes z
 * (Alg. 2 l.7-10).  Models:
 *   DUHL_LASSO    (App. C eq. lassoobj):  (1/2d)||A alpha - b||^2 + lambda ||alpha||_1
 *   DUHL_SVM_DUAL (App. C eq. dualsvm,  P:773):  (1/n) sum(-y_i alpha_i)
 *                                                + (1/(2 lambda n^2)) ||A alpha||^2,  y_i alpha_i in [0,1]
 *
 * Conventions (all entry points):
 *   - Every function returns a duhl_status; 0 = DUHL_OK.  Nothing throws across
 *     the ABI.  On error, duhl_last_error(ctx) holds a message (owned by ctx,
 *     valid until the next call on that ctx).
 *   - Pointers named *_host / marked "host" are host memory owned by the caller;
 *     the library never keeps them past the call unless cfg.borrow_host = 1.
 *   - A duhl_ctx is not thread-safe; distinct contexts are independent.
 *   - Matrices are dense, column-major float32: column a_i starts at
 *     values + i*ld, ld >= d (Eq. 1: A = [a_1 ... a_n]).
 *   - Vectors alpha, z, gaps are float64 of length n; v, b are float64 of length d.
 *   - "shared vector" v~ = A alpha - b (Lasso) or v^ = A alpha (SVM)
 *     is the state unit B updates; w (App. E) = v~ (Lasso) or v^/(lambda n) (SVM).
 *   - All work runs in the library's CUDA kernels for sm_100a on cfg.device;
 *     there is no CPU fallback: without a usable B200 every call that computes
 *     returns DUHL_E_CUDA.
 */
#ifndef DUHL_H
#define DUHL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct duhl_ctx duhl_ctx; /* opaque; one per problem instance */

typedef enum { DUHL_LASSO = 0, DUHL_SVM_DUAL = 1, DUHL_RIDGE = 2, DUHL_ELASTIC_NET = 3 } duhl_model;

/* Block selection policies: Eq. 11 gap memory, and the paper's
 * reference schemes: sequential blocks [Yu 2012], uniform. */
typedef enum { DUHL_SEL_GAP = 0, DUHL_SEL_SEQUENTIAL = 1, DUHL_SEL_UNIFORM = 2, DUHL_SEL_IMPORTANCE = 3 } duhl_policy;

typedef enum {
    DUHL_OK = 0,
    DUHL_E_INVALID = 2,       /* bad argument: d,n < 1, non-finite data, y not +-1, lambda <= 0, m > n, budget too small */
    DUHL_E_IO = 3,
    DUHL_E_NUMERIC = 4,       /* non-finite state, or a gap below -1e-12 x its scale (reading R17) */
    DUHL_E_BOUND = 5,         /* Lasso |alpha_i| > B: the Lipschitzing bound was violated */
    DUHL_E_NOMEM = 6,
    DUHL_E_CUDA = 7,          /* CUDA runtime failure or no sm_100 device */
    DUHL_E_NCCL = 8,
    DUHL_E_NOT_CONVERGED = 9  /* max_rounds reached; outputs are still valid */
} duhl_status;

typedef struct {
    int64_t d;            /* rows (Lasso: samples; SVM: features) */
    int64_t n;            /* columns = coordinates of alpha (Lasso: features; SVM: samples) */
    const float* values;  /* host, column-major: a_i at values + i*ld */
    int64_t ld;           /* leading dimension, ld >= d */
} duhl_matrix;

/* Sparse matrix in compressed sparse columns: column i holds
 * values[k], row_idx[k] for k in [col_ptr[i], col_ptr[i+1]); rows strictly
 * ascending in [0, d); col_ptr[0] = 0, nondecreasing.  Host memory, read
 * during duhl_create_csc only (copied to HBM). */
typedef struct {
    int64_t d;              /* rows */
    int64_t n;              /* columns = coordinates */
    const int64_t* col_ptr; /* [n + 1] */
    const int32_t* row_idx; /* [col_ptr[n]] */
    const float* values;    /* [col_ptr[n]] */
} duhl_csc;

typedef struct {
    size_t hbm_budget_bytes;  /* HBM for the working-set slot pool; 0 = all n columns resident */
    int64_t m;                /* working-set size |P|; 0 = as many columns as the budget holds (n if budget 0) */
    int device;               /* CUDA device ordinal */
    int scd_block;            /* W: coordinates per Gram block of the exact SCD kernel; 0 = auto */
    int scd_ctas;             /* CTAs of the SCD epoch (row partition); 0 = auto */
    double refresh_fraction;  /* unit-A refresh per round, fraction of n (rotating cursor, reading R8); 1 = o-DuHL */
    int64_t cert_every;       /* certificate (full duality gap) every R rounds in duhl_solve; >= 1 */
    uint64_t seed;            /* seeds the counter-based permutation generator */
    int borrow_host;          /* 1: pin the caller's matrix in place (it must outlive the ctx); 0: copy */
    int cert_adaptive;        /* 1: duhl_solve also certifies when the gap-memory sum sum_i z_i <= eps */
    int profile;              /* 1: time every kernel launch with CUDA events (duhl_get_kernel_stats) */
    int scd_exact;            /* 1: fp64 Gram products -- the SCD pass equals sequential SCD to rounding;
                                 0: fp32 Gram accumulation inside a warp (fp64 beyond), ~1e-7 relative */
    int64_t n_global;         /* multi-GPU: total columns of the problem (0 = this matrix is all of it) */
    int64_t col_offset;       /* multi-GPU: global index of this shard's first column */
    int linesearch;           /* 1: exact line search on the aggregation weight gamma in [0,1] after each
                                 round's epoch; 0: gamma = 1 (Alg. 2 l.11) */
    int unit_a_ctas;          /* unit-A refresh beside the epoch: CTAs of its persistent gap kernel; the
                                 SCD grid leaves them their SMs.  0 = auto (8 when the data exceeds the
                                 budget and refresh_fraction > 0), -1 = off (the refresh runs on the
                                 whole GPU before the epoch) */
    int scd_kernel;           /* dense exact SCD kernel: 1 = k_scd_gram (warp-specialised: a control warp
                                 in every CTA, W <= 16; block b+1's partials include the cross Gram
                                 A_{b+1}^T A_b); 2 = k_scd_pipe (one control CTA runs the sequential
                                 steps; W <= 32); 3 = k_scd_ser (k_scd_gram's layout without the cross
                                 Gram: the compute warps assemble u_{b+1} = A_{b+1}^T v_b +
                                 A_{b+1}^T (A_b delta_b) after each block, W <= 16); 0 = auto
                                 (k_scd_pipe where shared memory holds W >= 24, else k_scd_ser).  All
                                 execute the same sequential order (App. D), up to summation order. */
    double eta;               /* DUHL_ELASTIC_NET only: g_i = lambda (eta/2 alpha_i^2 + (1-eta)|alpha_i|)
                                 (P:796-800), 0 < eta < 1; eta = 0 is DUHL_LASSO, eta = 1 DUHL_RIDGE */
    int unit_a_host_threads;  /* unit A on the host (Alg. 2 l.7-10 as the paper's CPU unit):
                                 host threads that compute a_i^T v~ for part of the refresh's (and of every
                                 certificate's) non-resident columns from the pinned store (DRAM, not PCIe);
                                 the device finishes their gaps.  With an HBM budget they also take 70 % of
                                 duhl_create's ingest pass (norms + gaps at alpha = 0 of the last columns;
                                 the GPU keeps at least the S columns it leaves in the pool).  0 = off (the
                                 GPU reads them over PCIe) */
    double unit_a_host_share; /* share of the refresh's non-resident columns given to those threads, in
                                 [0, 1]; < 0 = balanced each round from the measured host and PCIe rates */
    int scd_async;            /* dense problems: 0 = exact sequential Gram-block epoch (k_scd_gram /
                                 k_scd_pipe, above); 1 = asynchronous TPA-SCD-style epoch (App. D):
                                 scd_block (default 16) coordinates in flight, each on a cluster of CTAs
                                 that splits its column by rows, atomic fp32 updates of a shadow of v,
                                 then the exact fp64 resync v = v0 + A_P (alpha_P - alpha_P0).  Results
                                 depend on the interleaving (staleness <= scd_block); duhl_round takes
                                 the exact gamma line search.  scd_exact is ignored in this mode. */
} duhl_config;

/* One entry per round of duhl_solve (SPEC RoundTrace columns). */
typedef struct {
    int64_t round;
    int64_t swaps;            /* |P_t \ P_{t-1}|: columns copied host -> HBM (Fig. 4b) */
    int64_t refreshed;        /* unit-A gap refreshes this round */
    double cert_gap;          /* certified duality gap after the round; -1 if not computed */
    double z_sum;             /* sum_i z_i after the round: the (time-delayed) gap estimate of the gap memory */
    double gamma;             /* aggregation weight applied this round (1 without line search) */
    double time_s;            /* wall seconds since duhl_solve entry (duhl_round: duration of the round) */
    double rho;               /* rho_{t,P} (Eq. 6) on the gap memory at selection time:
                                 (mean of z over P) / (mean of z over this rank's columns); 1 if z = 0 */
    double gap_est;           /* estimate of the duality gap after the round from fresh gaps only:
                                 sum of z over P + (n - m) x the mean z of this round's refreshed
                                 columns outside P (summed over ranks); -1 when no refresh ran.
                                 duhl_solve's adaptive certificates use it (else z_sum) */
} duhl_round_record;

/* Fills *cfg with defaults: budget 0, m 0, device 0, auto SCD shape,
 * refresh_fraction 0.05, cert_every 10, seed 170805357, borrow_host 0,
 * cert_adaptive 1, profile 0, scd_exact 1, n_global 0, col_offset 0,
 * linesearch 0, unit_a_ctas 0, scd_kernel 0. */
void duhl_default_config(duhl_config* cfg);

/* Creates a problem instance.
 *   A       host dense matrix (copied into library-owned pinned memory unless borrow_host)
 *   b_or_y  host float64: Lasso b[d] (labels); SVM y[n] in {-1,+1}
 *   lambda  > 0: Lasso L1 weight; SVM L2 weight
 * Precomputes ||a_i||^2 and B = ||b||^2/(2 lambda d), sets alpha = 0 and
 * the gap memory z to the exact gaps at alpha = 0 (reading R6).
 * Errors: DUHL_E_INVALID, DUHL_E_NOMEM, DUHL_E_CUDA.  *out = NULL on error. */
duhl_status duhl_create(const duhl_matrix* A, const double* b_or_y, double lambda,
                        duhl_model model, const duhl_config* cfg, duhl_ctx** out);

/* Sparse variant (SURVEY 8 C5, P:433 sparse Lasso setting): same semantics as
 * duhl_create on a CSC matrix.  The matrix is held resident in HBM (8 bytes per
 * nonzero); hbm_budget_bytes must be 0 or at least that (DUHL_E_INVALID
 * otherwise); no staging, borrow_host ignored.  The SCD epoch is the
 * warp-per-coordinate asynchronous form (App. D; fp64 RED updates of v):
 * scd_exact = 1 runs the positions strictly in order on one warp (sequential
 * SCD up to summation order), scd_exact = 0 runs them concurrently on all SMs
 * (stale reads possible; v stays exactly A alpha - b up to rounding).
 * Errors: as duhl_create (DUHL_E_INVALID also for unsorted / out-of-range rows,
 * non-finite values, a non-monotone col_ptr). */
duhl_status duhl_create_csc(const duhl_csc* A, const double* b_or_y, double lambda,
                            duhl_model model, const duhl_config* cfg, duhl_ctx** out);

duhl_status duhl_destroy(duhl_ctx* ctx);

/* Duality-gap pass (Eq. 4; App. E closed forms P:852 / P:867) at the
 * current state for the k columns idx[0..k) (host int64; idx = NULL: all n
 * columns, k ignored).  Writes z_i = max(gap_i, 0) into the gap memory and, if
 * non-NULL, gap_i to z_out[k] and s_i = a_i^T w to s_out[k] (host float64).
 * Resident columns are read from HBM, the others from pinned host memory.
 * Errors: DUHL_E_INVALID (index out of range), DUHL_E_NUMERIC, DUHL_E_CUDA. */
duhl_status duhl_gaps(duhl_ctx* ctx, const int64_t* idx, int64_t k, double* z_out, double* s_out);

/* Working-set selection (Eq. 11 for DUHL_SEL_GAP: the m largest z, ties to the
 * lowest index, reading R7; the baselines of P:400-404: DUHL_SEL_SEQUENTIAL blocks
 * [k m, (k+1) m), k = round mod ceil(n/m); DUHL_SEL_UNIFORM the m smallest counter
 * keys key(seed, round, -1, j); DUHL_SEL_IMPORTANCE m draws without replacement with
 * probability proportional to ||a_j||^2, i.e. the m smallest exponential clocks
 * -ln(u_j)/||a_j||^2, u_j = ((key(seed, round, -2, j) >> 11) + 1/2) 2^-53, zero columns
 * last) for round `round`, then stages A_[P] into the HBM
 * slot pool (Alg. 2 l.4).  m = 0 uses cfg.m.  P_out (host int64[m], may be NULL)
 * receives P in ascending index order; *n_swaps_out (may be NULL) the number of
 * columns copied host -> HBM.  Errors: DUHL_E_INVALID (m > n or > pool), DUHL_E_CUDA. */
duhl_status duhl_select(duhl_ctx* ctx, duhl_policy policy, int64_t m, int64_t round,
                        int64_t* P_out, int64_t* n_swaps_out);

/* `passes` randomized coordinate-descent passes over the working set (App. D:
 * Lasso soft-threshold step P:804-815 with eta = 0, SVM box step P:824-827),
 * updating alpha_P and the shared vector.  Position t of pass p processes
 * P[pi(t)] (P ascending), pi the Feistel bijection keyed by (seed, round, p)
 * (DESIGN.md "Randomness").  If perm (host int64) is
 * given, exactly one pass is run in the order perm[0..perm_len), whose entries
 * must be distinct, resident members of P.  The kernel executes the sequential
 * SCD semantics exactly (Gram-block reformulation).
 * Errors: DUHL_E_INVALID, DUHL_E_CUDA. */
duhl_status duhl_scd_epoch(duhl_ctx* ctx, int passes, uint64_t seed, int64_t round,
                           const int64_t* perm, int64_t perm_len);

/* Certificate (Eq. 2 = sum of Eq. 4 terms) at the current state over all n
 * columns, plus the primal objective O(alpha) and the dual value D so that
 * gap = O - D (D per App. E conjugates).  Any output may be NULL.
 * The per-coordinate gaps it computes also refresh the whole gap memory z (a full
 * unit-A pass, Alg. 2 l.7-10; reading R25).
 * Errors: DUHL_E_NUMERIC, DUHL_E_BOUND (Lasso max|alpha_i| > B), DUHL_E_CUDA. */
duhl_status duhl_duality_gap(duhl_ctx* ctx, double* gap, double* primal, double* dual);

/* One DuHL round t (Alg. 2 body): select (policy) -> stage A_[P] into HBM ->
 * unit-A refresh of ceil(refresh_fraction n) gaps at the round-start state
 * (rotating cursor, reading R8) -> `passes` SCD passes (permutation keyed by
 * (cfg.seed, round, pass)) -> refresh z_P at the new state (reading R9) ->
 * if certify != 0, the certificate.  rec (host, may be NULL) receives the
 * round's record (time_s = its duration).  Errors as duhl_select/duhl_scd_epoch. */
duhl_status duhl_round(duhl_ctx* ctx, int64_t round, int passes, duhl_policy policy, int certify,
                       duhl_round_record* rec);

/* DuHL rounds (Alg. 2): select -> swap -> [unit-A refresh of
 * ceil(refresh_fraction n) gaps at the round-start state] -> `passes` SCD
 * passes -> refresh z_P at the new state; certificate every cfg.cert_every
 * rounds; stops when the certified gap <= eps.  trace (host, may be NULL)
 * receives up to trace_cap records.  Returns DUHL_OK when certified,
 * DUHL_E_NOT_CONVERGED after max_rounds (outputs valid). */
duhl_status duhl_solve(duhl_ctx* ctx, double eps, int64_t max_rounds, int passes,
                       duhl_policy policy, duhl_round_record* trace, int64_t trace_cap,
                       int64_t* rounds_out, double* gap_out);

/* Copies the state to host buffers (any may be NULL): alpha[n], shared vector
 * v[d] (v~ or v^ as above), gap memory z[n]. */
duhl_status duhl_get_state(duhl_ctx* ctx, double* alpha_out, double* v_out, double* z_out);

/* Sets alpha (host float64[n]; SVM entries must satisfy y_i alpha_i in [0,1]),
 * recomputes the shared vector exactly from A and resets z to the exact gaps.
 * On a ctx joined to a communicator this is collective: every rank passes its
 * shard's alpha and v = sum_k A_k alpha_k (- b) is reduced over the ranks. */
duhl_status duhl_set_state(duhl_ctx* ctx, const double* alpha);

/* Multi-GPU (CoCoA-style): one process per GPU, each
 * holding a contiguous column shard (cfg.n_global, cfg.col_offset).  The
 * shared vector v is replicated; each round every rank selects and solves on
 * its own shard from the common v, then dv is summed with ncclAllReduce over
 * NVLink and applied with weight gamma chosen by the exact line search (forced
 * on when nranks > 1: sigma' = 1 local steps summed with weight 1 can diverge).
 * A communicator of one rank still runs ncclAllReduce.  duhl_set_state is
 * collective on a joined ctx (v = sum over ranks of A_k alpha_k, minus b).  Certificates sum the
 * per-column terms over ranks.  duhl_comm_unique_id (one rank) returns the 128
 * byte NCCL id that the caller broadcasts; every rank then calls
 * duhl_comm_init on its ctx.  All later calls that reduce must be made by all
 * ranks in the same order.  Errors: DUHL_E_NCCL (libnccl.so.2 missing / NCCL failure). */
duhl_status duhl_comm_unique_id(void* id_out);
duhl_status duhl_comm_init(duhl_ctx* ctx, const void* id, int nranks, int rank);

/* In-process group (SURVEY 8(e) "single process, one host thread per GPU"): the
 * contexts of one process, each driven by its own host thread (on the same or on
 * different GPUs), join a group instead of an NCCL communicator.  Collectives copy
 * the buffer to host memory, wait for every rank (bounded: 600 s, then
 * DUHL_E_NCCL), and every rank sums the buffers in rank order, so all ranks hold
 * bit-identical results.  The same rules as duhl_comm_init apply (all ranks call
 * every reducing function in the same order; aggregation takes the exact line
 * search when nranks > 1).  The group must outlive its contexts; the caller owns it.
 * Errors: DUHL_E_INVALID (nranks < 1, rank out of range, ctx already joined). */
typedef struct duhl_group duhl_group;
duhl_status duhl_group_create(int nranks, duhl_group** out);
duhl_status duhl_group_destroy(duhl_group* g);
duhl_status duhl_comm_init_group(duhl_ctx* ctx, duhl_group* g, int rank);

/* The current working set P (Alg. 2 l.3, ascending local column indices) as chosen
 * by the last duhl_select / duhl_round / duhl_solve round: *m_out = |P|; P_out
 * (host int64[cap], may be NULL) receives it.  Errors: DUHL_E_INVALID (cap < |P|). */
duhl_status duhl_get_working_set(duhl_ctx* ctx, int64_t* P_out, int64_t cap, int64_t* m_out);

/* Per-round callback of duhl_solve (SURVEY 8(b) duhl_trace_cb): called on the calling
 * thread after every round with that round's record (valid during the call only) and
 * `user`; cb = NULL removes it.  It is called in addition to filling the trace array. */
typedef void (*duhl_trace_cb)(const duhl_round_record* rec, void* user);
duhl_status duhl_set_trace_callback(duhl_ctx* ctx, duhl_trace_cb cb, void* user);

/* Device-side view for callers that time kernels on their own stream:
 * returns the CUDA stream (cudaStream_t) all compute of ctx is issued on. */
duhl_status duhl_get_stream(duhl_ctx* ctx, void** stream_out);

/* Per-kind kernel timing (cfg.profile = 1), accumulated since creation:
 * kind 0 = SCD epoch kernel, 1 = gap pass (compute stream: z_P refresh,
 * certificate, duhl_gaps), 2 = top-m select, 3 = working-set H2D staging (copy
 * stream: copy engine or the k_stage_gather kernel), 4 = unit-A refresh gap pass (its own stream,
 * concurrent with SCD), 5 = SCD epoch launches that consume staged columns as they land (pass 0
 * of a round whose staging overlaps the epoch: bound by the staging, not by HBM; kind 0 then
 * holds only the launches that wait for nothing), 6 = the exact fp64 resync after an asynchronous
 * epoch (cfg.scd_async).  *launches = timed launches, *ms = summed
 * CUDA-event milliseconds, *bytes = summed ALGORITHMIC bytes (DESIGN.md
 * "Roofline"): SCD  L (4 d4 + 24) + 16 d4;  gap  k (4 d4 + 24) + 8 d4 tiles;
 * top-m  8 n x passes;  staging  columns x 4 d4. */
duhl_status duhl_get_kernel_stats(duhl_ctx* ctx, int kind, int64_t* launches, double* ms,
                                  double* bytes);

/* Counters since creation: kernel launches issued, bytes copied host->device
 * (copy engine: cold fill + swaps), bytes the gap kernels read from pinned host
 * memory over PCIe (zero-copy: unit-A refresh + certificates of non-resident
 * columns, 4 d4 per column), SCD coordinate updates, bytes read back device->host
 * (status flags, reductions, P, state, the host unit A's v snapshot).  Any may be NULL. */
duhl_status duhl_get_counters(duhl_ctx* ctx, int64_t* launches, int64_t* h2d_bytes,
                              int64_t* zc_bytes, int64_t* updates, int64_t* d2h_bytes);

/* Host-thread unit A (cfg.unit_a_host_threads): columns whose refresh dots the host
 * threads computed (all rounds so far) and the current share of the refresh's
 * non-resident columns they take.  0 / 0 when off.  Either pointer may be NULL. */
duhl_status duhl_get_unit_a_host(duhl_ctx* ctx, int64_t* cols, double* share);

/* Launch shape of the dense exact SCD epoch chosen at create (cfg.scd_kernel, shared
 * memory): *kernel 1 = k_scd_gram (warp-specialised), 2 = k_scd_pipe (control CTA),
 * 3 = k_scd_tpa (cfg.scd_async: W coordinates in flight, G = W x cluster CTAs, R rows per CTA),
 * 4 = k_scd_ser (no cross Gram, see cfg.scd_kernel);
 * W coordinates per Gram block, G (compute) CTAs of R rows each.  CSC problems report
 * kernel 0 (k_csc_scd).  Any pointer may be NULL. */
duhl_status duhl_get_scd_shape(duhl_ctx* ctx, int* kernel, int* W, int* G, int* R);

const char* duhl_last_error(const duhl_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DUHL_H */
