// kernels.h -- internal launch interface of the DuHL sm_100a kernels (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace duhl {

// Where column i of A lives: HBM slot (col_slot[i] >= 0) or pinned host memory
// mapped into the device address space (zero-copy over PCIe).
struct ColSrc {
    const float* pool;     // HBM slot pool, slot s at pool + s*ld_dev
    int64_t ld_dev;        // multiple of 4 floats
    const float* host;     // device alias of the pinned host store, column i at host + i*ld_host
    int64_t ld_host;       // multiple of 4 floats
    const int* col_slot;   // [n] device, -1 = not resident
};

struct GapParams {
    int model;
    int64_t d, d4, n;          // d4 = d rounded up to 4 (zero-padded rows)
    ColSrc src;
    const int64_t* cols;       // [k] device column list; nullptr = columns 0..k-1
    int64_t k;
    const double* vt;          // shared vector, [d4], zero padded
    double wscale;             // w = wscale * vt (Lasso 1, SVM 1/(lambda n))
    const double* alpha;       // [n]
    const double* y;           // [n] SVM labels (nullptr for Lasso)
    double lambda, B;
    double eta;                // elastic net only
    double* s_acc;             // [k] partial-dot accumulator (multi-tile passes), zero on entry
    double* z;                 // [n] gap memory or nullptr
    double* gap_out;           // [k] or nullptr
    double* s_out;             // [k] or nullptr
    double* sums;              // [4] certificate sums or nullptr: sum gap, sum aux, sum |a| / sum y a, max |a| (bits)
    int* flag;                 // bit0 negative gap, bit1 non-finite
    double* norms_out;         // create's ingest pass: ||a_i||^2 by column index (zero on entry) or nullptr
    float* fill_pool;          // create's ingest pass: columns i < fill_cols also stored to slot i
    int64_t fill_ld, fill_cols;  //   of the HBM pool (stride fill_ld floats); nullptr / 0 = off
};

struct ScdParams {
    int model;
    int64_t d, d4, n;
    double lambda;
    const float* pool;
    int64_t ld_dev;
    const int64_t* order_j;    // [L] coordinate processed at position t
    const int* order_slot;     // [L] its HBM slot
    int64_t L;
    const double* norms;       // [n] ||a_j||^2
    const double* y;           // [n] (SVM) or nullptr
    double* alpha;             // [n]
    double* vt;                // [d4] shared vector
    int W, R, G, NB;           // block size (% 4 == 0; <= 16 legacy, <= 32 pipe), rows per CTA, (compute) CTAs, TMA stages
    // pipe kernel: bar = cnt[6] (arrivals per reduction buffer) + flg[6] at bar + 8 (delta tags)
    int exact;                 // 1: fp64 Gram products (bit-level parity mode); 0: fp32 Gram within a warp
    double lam_q, lam_l1;      // ridge / elastic-net kernels: lambda eta d (quadratic), lambda (1-eta) d (l1)
    double* red;               // [scd_red_doubles(W)] zero on entry
    unsigned* bar;             // [2] grid-barrier counters (per block parity), zero on entry
    unsigned long long* trace; // developer phase timer [16] or nullptr
    const unsigned* order_batch;  // [L] staging-copy sequence number of each column (0 = resident)
    const double *order_a, *order_inv, *order_y;  // [L] alpha at pass start, 1/||a||^2 (-1: zero column), y
    const unsigned* progress;     // last landed staging copy, written by the copy stream; or nullptr
    int* err;                     // set (bit 0: staging wait, bit 1: grid barrier) on a wait timeout
    int gram_tc;                  // pipe kernel, fast mode, W = 32: Gram tiles on the tensor cores (3xTF32; default 1)
    int stage_ctas;               // > 0: order_batch holds gather-plan entries + 1 (k_stage_gather with this many
                                  // CTAs, progress[q % stage_ctas]); 0: copy-engine sequence numbers (progress[0])
};

// Sparse matrix, compressed sparse columns, resident in HBM:
// column i = values/rows [col_ptr[i], col_ptr[i+1]), rows ascending in [0, d).
struct CscMat {
    const int64_t* col_ptr;  // [n + 1]
    const int* rows;         // [nnz]
    const float* vals;       // [nnz]
};

// Asynchronous SCD epoch on a CSC working set (TPA-SCD style, P:336 / App. D):
// one warp per coordinate in visiting order, warp-reduced a_j^T v, closed-form
// step, fp64 RED update of v.  warps = 1 runs the positions strictly in order
// (== sequential SCD up to summation order); more warps run them concurrently.
struct CscScdParams {
    int model;
    int64_t d, n;
    double lambda;
    CscMat A;
    const int64_t* order_j;  // [L]
    int64_t L;
    const double* norms;     // [n]
    const double* y;         // [n] (SVM) or nullptr
    double* alpha;           // [n]
    double* vt;              // [d4]
    double eta;              // elastic net only
};

// Asynchronous (TPA-SCD style) dense epoch, scd_tpa.cu: W clusters of C CTAs, CTA rank r of a
// cluster owns rows [r Rc, (r + 1) Rc) of every column; v~f = fp32 shadow of the shared vector.
struct TpaParams {
    int model;
    int64_t d, d4, n;
    double lambda, eta;
    const float* pool;
    int64_t ld_dev;
    const int64_t* order_j;    // [L] coordinate at position t
    const int* order_slot;     // [L] its HBM slot
    const double* order_a;     // [L] alpha at pass start
    int64_t L;
    const double* norms;       // [n]
    const double* y;           // [n] SVM labels or nullptr
    double* alpha;             // [n]
    float* vf;                 // [d4] fp32 shadow of the epoch's updates of v~ (zero at start), REDed
    const double* v0;          // [d4] v~ at epoch start (fp64)
    int v0_smem;               // unused (kept 0)
    const double* u0;          // [n] a_j^T v~0 for j in P (taken before the epoch)
    int C;                     // CTAs per cluster
    int64_t Rc;                // rows per CTA (multiple of 4)
    const unsigned* progress;  // staging waits (nullptr: columns resident)
    int stage_ctas;
    const unsigned* order_batch;
    int* err;
};
size_t tpa_smem_bytes(int64_t Rc, bool v0_smem);
cudaError_t launch_scd_tpa(const TpaParams& p, int W, cudaStream_t st, int64_t* launches);
// v~ = v~0 + A_P (alpha_P - a0) in fp64 over the working set's HBM slots
cudaError_t launch_tpa_resync(const float* pool, int64_t ld_dev, const int* P_slot, const int64_t* P,
                              const double* alpha, const double* a0, int64_t m, const double* v0, double* vt,
                              int64_t d4, cudaStream_t st, int64_t* launches);
cudaError_t launch_f64_to_f32(const double* x, float* y, int64_t k, cudaStream_t st, int64_t* launches);
cudaError_t launch_scatter_scaled(const double* s, const int64_t* P, int64_t m, double scale, double* u0,
                                  cudaStream_t st, int64_t* launches);
cudaError_t preload_tpa_kernels();

__host__ __device__ int scd_nred(int W);
size_t scd_red_doubles(int W);  // size of ScdParams::red
size_t scd_smem_bytes(int W, int R, int NB);

cudaError_t launch_gap_pass(const GapParams& p, int tile_rows, cudaStream_t st, int64_t* launches,
                            int max_ctas = 0);
// k_gap_finalize alone: gap_i from the complete dots p.s_acc[t] of columns p.cols[t] (s_acc is zeroed).
cudaError_t launch_gap_finalize(const GapParams& p, cudaStream_t st, int64_t* launches);
cudaError_t launch_col_norms(const ColSrc& src, int64_t d4, int64_t n, double* norms,
                             cudaStream_t st, int64_t* launches);
// work: device scratch of launch_topm_work_bytes() (multi-CTA form for large n; nullptr = one CTA)
cudaError_t launch_topm(const double* z, int64_t n, int64_t m, int keymode, uint64_t seed,
                        int64_t round, int64_t* P_out, int* flag, cudaStream_t st,
                        int64_t* launches, void* work = nullptr);
size_t launch_topm_work_bytes();
// resident working set bookkeeping on the device (see k_resident_select); out[0] swaps, out[1] nnz over P
cudaError_t launch_resident_select(const int64_t* P, int64_t m, int* stamp, int sel, int* P_slot,
                                   unsigned* P_batch, const int64_t* col_ptr, unsigned long long* out,
                                   cudaStream_t st, int64_t* launches);
// Pass order + per-position inputs.  P == nullptr: order_j/slot/batch already
// hold an explicit order of length m; only alpha / 1/norm / y are gathered.
cudaError_t launch_perm_order(const int64_t* P, const int* P_slot, const unsigned* P_batch, int64_t m,
                              uint64_t seed, int64_t round, int64_t pass, int64_t* order_j,
                              int* order_slot, unsigned* order_batch, double* order_a, double* order_inv,
                              double* order_y, const double* alpha, const double* norms, const double* y,
                              cudaStream_t st, int64_t* launches, double ridge_ld = 0.0);
cudaError_t launch_scd_gram(const ScdParams& p, cudaStream_t st, int64_t* launches);
// light-round staging: plan entries (cols[q] -> slots[q]) gathered host -> HBM by `ctas` CTAs;
// progress[c] = entries done by CTA c (zero on entry)
cudaError_t launch_stage_gather(const float* host, int64_t ld_host, float* pool, int64_t ld_dev, int64_t d4,
                                const int64_t* cols, const int* slots, int64_t nplan, unsigned* progress,
                                int ctas, cudaStream_t st, int64_t* launches);
// pipelined form (scd_pipe.cuh): p.G compute CTAs + one control CTA, W <= 32, p.NB in {3, 4}
size_t pipe_red_doubles(int W);   // size of ScdParams::red (reduction + delta buffers)
size_t pipe_smem_bytes(int W, int R, int NS);
cudaError_t launch_scd_pipe(const ScdParams& p, cudaStream_t st, int64_t* launches);
// k_scd_ser (scd_ser.cuh): k_scd_gram's layout without the cross Gram, u taken after each update
cudaError_t launch_scd_ser(const ScdParams& p, cudaStream_t st, int64_t* launches);
cudaError_t preload_kernels();
cudaError_t launch_csc_norms(const CscMat& A, int64_t n, double* norms, cudaStream_t st, int64_t* launches);
cudaError_t launch_csc_gap(const GapParams& p, const CscMat& A, int max_ctas, cudaStream_t st, int64_t* launches);
cudaError_t launch_csc_scd(const CscScdParams& p, int warps, cudaStream_t st, int64_t* launches);
// vt += A alpha over the columns with alpha != 0 (fp64 REDs)
cudaError_t launch_csc_matvec(const CscMat& A, const double* alpha, int64_t n, double* vt, cudaStream_t st,
                              int64_t* launches);
cudaError_t launch_matvec(const ColSrc& src, const double* alpha, int64_t n, int64_t d,
                          int64_t d4, const double* b, double* vt, cudaStream_t st,
                          int64_t* launches);
cudaError_t launch_set_slots(int* col_slot, const int64_t* cols, const int* slots, int64_t cnt,
                             cudaStream_t st, int64_t* launches);
cudaError_t launch_gather_f64(const double* x, const int64_t* idx, int64_t k, double* out, cudaStream_t st,
                              int64_t* launches);
cudaError_t launch_delta_v(const double* v, const double* v0, int64_t d4, double* dv, double* sums,
                           cudaStream_t st, int64_t* launches);
cudaError_t launch_ydalpha(const double* alpha, const double* y, const int64_t* P, const double* aold, int64_t k,
                           double* sums, cudaStream_t st, int64_t* launches);
// ridge line search: sums[0] += sum_q aold_q da_q, sums[1] += sum_q da_q^2 (da_q = alpha_P[q] - aold_q)
cudaError_t launch_ridge_sums(const double* alpha, const int64_t* P, const double* aold, int64_t k, double* sums,
                              cudaStream_t st, int64_t* launches);
cudaError_t launch_lasso_dgrid(const double* alpha, const int64_t* P, const double* aold, int64_t k,
                               const double* gam, int ng, double* out, cudaStream_t st, int64_t* launches);
cudaError_t launch_apply_gamma(double* v, const double* v0, const double* dv, int64_t d4, double* alpha,
                               const int64_t* P, const double* aold, int64_t k, double gamma, cudaStream_t st,
                               int64_t* launches);
cudaError_t launch_sum(const double* x, int64_t n, double* out, cudaStream_t st, int64_t* launches);
cudaError_t launch_vec_sums(const double* vt, const double* b, int64_t d4, double* out2,
                            cudaStream_t st, int64_t* launches);

}  // namespace duhl
