// kernels.cu -- sm_100a kernels of the DuHL hot path (arXiv 1708.05357).
//
//   gap pass      k_gap_tile / k_gap_finalize   Eq. 4 + App. E
//   top-m select  k_topm                        Eq. 9 / Eq. 11   (a3)
//   SCD epoch     k_scd_gram                    App. D           (a5)
//   helpers       norms (a1), permutation keys, matvec (set_state), slot table, sums
//
// Data layout: A column-major float32; every column padded with zeros to d4 =
// round_up(d, 4) rows so each column is a whole number of 16-byte vectors.
// All accumulation is fp64 (fp32 x fp32 products are exact in fp64).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "device.cuh"
#include "kernels.h"

namespace duhl {

__device__ __forceinline__ const float* col_ptr(const ColSrc& s, int64_t i) {
    int sl = s.col_slot[i];
    return sl >= 0 ? s.pool + (int64_t)sl * s.ld_dev : s.host + i * s.ld_host;
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// =====================================================================================
// Gap pass.  Grid (column groups, row tiles).  A CTA stages its row tile of
// w = wscale * vt in shared memory (fp64) once and streams the tile of each of
// its columns from HBM (or pinned host memory over PCIe) with 16-byte
// no-L1-allocate loads; one warp per column, fp64 FMAs, warp-shuffle reduction.
// Single row tile: the gap is finalised in place.  Several tiles: partial dots
// are added into s_acc and k_gap_finalize completes them.
// =====================================================================================
constexpr int kGapThreads = 256;
constexpr int kGapColsPerCta = 32;

struct SumAcc {
    double g = 0, aux = 0, a = 0, amax = 0;
};

__device__ __forceinline__ void gap_finish_one(const GapParams& p, int64_t t, int64_t i, double s,
                                               SumAcc& acc, int& flag) {
    double a = p.alpha[i];
    double yy = p.model == kSvm ? p.y[i] : 0.0;
    double scale, aux;
    double g = coord_gap(p.model, a, s, yy, p.lambda, p.B, (double)p.d, (double)p.n, &scale, &aux);
    if (!isfinite(g)) flag |= 2;
    else if (g < -1e-12 * (scale > 1.0 ? scale : 1.0)) flag |= 1;
    double gz = g > 1e-12 * scale ? g : 0.0;  // rounding noise reads as +0.0 (reading R17)
    if (p.z) p.z[i] = gz;
    if (p.gap_out) p.gap_out[t] = gz;
    if (p.s_out) p.s_out[t] = s;
    acc.g += gz;
    acc.aux += aux;
    acc.a += p.model == kLasso ? fabs(a) : yy * a;
    acc.amax = fmax(acc.amax, fabs(a));
}

__device__ void block_flush_sums(const GapParams& p, SumAcc acc, int flag) {
    __shared__ double sh[4][kGapThreads / 32];
    __shared__ int shf;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) shf = 0;
    __syncthreads();
    if (flag) atomicOr(&shf, flag);
    if (p.sums) {
        acc.g = warp_sum(acc.g);
        acc.aux = warp_sum(acc.aux);
        acc.a = warp_sum(acc.a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc.amax = fmax(acc.amax, __shfl_xor_sync(~0u, acc.amax, o));
        if (lane == 0) {
            sh[0][warp] = acc.g;
            sh[1][warp] = acc.aux;
            sh[2][warp] = acc.a;
            sh[3][warp] = acc.amax;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (shf) atomicOr(p.flag, shf);
        if (p.sums) {
            double g = 0, x = 0, a = 0, mx = 0;
            for (int w = 0; w < kGapThreads / 32; ++w) {
                g += sh[0][w];
                x += sh[1][w];
                a += sh[2][w];
                mx = fmax(mx, sh[3][w]);
            }
            atomicAdd(&p.sums[0], g);
            atomicAdd(&p.sums[1], x);
            atomicAdd(&p.sums[2], a);
            atomicMax(reinterpret_cast<unsigned long long*>(&p.sums[3]),
                      (unsigned long long)__double_as_longlong(mx));
        }
    }
}

__global__ void __launch_bounds__(kGapThreads) k_gap_tile(GapParams p, int tile_rows, int ntiles) {
    extern __shared__ double ws[];
    const int64_t r0 = (int64_t)blockIdx.y * tile_rows;
    const int rows = (int)imin64(tile_rows, p.d4 - r0);  // multiple of 4
    for (int r = threadIdx.x; r < rows; r += blockDim.x) ws[r] = p.vt[r0 + r] * p.wscale;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * kGapColsPerCta;
    const int64_t t1 = imin64(p.k, t0 + kGapColsPerCta);
    const int nv = rows >> 2;
    const double2* w2 = reinterpret_cast<const double2*>(ws);
    SumAcc acc;
    int flag = 0;
    for (int64_t t = t0 + warp; t < t1; t += nw) {
        const int64_t i = p.cols ? p.cols[t] : t;
        const float4* a = reinterpret_cast<const float4*>(col_ptr(p.src, i) + r0);
        double s0 = 0.0, s1 = 0.0;
        int q = lane;
        for (; q + 96 < nv; q += 128) {  // 4 independent 16-B loads in flight per lane
            float4 f0 = ld_stream_f4(a + q), f1 = ld_stream_f4(a + q + 32);
            float4 f2 = ld_stream_f4(a + q + 64), f3 = ld_stream_f4(a + q + 96);
            double2 u, v;
            u = w2[2 * q]; v = w2[2 * q + 1];
            s0 = fma((double)f0.x, u.x, s0); s1 = fma((double)f0.y, u.y, s1);
            s0 = fma((double)f0.z, v.x, s0); s1 = fma((double)f0.w, v.y, s1);
            u = w2[2 * (q + 32)]; v = w2[2 * (q + 32) + 1];
            s0 = fma((double)f1.x, u.x, s0); s1 = fma((double)f1.y, u.y, s1);
            s0 = fma((double)f1.z, v.x, s0); s1 = fma((double)f1.w, v.y, s1);
            u = w2[2 * (q + 64)]; v = w2[2 * (q + 64) + 1];
            s0 = fma((double)f2.x, u.x, s0); s1 = fma((double)f2.y, u.y, s1);
            s0 = fma((double)f2.z, v.x, s0); s1 = fma((double)f2.w, v.y, s1);
            u = w2[2 * (q + 96)]; v = w2[2 * (q + 96) + 1];
            s0 = fma((double)f3.x, u.x, s0); s1 = fma((double)f3.y, u.y, s1);
            s0 = fma((double)f3.z, v.x, s0); s1 = fma((double)f3.w, v.y, s1);
        }
        for (; q < nv; q += 32) {
            float4 f = ld_stream_f4(a + q);
            double2 u = w2[2 * q], v = w2[2 * q + 1];
            s0 = fma((double)f.x, u.x, s0); s1 = fma((double)f.y, u.y, s1);
            s0 = fma((double)f.z, v.x, s0); s1 = fma((double)f.w, v.y, s1);
        }
        double s = warp_sum(s0 + s1);
        if (lane == 0) {
            if (ntiles == 1) gap_finish_one(p, t, i, s, acc, flag);
            else atomicAdd(&p.s_acc[t], s);
        }
    }
    if (ntiles == 1) block_flush_sums(p, acc, flag);
}

__global__ void __launch_bounds__(kGapThreads) k_gap_finalize(GapParams p) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    SumAcc acc;
    int flag = 0;
    if (t < p.k) {
        double s = p.s_acc[t];
        p.s_acc[t] = 0.0;  // ready for the next pass
        gap_finish_one(p, t, p.cols ? p.cols[t] : t, s, acc, flag);
    }
    block_flush_sums(p, acc, flag);
}

cudaError_t launch_gap_pass(const GapParams& p, int tile_rows, cudaStream_t st, int64_t* launches) {
    if (p.k <= 0) return cudaSuccess;
    int ntiles = (int)cdiv(p.d4, tile_rows);
    if (ntiles == 1) tile_rows = (int)p.d4;
    dim3 grid((unsigned)cdiv(p.k, kGapColsPerCta), (unsigned)ntiles);
    size_t smem = (size_t)tile_rows * sizeof(double);
    k_gap_tile<<<grid, kGapThreads, smem, st>>>(p, tile_rows, ntiles);
    ++*launches;
    if (ntiles > 1) {
        k_gap_finalize<<<(unsigned)cdiv(p.k, kGapThreads), kGapThreads, 0, st>>>(p);
        ++*launches;
    }
    return cudaGetLastError();
}

// =====================================================================================
// Column norms ||a_i||^2: warp per column, fp64 accumulation.
// =====================================================================================
__global__ void k_col_norms(ColSrc src, int64_t d4, int64_t n, double* norms) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const float4* a = reinterpret_cast<const float4*>(col_ptr(src, i));
    double s0 = 0, s1 = 0;
    for (int64_t q = lane; q < d4 / 4; q += 32) {
        float4 f = ld_stream_f4(a + q);
        s0 = fma((double)f.x, (double)f.x, s0);
        s1 = fma((double)f.y, (double)f.y, s1);
        s0 = fma((double)f.z, (double)f.z, s0);
        s1 = fma((double)f.w, (double)f.w, s1);
    }
    double s = warp_sum(s0 + s1);
    if (lane == 0) norms[i] = s;
}

cudaError_t launch_col_norms(const ColSrc& src, int64_t d4, int64_t n, double* norms,
                             cudaStream_t st, int64_t* launches) {
    k_col_norms<<<(unsigned)cdiv(n * 32, 256), 256, 0, st>>>(src, d4, n, norms);
    ++*launches;
    return cudaGetLastError();
}

// =====================================================================================
// Top-m selection (Eq. 9 / Eq. 11): radix select of the m-th largest key, then
// a stable compaction that keeps every key above the threshold and the
// lowest-index keys equal to it (reading R7).  Keys: keymode 0 = IEEE bits of
// z_i >= +0 (nonnegative doubles order as uint64); keymode 1 = ~key(seed,
// round, -1, i) (uniform baseline: the m smallest counter keys).
// One CTA of 1024 threads; 11-bit digits, 6 passes.  P_out ascending.
// =====================================================================================
constexpr int kTopThreads = 1024;
constexpr int kRadixBits = 11;
constexpr int kBins = 1 << kRadixBits;

__device__ __forceinline__ uint64_t select_key(const double* z, int64_t i, int keymode,
                                               uint64_t seed, int64_t round, int* bad) {
    if (keymode == 1) return ~perm_key(seed, round, -1, i);
    double v = z[i];
    if (!(v >= 0.0)) { *bad = 1; v = 0.0; }  // NaN or negative: flagged, treated as 0
    return (uint64_t)__double_as_longlong(v + 0.0);  // +0.0 canonicalises -0.0
}

__global__ void __launch_bounds__(kTopThreads) k_topm(const double* z, int64_t n, int64_t m,
                                                      int keymode, uint64_t seed, int64_t round,
                                                      int64_t* P_out, int* flag) {
    typedef cub::BlockScan<int, kTopThreads> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int hist[kBins];
    __shared__ int s_digit, s_above;
    const int tid = threadIdx.x;
    int bad = 0;
    uint64_t prefix = 0, pmask = 0;
    long long need = m;
    if (m <= 0) return;
    for (int hi = 64; hi > 0;) {
        const int nbits = min(kRadixBits, hi);
        const int shift = hi - nbits;
        const uint64_t dmask = (1ull << nbits) - 1;
        for (int b = tid; b < kBins; b += kTopThreads) hist[b] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += kTopThreads) {
            uint64_t k = select_key(z, i, keymode, seed, round, &bad);
            if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & dmask], 1);
        }
        __syncthreads();
        // counts from the top digit down: thread t owns reversed bins 2t, 2t+1
        const int e0 = kBins - 1 - 2 * tid, e1 = e0 - 1;
        int c0 = hist[e0], c1 = hist[e1];
        int excl;
        Scan(scan_tmp).ExclusiveSum(c0 + c1, excl);
        // above(e) = number of candidate keys with digit > e; exactly one bin holds the m-th key
        if (excl < need && need <= excl + c0) { s_digit = e0; s_above = excl; }
        else if (excl + c0 < need && need <= excl + c0 + c1) { s_digit = e1; s_above = excl + c0; }
        __syncthreads();
        need -= s_above;
        prefix |= (uint64_t)s_digit << shift;
        pmask |= dmask << shift;
        hi = shift;
        __syncthreads();
    }
    // prefix = threshold key T; need = how many keys equal to T to keep (lowest indices)
    long long base = 0, eqbase = 0;
    for (int64_t i0 = 0; i0 < n; i0 += kTopThreads) {
        const int64_t i = i0 + tid;
        int gt = 0, eq = 0;
        if (i < n) {
            uint64_t k = select_key(z, i, keymode, seed, round, &bad);
            gt = k > prefix;
            eq = k == prefix;
        }
        int eq_excl, eq_tot;
        Scan(scan_tmp).ExclusiveSum(eq, eq_excl, eq_tot);
        __syncthreads();
        int take = gt || (eq && (eqbase + eq_excl) < need);
        int pos, tot;
        Scan(scan_tmp).ExclusiveSum(take, pos, tot);
        if (take) P_out[base + pos] = i;
        base += tot;
        eqbase += eq_tot;
        __syncthreads();
    }
    if (bad) atomicOr(flag, 1);
}

cudaError_t launch_topm(const double* z, int64_t n, int64_t m, int keymode, uint64_t seed,
                        int64_t round, int64_t* P_out, int* flag, cudaStream_t st,
                        int64_t* launches) {
    k_topm<<<1, kTopThreads, 0, st>>>(z, n, m, keymode, seed, round, P_out, flag);
    ++*launches;
    return cudaGetLastError();
}

// =====================================================================================
// Pass permutation: P sorted by (key(seed, round, pass, j), j).  P is ascending
// and the radix sort is stable, so equal keys keep index order.
// =====================================================================================
__global__ void k_perm_keys(const int64_t* P, int64_t m, uint64_t seed, int64_t round,
                            int64_t pass, uint64_t* keys, int* idx) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) {
        keys[t] = perm_key(seed, round, pass, P[t]);
        idx[t] = (int)t;
    }
}
cudaError_t launch_perm_keys(const int64_t* P, int64_t m, uint64_t seed, int64_t round,
                             int64_t pass, uint64_t* keys, int* idx, cudaStream_t st,
                             int64_t* launches) {
    k_perm_keys<<<(unsigned)cdiv(m, 256), 256, 0, st>>>(P, m, seed, round, pass, keys, idx);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_gather_order(const int* sidx, const int64_t* P, const int* P_slot, int64_t m,
                               int64_t* order_j, int* order_slot) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) {
        int q = sidx[t];
        order_j[t] = P[q];
        order_slot[t] = P_slot[q];
    }
}
cudaError_t launch_gather_order(const int* sorted_idx, const int64_t* P, const int* P_slot,
                                int64_t m, int64_t* order_j, int* order_slot, cudaStream_t st,
                                int64_t* launches) {
    k_gather_order<<<(unsigned)cdiv(m, 256), 256, 0, st>>>(sorted_idx, P, P_slot, m, order_j,
                                                            order_slot);
    ++*launches;
    return cudaGetLastError();
}

size_t sort_temp_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int*)nullptr, (int*)nullptr, (int)m);
    return bytes;
}
cudaError_t sort_pairs(void* temp, size_t temp_bytes, const uint64_t* keys_in, uint64_t* keys_out,
                       const int* idx_in, int* idx_out, int64_t m, cudaStream_t st,
                       int64_t* launches) {
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, idx_in,
                                                    idx_out, (int)m, 0, 64, st);
    *launches += 8;  // onesweep: histogram + exclusive-sum + 8-bit passes (counted conservatively)
    return e;
}

// =====================================================================================
// Exact SCD epoch, Gram-block form (App. D closed forms executed in the exact
// sequential order).
//
// Cooperative persistent kernel, G CTAs, CTA c owns rows [cR, cR + R) of the
// shared vector v (kept in shared memory, fp64) and of every working-set column.
// For each block B of W coordinates (positions bW .. bW+W of the order):
//   1. the TMA engine stages the CTA's row slice of the W columns into shared
//      memory (cp.async.bulk, double buffered: block b+1 streams in while block
//      b computes and synchronises);
//   2. partial s_j = a_j^T v (j in B) and partial Gram G_jk = a_j^T a_k (k < j)
//      over the CTA's rows, fp64, register-tiled 4x4 per warp task;
//   3. fp64 atomics into a global reduction buffer + one grid barrier;
//   4. every CTA (redundantly, identically) runs the W closed-form updates in
//      sequence with s_j <- s_j + sum_{k<j} G_jk delta_k -- exactly sequential
//      SCD -- and CTA 0 writes alpha;
//   5. v_slice += sum_j delta_j a_j (own rows; no atomics).
// =====================================================================================
constexpr int kScdThreads = 512;
constexpr int kScdWarps = kScdThreads / 32;

__host__ __device__ __forceinline__ int scd_rc_dev(int W, int nt) {
    (void)W;
    int rc = (kScdWarps + nt - 1) / nt;
    return rc < 1 ? 1 : rc;
}
__host__ __device__ __forceinline__ size_t align_up_dev(size_t x) { return (x + 127) / 128 * 128; }
int scd_nred(int W) { return W + W * (W - 1) / 2; }
int scd_rc(int W) {
    int T = W / 4;
    return scd_rc_dev(W, T * (T + 1) / 2 + T);
}
static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
size_t scd_smem_bytes(int W, int R) {
    size_t off = 128;                                             // mbarriers
    off += align_up((size_t)2 * W * R * sizeof(float), 128);      // A slices, 2 stages
    off += align_up((size_t)R * sizeof(double), 128);             // v slice
    off += align_up((size_t)scd_rc(W) * scd_nred(W) * sizeof(double), 128);  // CTA partials
    off += align_up((size_t)scd_nred(W) * sizeof(double), 128);   // reduced s, G
    off += align_up((size_t)32 * sizeof(double), 128);            // deltas
    return off;
}

__device__ __forceinline__ void scd_issue(const ScdParams& p, float* dst, int64_t base, int Wb,
                                          int64_t r0, int rows, uint64_t* bar) {
    const unsigned bytes = (unsigned)rows * 4u;
    mbar_arrive_expect_tx(bar, bytes * (unsigned)Wb);
    for (int j = 0; j < Wb; ++j) {
        const float* src = p.pool + (int64_t)p.order_slot[base + j] * p.ld_dev + r0;
        bulk_g2s(dst + (size_t)j * p.R, src, bytes, bar);
    }
}

__global__ void __launch_bounds__(kScdThreads, 1) k_scd_gram(ScdParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = p.W, R = p.R;
    const int NRED = W + W * (W - 1) / 2;
    const int T = W / 4;
    const int NG = T * (T + 1) / 2;
    const int NT = NG + T;
    const int RC = scd_rc_dev(W, NT);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    size_t off = 128;
    float* Abuf = reinterpret_cast<float*>(smem + off);
    off += align_up_dev((size_t)2 * W * R * sizeof(float));
    double* vs = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)R * sizeof(double));
    double* acc = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)RC * NRED * sizeof(double));
    double* sG = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)NRED * sizeof(double));
    double* delta = reinterpret_cast<double*>(smem + off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = (int64_t)c * R;
    const int rows = (int)imin64(R, p.d4 - r0);
    const double dd = (double)p.d, nn = (double)p.n;

    // init: zero the stage buffers (tail rows of the last CTA stay zero), load v slice
    for (int q = tid; q < 2 * W * R; q += kScdThreads) Abuf[q] = 0.0f;
    for (int r = tid; r < R; r += kScdThreads) vs[r] = r < rows ? p.vt[r0 + r] : 0.0;
    for (int q = tid; q < RC * NRED; q += kScdThreads) acc[q] = 0.0;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();

    const int64_t nblk = (p.L + W - 1) / W;
    if (tid == 0 && nblk > 0) scd_issue(p, Abuf, 0, (int)imin64(W, p.L), r0, rows, &mbar[0]);

    for (int64_t b = 0; b < nblk; ++b) {
        const int buf = (int)(b & 1);
        const int64_t base = b * W;
        const int Wb = (int)imin64(W, p.L - base);
        float* A = Abuf + (size_t)buf * W * R;
        if (tid == 0 && b + 1 < nblk)
            scd_issue(p, Abuf + (size_t)(buf ^ 1) * W * R, base + W,
                      (int)imin64(W, p.L - base - W), r0, rows, &mbar[buf ^ 1]);
        mbar_wait(&mbar[buf], (unsigned)((b >> 1) & 1));

        // ---- 2. partial dots: tasks = Gram 4x4 tiles (jt >= kt) + s tiles, x RC row chunks
        const int chunk = (rows + RC - 1) / RC;
        for (int item = warp; item < NT * RC; item += kScdWarps) {
            const int task = item % NT, rc = item / NT;
            const int lo = rc * chunk, hi = min(rows, lo + chunk);
            double* out = acc + (size_t)rc * NRED;
            if (task < NG) {
                int jt = (int)((sqrtf(8.0f * task + 1.0f) - 1.0f) * 0.5f);
                while ((jt + 1) * (jt + 2) / 2 <= task) ++jt;
                while (jt * (jt + 1) / 2 > task) --jt;
                const int kt = task - jt * (jt + 1) / 2;
                const float* Aj = A + (size_t)(4 * jt) * R;
                const float* Ak = A + (size_t)(4 * kt) * R;
                double g[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) g[e] = 0.0;
                for (int r = lo + lane; r < hi; r += 32) {
                    double x0 = Aj[r], x1 = Aj[R + r], x2 = Aj[2 * R + r], x3 = Aj[3 * R + r];
                    double y0 = Ak[r], y1 = Ak[R + r], y2 = Ak[2 * R + r], y3 = Ak[3 * R + r];
                    g[0] = fma(x0, y0, g[0]); g[1] = fma(x0, y1, g[1]); g[2] = fma(x0, y2, g[2]); g[3] = fma(x0, y3, g[3]);
                    g[4] = fma(x1, y0, g[4]); g[5] = fma(x1, y1, g[5]); g[6] = fma(x1, y2, g[6]); g[7] = fma(x1, y3, g[7]);
                    g[8] = fma(x2, y0, g[8]); g[9] = fma(x2, y1, g[9]); g[10] = fma(x2, y2, g[10]); g[11] = fma(x2, y3, g[11]);
                    g[12] = fma(x3, y0, g[12]); g[13] = fma(x3, y1, g[13]); g[14] = fma(x3, y2, g[14]); g[15] = fma(x3, y3, g[15]);
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) g[e] = warp_sum(g[e]);
                if (lane == 0) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int j = 4 * jt + (e >> 2), k = 4 * kt + (e & 3);
                        if (k < j) out[W + j * (j - 1) / 2 + k] += g[e];
                    }
                }
            } else {
                const int jt = task - NG;
                const float* Aj = A + (size_t)(4 * jt) * R;
                double g0 = 0, g1 = 0, g2 = 0, g3 = 0;
                for (int r = lo + lane; r < hi; r += 32) {
                    const double v = vs[r];
                    g0 = fma((double)Aj[r], v, g0);
                    g1 = fma((double)Aj[R + r], v, g1);
                    g2 = fma((double)Aj[2 * R + r], v, g2);
                    g3 = fma((double)Aj[3 * R + r], v, g3);
                }
                g0 = warp_sum(g0); g1 = warp_sum(g1); g2 = warp_sum(g2); g3 = warp_sum(g3);
                if (lane == 0) {
                    out[4 * jt] += g0; out[4 * jt + 1] += g1; out[4 * jt + 2] += g2; out[4 * jt + 3] += g3;
                }
            }
        }
        __syncthreads();
        // ---- 3. cross-CTA reduction + grid barrier
        double* red_b = p.red + (size_t)(b % 3) * NRED;
        for (int q = tid; q < NRED; q += kScdThreads) {
            double v = 0.0;
            for (int rc = 0; rc < RC; ++rc) { v += acc[(size_t)rc * NRED + q]; acc[(size_t)rc * NRED + q] = 0.0; }
            atomicAdd(&red_b[q], v);
        }
        grid_barrier(p.bar, (unsigned)((b + 1) * (int64_t)p.G));
        if (c == 0)  // buffer of block b-1 is no longer read by anyone; block b+2 will use it
            for (int q = tid; q < NRED; q += kScdThreads) p.red[(size_t)((b + 2) % 3) * NRED + q] = 0.0;
        for (int q = tid; q < NRED; q += kScdThreads) sG[q] = ld_cg_f64(&red_b[q]);
        __syncthreads();
        // ---- 4. W sequential closed-form updates (warp 0; lane j owns coordinate j)
        if (warp == 0) {
            int64_t jg = 0;
            double a = 0, nrm = 0, yy = 0, sj = 0;
            if (lane < Wb) {
                jg = p.order_j[base + lane];
                a = p.alpha[jg];
                nrm = p.norms[jg];
                yy = p.model == kSvm ? p.y[jg] : 0.0;
                sj = sG[lane];
            }
            for (int j = 0; j < Wb; ++j) {
                double dl = 0.0;
                if (lane == j) {
                    double an = coord_step(p.model, a, sj, nrm, yy, p.lambda, dd, nn);
                    dl = an - a;
                    if (c == 0) p.alpha[jg] = an;
                }
                dl = __shfl_sync(~0u, dl, j);
                if (lane > j && lane < Wb) sj = fma(sG[W + lane * (lane - 1) / 2 + j], dl, sj);
                if (lane == 0) delta[j] = dl;
            }
            if (lane >= Wb && lane < W) delta[lane] = 0.0;
        }
        __syncthreads();
        // ---- 5. v slice update, sequential order of j (as in the paper's v~ update)
        for (int r = tid; r < rows; r += kScdThreads) {
            double v = vs[r];
            for (int j = 0; j < Wb; ++j) v = fma(delta[j], (double)A[(size_t)j * R + r], v);
            vs[r] = v;
        }
        __syncthreads();
    }
    for (int r = tid; r < rows; r += kScdThreads) p.vt[r0 + r] = vs[r];
}

cudaError_t launch_scd_gram(const ScdParams& p, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    size_t smem = scd_smem_bytes(p.W, p.R);
    cudaError_t e = cudaFuncSetAttribute(k_scd_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    ScdParams q = p;
    void* args[] = {&q};
    e = cudaLaunchCooperativeKernel((const void*)k_scd_gram, dim3(p.G), dim3(kScdThreads), args,
                                    smem, st);
    ++*launches;
    return e;
}

// =====================================================================================
// v = A alpha (- b): exact shared-vector recompute for set_state.  CTA per row
// tile of 1024 rows; loops over the columns with alpha_i != 0.
// =====================================================================================
__global__ void k_matvec(ColSrc src, const double* alpha, int64_t n, int64_t d, int64_t d4,
                         const double* b, double* vt) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = alpha[i];
        if (a == 0.0) continue;
        if (r < d4) acc = fma((double)col_ptr(src, i)[r], a, acc);
    }
    if (r < d4) vt[r] = (b && r < d) ? acc - b[r] : acc;
}
cudaError_t launch_matvec(const ColSrc& src, const double* alpha, int64_t n, int64_t d, int64_t d4,
                          const double* b, double* vt, cudaStream_t st, int64_t* launches) {
    k_matvec<<<(unsigned)cdiv(d4, 256), 256, 0, st>>>(src, alpha, n, d, d4, b, vt);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_set_slots(int* col_slot, const int64_t* cols, const int* slots, int64_t cnt) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < cnt) col_slot[cols[t]] = slots[t];
}
cudaError_t launch_set_slots(int* col_slot, const int64_t* cols, const int* slots, int64_t cnt,
                             cudaStream_t st, int64_t* launches) {
    if (cnt <= 0) return cudaSuccess;
    k_set_slots<<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(col_slot, cols, slots, cnt);
    ++*launches;
    return cudaGetLastError();
}

// out2[0] += ||vt||^2, out2[1] += vt^T b (b may be null)
__global__ void k_vec_sums(const double* vt, const double* b, int64_t d4, double* out2) {
    double s0 = 0, s1 = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d4;
         r += (int64_t)gridDim.x * blockDim.x) {
        double v = vt[r];
        s0 = fma(v, v, s0);
        if (b) s1 = fma(v, b[r], s1);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    __shared__ double sh[2][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { sh[0][warp] = s0; sh[1][warp] = s1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += sh[0][w]; c += sh[1][w]; }
        atomicAdd(&out2[0], a);
        atomicAdd(&out2[1], c);
    }
}
cudaError_t launch_vec_sums(const double* vt, const double* b, int64_t d4, double* out2,
                            cudaStream_t st, int64_t* launches) {
    k_vec_sums<<<(unsigned)imin64(cdiv(d4, 256), 296), 256, 0, st>>>(vt, b, d4, out2);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace duhl
