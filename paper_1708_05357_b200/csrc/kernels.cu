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
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

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
    double g = coord_gap(p.model, a, s, yy, p.lambda, p.B, (double)p.d, (double)p.n, &scale, &aux, p.eta);
    if (!isfinite(g)) flag |= 2;
    else if (g < -1e-12 * (scale > 1.0 ? scale : 1.0)) flag |= 1;
    double gz = g > 0.0 ? g : 0.0;  // gap_i >= 0 in exact arithmetic: clamp at +0.0 (reading R17)
    if (p.z) p.z[i] = gz;
    if (p.gap_out) p.gap_out[t] = gz;
    if (p.s_out) p.s_out[t] = s;
    acc.g += gz;
    acc.aux += aux;
    acc.a += p.model == kLasso ? fabs(a)
             : p.model == kRidge ? a * a
             : p.model == kElastic ? 0.5 * p.eta * a * a + (1.0 - p.eta) * fabs(a) : yy * a;
    acc.amax = fmax(acc.amax, fabs(a));
}

template <int NT = kGapThreads>
__device__ void block_flush_sums(const GapParams& p, SumAcc acc, int flag) {
    __shared__ double sh[4][NT / 32];
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
            for (int w = 0; w < NT / 32; ++w) {
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

// Work item vb = (column group vb % ngroups, row tile vb / ngroups); a grid
// smaller than the item count loops (a persistent unit-A grid beside the SCD epoch).
// INGEST (duhl_create's one pass over A): also ||a_i||^2 into
// p.norms_out (fp64; added atomically across row tiles, zero on entry) -- a non-finite
// element makes it non-finite, which is how create detects invalid data -- and, for
// columns i < p.fill_cols, the column itself into HBM slot i (the pass reads it anyway).
template <bool INGEST>
__global__ void __launch_bounds__(kGapThreads, 4) k_gap_tile(GapParams p, int tile_rows, int ntiles, int64_t ngroups) {
    extern __shared__ double ws[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const double2* w2 = reinterpret_cast<const double2*>(ws);
    SumAcc acc;
    int flag = 0;
    int64_t cur_tile = -1;
    for (int64_t vb = blockIdx.x; vb < ngroups * ntiles; vb += gridDim.x) {
    const int64_t tile = vb / ngroups;
    const int64_t r0 = tile * tile_rows;
    const int rows = (int)imin64(tile_rows, p.d4 - r0);  // multiple of 4
    if (tile != cur_tile) {
        __syncthreads();
        for (int r = threadIdx.x; r < rows; r += blockDim.x) ws[r] = p.vt[r0 + r] * p.wscale;
        __syncthreads();
        cur_tile = tile;
    }
    const int64_t t0 = (vb % ngroups) * kGapColsPerCta;
    const int64_t t1 = imin64(p.k, t0 + kGapColsPerCta);
    const int nv = rows >> 2;
    for (int64_t t = t0 + warp; t < t1; t += nw) {
        const int64_t i = p.cols ? p.cols[t] : t;
        const float4* a = reinterpret_cast<const float4*>(col_ptr(p.src, i) + r0);
        double s0 = 0.0, s1 = 0.0, n0 = 0.0, n1 = 0.0;
        auto sq = [&](const float4& f) {
            if (INGEST) {
                n0 = fma((double)f.x, (double)f.x, n0); n1 = fma((double)f.y, (double)f.y, n1);
                n0 = fma((double)f.z, (double)f.z, n0); n1 = fma((double)f.w, (double)f.w, n1);
            }
        };
        // INGEST: the first fill_cols columns also land in their HBM slots (slot i = column i)
        float4* fill = (INGEST && i < p.fill_cols)
                           ? reinterpret_cast<float4*>(p.fill_pool + i * p.fill_ld + r0) : nullptr;
        int q = lane;
        for (; q + 96 < nv; q += 128) {  // 4 independent 16-B loads in flight per lane
            float4 f0 = ld_stream_f4(a + q), f1 = ld_stream_f4(a + q + 32);
            float4 f2 = ld_stream_f4(a + q + 64), f3 = ld_stream_f4(a + q + 96);
            sq(f0); sq(f1); sq(f2); sq(f3);
            if (INGEST && fill) {
                __stcs(fill + q, f0); __stcs(fill + q + 32, f1);
                __stcs(fill + q + 64, f2); __stcs(fill + q + 96, f3);
            }
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
            sq(f);
            if (INGEST && fill) __stcs(fill + q, f);
            double2 u = w2[2 * q], v = w2[2 * q + 1];
            s0 = fma((double)f.x, u.x, s0); s1 = fma((double)f.y, u.y, s1);
            s0 = fma((double)f.z, v.x, s0); s1 = fma((double)f.w, v.y, s1);
        }
        double s = warp_sum(s0 + s1);
        if (INGEST) {
            const double nr = warp_sum(n0 + n1);
            if (lane == 0) {
                if (ntiles == 1) p.norms_out[i] = nr;
                else atomicAdd(&p.norms_out[i], nr);
            }
        }
        if (lane == 0) {
            if (ntiles == 1) gap_finish_one(p, t, i, s, acc, flag);
            else atomicAdd(&p.s_acc[t], s);
        }
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

cudaError_t launch_gap_pass(const GapParams& p, int tile_rows, cudaStream_t st, int64_t* launches, int max_ctas) {
    if (p.k <= 0) return cudaSuccess;
    int ntiles = (int)cdiv(p.d4, tile_rows);
    if (ntiles == 1) tile_rows = (int)p.d4;
    const int64_t ngroups = cdiv(p.k, kGapColsPerCta);
    int64_t items = ngroups * ntiles;
    if (max_ctas > 0 && items > max_ctas) items = max_ctas;
    size_t smem = (size_t)tile_rows * sizeof(double);
    const void* fn = p.norms_out ? (const void*)k_gap_tile<true> : (const void*)k_gap_tile<false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (p.norms_out) k_gap_tile<true><<<(unsigned)items, kGapThreads, smem, st>>>(p, tile_rows, ntiles, ngroups);
    else k_gap_tile<false><<<(unsigned)items, kGapThreads, smem, st>>>(p, tile_rows, ntiles, ngroups);
    ++*launches;
    if (ntiles > 1) {
        k_gap_finalize<<<(unsigned)cdiv(p.k, kGapThreads), kGapThreads, 0, st>>>(p);
        ++*launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_gap_finalize(const GapParams& p, cudaStream_t st, int64_t* launches) {
    if (p.k <= 0) return cudaSuccess;
    k_gap_finalize<<<(unsigned)cdiv(p.k, kGapThreads), kGapThreads, 0, st>>>(p);
    ++*launches;
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
// z_i >= +0 (nonnegative doubles order as uint64); keymode 2 = importance clocks
// (see select_key); keymode 1 = ~key(seed,
// round, -1, i) (uniform baseline: the m smallest counter keys).
// One CTA of 1024 threads; 11-bit digits, 6 passes.  P_out ascending.
// =====================================================================================
constexpr int kTopThreads = 1024;
constexpr int kRadixBits = 11;
constexpr int kBins = 1 << kRadixBits;
constexpr int64_t kTopmSmallN = 1 << 17;  // one CTA up to here, the multi-CTA form beyond

__device__ __forceinline__ uint64_t select_key(const double* z, int64_t i, int keymode,
                                               uint64_t seed, int64_t round, int* bad) {
    if (keymode == 1) return ~perm_key(seed, round, -1, i);
    if (keymode == 2) {
        // importance sampling: m draws without replacement with probability
        // proportional to ||a_i||^2 = the m smallest exponential clocks -ln(u_i)/||a_i||^2
        // (z = norms); nonnegative doubles order as their bits, ~ turns smallest into largest
        const double w = z[i];
        const double u = ((double)(perm_key(seed, round, -2, i) >> 11) + 0.5) * 0x1p-53;
        const double e = w > 0.0 ? -log(u) / w : __longlong_as_double(0x7ff0000000000000ll);
        return ~(uint64_t)__double_as_longlong(e);
    }
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

// ---- multi-CTA form for large n (same semantics, same output): per digit, a
// grid-wide histogram of the candidate keys + a one-CTA pick of the digit; then
// per-chunk counts, a one-CTA scan of the chunk offsets, and an in-order write.
struct TopmState {
    unsigned long long prefix, pmask;
    long long need;
};
constexpr int kTopChunks = 1024;  // CTAs (and contiguous index chunks) of the multi-CTA form

__global__ void __launch_bounds__(kTopThreads) k_topm_hist(const double* z, int64_t n, int keymode, uint64_t seed,
                                                           int64_t round, const TopmState* stt, int shift,
                                                           int nbits, int* ghist, int* flag) {
    __shared__ int hist[kBins];
    const int tid = threadIdx.x;
    for (int b = tid; b < kBins; b += kTopThreads) hist[b] = 0;
    __syncthreads();
    const unsigned long long prefix = stt->prefix, pmask = stt->pmask, dmask = (1ull << nbits) - 1;
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * kTopThreads + tid; i < n; i += (int64_t)gridDim.x * kTopThreads) {
        const uint64_t k = select_key(z, i, keymode, seed, round, &bad);
        if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & dmask], 1);
    }
    __syncthreads();
    for (int b = tid; b < kBins; b += kTopThreads)
        if (hist[b]) atomicAdd(&ghist[b], hist[b]);
    if (bad && shift == 64 - kRadixBits) atomicOr(flag, 1);
}

__global__ void __launch_bounds__(kTopThreads) k_topm_pick(int* ghist, TopmState* stt, int shift, int nbits) {
    typedef cub::BlockScan<int, kTopThreads> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_digit, s_above;
    const int tid = threadIdx.x;
    const long long need = stt->need;
    const int e0 = kBins - 1 - 2 * tid, e1 = e0 - 1;
    const int c0 = ghist[e0], c1 = ghist[e1];
    int excl;
    Scan(scan_tmp).ExclusiveSum(c0 + c1, excl);
    if (excl < need && need <= excl + c0) { s_digit = e0; s_above = excl; }
    else if (excl + c0 < need && need <= excl + c0 + c1) { s_digit = e1; s_above = excl + c0; }
    __syncthreads();
    ghist[e0] = 0;  // ready for the next digit
    ghist[e1] = 0;
    if (tid == 0) {
        stt->need = need - s_above;
        stt->prefix |= (unsigned long long)s_digit << shift;
        stt->pmask |= ((1ull << nbits) - 1) << shift;
    }
}

// per chunk: keys above the threshold and keys equal to it
__global__ void __launch_bounds__(kTopThreads) k_topm_count(const double* z, int64_t n, int keymode, uint64_t seed,
                                                            int64_t round, const TopmState* stt, int64_t chunk,
                                                            int* cnt) {
    typedef cub::BlockReduce<int, kTopThreads> Red;
    __shared__ typename Red::TempStorage tmp;
    const unsigned long long thr = stt->prefix;
    int gt = 0, eq = 0, bad = 0;
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = imin64(n, lo + chunk);
    for (int64_t i = lo + threadIdx.x; i < hi; i += kTopThreads) {
        const uint64_t k = select_key(z, i, keymode, seed, round, &bad);
        gt += k > thr;
        eq += k == thr;
    }
    gt = Red(tmp).Sum(gt);
    __syncthreads();
    eq = Red(tmp).Sum(eq);
    if (threadIdx.x == 0) {
        cnt[2 * blockIdx.x] = gt;
        cnt[2 * blockIdx.x + 1] = eq;
    }
}

// chunk offsets: eq keys before the chunk, then the output position of its first kept key
__global__ void __launch_bounds__(kTopThreads) k_topm_offsets(int* cnt, const TopmState* stt, int nch) {
    typedef cub::BlockScan<long long, kTopThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int c = threadIdx.x;
    const long long gt = c < nch ? cnt[2 * c] : 0, eq = c < nch ? cnt[2 * c + 1] : 0;
    long long eq_before;
    Scan(tmp).ExclusiveSum(eq, eq_before);
    __syncthreads();
    const long long need = stt->need;
    long long eq_take = need - eq_before;
    eq_take = eq_take < 0 ? 0 : (eq_take > eq ? eq : eq_take);
    long long out;
    Scan(tmp).ExclusiveSum(gt + eq_take, out);
    if (c < nch) {
        cnt[2 * c] = (int)out;         // output offset of the chunk
        cnt[2 * c + 1] = (int)eq_before;  // equal keys before the chunk
    }
}

__global__ void __launch_bounds__(kTopThreads) k_topm_write(const double* z, int64_t n, int keymode, uint64_t seed,
                                                            int64_t round, const TopmState* stt, int64_t chunk,
                                                            const int* cnt, int64_t* P_out) {
    typedef cub::BlockScan<int, kTopThreads> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    const int tid = threadIdx.x;
    const unsigned long long thr = stt->prefix;
    const long long need = stt->need;
    long long base = cnt[2 * blockIdx.x], eqbase = cnt[2 * blockIdx.x + 1];
    int bad = 0;
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = imin64(n, lo + chunk);
    for (int64_t i0 = lo; i0 < hi; i0 += kTopThreads) {
        const int64_t i = i0 + tid;
        int gt = 0, eq = 0;
        if (i < hi) {
            const uint64_t k = select_key(z, i, keymode, seed, round, &bad);
            gt = k > thr;
            eq = k == thr;
        }
        int eq_excl, eq_tot;
        Scan(scan_tmp).ExclusiveSum(eq, eq_excl, eq_tot);
        __syncthreads();
        const int take = gt || (eq && (eqbase + eq_excl) < need);
        int pos, tot;
        Scan(scan_tmp).ExclusiveSum(take, pos, tot);
        if (take) P_out[base + pos] = i;
        base += tot;
        eqbase += eq_tot;
        __syncthreads();
    }
}

cudaError_t launch_topm(const double* z, int64_t n, int64_t m, int keymode, uint64_t seed,
                        int64_t round, int64_t* P_out, int* flag, cudaStream_t st,
                        int64_t* launches, void* work) {
    if (m <= 0) return cudaSuccess;
    if (n <= kTopmSmallN || !work) {
        k_topm<<<1, kTopThreads, 0, st>>>(z, n, m, keymode, seed, round, P_out, flag);
        ++*launches;
        return cudaGetLastError();
    }
    // work: TopmState | ghist[kBins] | cnt[2 kTopChunks]  (launch_topm_work_bytes)
    TopmState* stt = reinterpret_cast<TopmState*>(work);
    int* ghist = reinterpret_cast<int*>(reinterpret_cast<char*>(work) + 64);
    int* cnt = ghist + kBins;
    TopmState init{0ull, 0ull, (long long)m};
    cudaError_t e = cudaMemcpyAsync(stt, &init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ghist, 0, kBins * sizeof(int), st);
    if (e != cudaSuccess) return e;
    const int grid = (int)imin64(kTopChunks, cdiv(n, 4 * kTopThreads));
    for (int hi = 64; hi > 0;) {
        const int nbits = hi < kRadixBits ? hi : kRadixBits;
        const int shift = hi - nbits;
        k_topm_hist<<<grid, kTopThreads, 0, st>>>(z, n, keymode, seed, round, stt, shift, nbits, ghist, flag);
        k_topm_pick<<<1, kTopThreads, 0, st>>>(ghist, stt, shift, nbits);
        *launches += 2;
        hi = shift;
    }
    const int64_t chunk = cdiv(n, grid);
    k_topm_count<<<grid, kTopThreads, 0, st>>>(z, n, keymode, seed, round, stt, chunk, cnt);
    k_topm_offsets<<<1, kTopThreads, 0, st>>>(cnt, stt, grid);
    k_topm_write<<<grid, kTopThreads, 0, st>>>(z, n, keymode, seed, round, stt, chunk, cnt, P_out);
    *launches += 3;
    return cudaGetLastError();
}

size_t launch_topm_work_bytes() { return 64 + kBins * sizeof(int) + 2 * kTopChunks * sizeof(int); }

// =====================================================================================
// Working-set staging host -> HBM by a zero-copy gather (light rounds, Alg. 2 l.4).
// The copy engine moves one 803-KB C4 column per cudaMemcpyAsync at 42.7 GB/s on this
// box (per-copy overhead; 1, 2, 4 or 8 streams alike), 16 CTAs of this kernel read
// scattered pinned host columns at 51.5 GB/s (tools/micro/stage.cu).  CTA c copies plan
// entries q = c, c + G, c + 2G, ... in order (4 x 16-byte loads in flight per thread)
// and then publishes progress[c] = entries done (release); the SCD kernels wait for
// entry q on progress[q % G] > q / G (wait_staged), so the epoch consumes columns as
// they land.
// =====================================================================================
constexpr int kStageThreads = 256;
constexpr int kStageUnroll = 8;  // 16-byte loads in flight per thread (32 KB per CTA)
__global__ void __launch_bounds__(kStageThreads) k_stage_gather(const float* host, int64_t ld_host, float* pool,
                                                                 int64_t ld_dev, int64_t d4, const int64_t* cols,
                                                                 const int* slots, int64_t nplan, unsigned* progress) {
    const int64_t n4 = d4 / 4;
    unsigned done = 0;
    for (int64_t q = blockIdx.x; q < nplan; q += gridDim.x) {
        const float4* src = reinterpret_cast<const float4*>(host + cols[q] * ld_host);
        float4* dst = reinterpret_cast<float4*>(pool + (int64_t)slots[q] * ld_dev);
        int64_t i = threadIdx.x;
        for (; i + (kStageUnroll - 1) * kStageThreads < n4; i += kStageUnroll * kStageThreads) {
            float4 x[kStageUnroll];
            // plain loads: 45.1 vs 43.2 GB/s with ld.global.nc.L1::no_allocate inside the C4 step
#pragma unroll
            for (int u = 0; u < kStageUnroll; ++u) x[u] = src[i + u * kStageThreads];
#pragma unroll
            for (int u = 0; u < kStageUnroll; ++u) dst[i + u * kStageThreads] = x[u];
        }
        for (; i < n4; i += kStageThreads) dst[i] = src[i];
        // the consumer reads the slot with the TMA engine (async proxy): order this thread's
        // generic-proxy stores before the async proxy, then device-wide before the release
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release_gpu_u32(progress + (size_t)blockIdx.x * kProgressStride, ++done);
    }
}

cudaError_t launch_stage_gather(const float* host, int64_t ld_host, float* pool, int64_t ld_dev, int64_t d4,
                                const int64_t* cols, const int* slots, int64_t nplan, unsigned* progress,
                                int ctas, cudaStream_t st, int64_t* launches) {
    if (nplan <= 0) return cudaSuccess;
    k_stage_gather<<<ctas, kStageThreads, 0, st>>>(host, ld_host, pool, ld_dev, d4, cols, slots, nplan, progress);
    ++*launches;
    return cudaGetLastError();
}

// =====================================================================================
// Pass permutation: position t takes P[pi(t)], pi a
// keyed 8-round Feistel bijection on [0, 4^h) >= m, restricted to [0, m) by
// cycle walking.  One thread per position, no sort.
// =====================================================================================
__device__ __forceinline__ int64_t feistel_index(uint64_t key, int h, int64_t m, int64_t t) {
    const uint64_t mask = (1ull << h) - 1;
    uint64_t x = (uint64_t)t;
    do {
        uint64_t L = x >> h, R = x & mask;
#pragma unroll
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

// Per-position inputs of a pass, gathered once before the launch: the
// coordinate, its HBM slot and staging sequence number, alpha at the start of
// the pass (each coordinate is visited once per pass, so this is also its value
// at the visit), 1/||a_j||^2 (-1 marks a zero column) and y_j.
struct OrderOut {
    int64_t* j;
    int* slot;
    unsigned* batch;
    double *a, *inv, *y;
};
// inv: 1/||a_j||^2 (-1: zero column); ridge (ridge_ld = lambda d > 0): 1/(||a_j||^2 + lambda d)
__device__ __forceinline__ void order_info(const OrderOut& o, int64_t t, int64_t j, const double* alpha,
                                           const double* norms, const double* y, double ridge_ld) {
    const double nrm = norms[j];
    o.a[t] = alpha[j];
    o.inv[t] = ridge_ld > 0.0 ? 1.0 / (nrm + ridge_ld) : (nrm > 0.0 ? 1.0 / nrm : -1.0);
    o.y[t] = y ? y[j] : 0.0;
}

__global__ void k_perm_order(const int64_t* P, const int* P_slot, const unsigned* P_batch, int64_t m,
                             uint64_t key, int h, OrderOut o, const double* alpha, const double* norms,
                             const double* y, double ridge_ld) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) {
        int64_t q = feistel_index(key, h, m, t);
        const int64_t j = P[q];
        o.j[t] = j;
        o.slot[t] = P_slot[q];
        o.batch[t] = P_batch[q];
        order_info(o, t, j, alpha, norms, y, ridge_ld);
    }
}

__global__ void k_order_info(int64_t L, OrderOut o, const double* alpha, const double* norms, const double* y,
                             double ridge_ld) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < L) order_info(o, t, o.j[t], alpha, norms, y, ridge_ld);
}

cudaError_t launch_perm_order(const int64_t* P, const int* P_slot, const unsigned* P_batch, int64_t m,
                              uint64_t seed, int64_t round, int64_t pass, int64_t* order_j,
                              int* order_slot, unsigned* order_batch, double* order_a, double* order_inv,
                              double* order_y, const double* alpha, const double* norms, const double* y,
                              cudaStream_t st, int64_t* launches, double ridge_ld) {
    if (m <= 0) return cudaSuccess;
    OrderOut o{order_j, order_slot, order_batch, order_a, order_inv, order_y};
    if (P == nullptr) {  // explicit order already in order_j / slot / batch: gather the rest
        k_order_info<<<(unsigned)cdiv(m, 256), 256, 0, st>>>(m, o, alpha, norms, y, ridge_ld);
    } else {
        int h = 1;
        while ((1ll << (2 * h)) < m) ++h;
        uint64_t key = mix64(mix64(mix64(seed) ^ (uint64_t)round) ^ (uint64_t)pass);
        k_perm_order<<<(unsigned)cdiv(m, 256), 256, 0, st>>>(P, P_slot, P_batch, m, key, h, o, alpha,
                                                              norms, y, ridge_ld);
    }
    ++*launches;
    return cudaGetLastError();
}

// =====================================================================================
// Exact SCD epoch, Gram-block form (App. D closed forms executed in the exact
// sequential order).  Cooperative persistent kernel,
// G CTAs; CTA c owns rows [cR, cR + R) of the shared vector v (in shared
// memory, fp64) and of every working-set column, streamed in by the TMA engine
// (cp.async.bulk + mbarrier, 3 stages).
// =====================================================================================
constexpr int kScdThreads = 256;
constexpr int kScdWarps = kScdThreads / 32;
constexpr int kScdStages = 3;
constexpr int kRedBufs = 6;     // rotating reduction buffers (see the zeroing rule below)
#ifndef DUHL_RED_GROUPS
#define DUHL_RED_GROUPS 1
#endif
constexpr int kRedGroups = DUHL_RED_GROUPS;  // CTA c adds into group c % kRedGroups ...
#ifndef DUHL_RED_STRIDE
#define DUHL_RED_STRIDE 4
#endif
constexpr int kRedStride = DUHL_RED_STRIDE;  // ... one 32-byte sector per (entry, group): the fp64
                                // atomics of 148 CTAs spread over sectors, the read-back over few lines

// Reduction entries of a block of W coordinates:
//   u_j   = a_j^T v_(block start)           [0, W)
//   G_jk  = a_j^T a_k, k < j (this block)   W + j(j-1)/2 + k
//   C_jk  = a_j^T a'_k (previous block)     W + W(W-1)/2 + j W + k
__host__ __device__ __forceinline__ int scd_off_G(int W) { return W; }
__host__ __device__ __forceinline__ int scd_off_C(int W) { return W + W * (W - 1) / 2; }
__host__ __device__ int scd_nred(int W) { return W + W * (W - 1) / 2 + W * W; }
size_t scd_red_doubles(int W) { return (size_t)kRedBufs * scd_nred(W) * kRedGroups * kRedStride; }
__host__ __device__ __forceinline__ size_t align_up_dev(size_t x) { return (x + 127) / 128 * 128; }
size_t scd_smem_bytes(int W, int R, int NB) {
    (void)NB;
    size_t off = 128;                                                             // mbarriers
    off += align_up_dev((size_t)kScdStages * W * R * sizeof(float));              // A stages
    off += align_up_dev((size_t)R * sizeof(double));                              // v slice
    off += align_up_dev((size_t)scd_nred(W) * sizeof(double));                    // reduced block
    off += align_up_dev((size_t)2 * 16 * sizeof(double));                         // deltas (2 blocks)
    return off;
}

// Warp reduce-scatter: on return lane l holds the warp-wide sum of g[l % N]
// (N - 1 shuffles instead of 5 N).
template <typename T, int N>
__device__ __forceinline__ T reduce_scatter(T (&g)[N], int lane) {
#pragma unroll
    for (int half = N / 2, off = N / 2; half >= 1; half >>= 1, off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            T send = upper ? g[i] : g[i + half];
            T keep = upper ? g[i + half] : g[i];
            g[i] = keep + __shfl_xor_sync(~0u, send, off);
        }
    }
    T v = g[0];
#pragma unroll
    for (int off = N; off < 32; off <<= 1) v += __shfl_xor_sync(~0u, v, off);
    return v;
}

// 4 x KW register tile over rows [lo, hi) (multiples of 4): lane l takes the
// 4-row group starting at lo + 4 l (+ 128 i), 16-byte shared loads.  Output
// element (a, q) -> row j = jbase + a, column k = kbase + q of G (LOWER, kept
// where k < j) or C.  EXACT: fp64 products/accumulation (fp32 -> fp64 exact);
// fast: fp32 FFMA inside the warp, fp64 from the warp reduction on.
// Where a tile's reduced entries go: fp64 REDs into the block's rotating
// reduction buffer, group grp (see kRedGroups), one 256-byte line per entry.
struct RedOut {
    double* buf;
    int grp;
    __device__ __forceinline__ void add(int q, double v) const {
#ifndef DUHL_EXP_NORED  // developer timing experiment only: results are wrong without the REDs
        atomicAdd(&buf[((size_t)q * kRedGroups + grp) * kRedStride], v);
#endif
    }
};

// XL (the pipelined kernel's expanded layout, see pipe_ne): G_jk at W + k W + j,
// C_jk at W + W^2 + k W + j, so the control warp reads rows with consecutive lanes.
template <bool EXACT, int KW, bool LOWER, bool XL = false>
__device__ __forceinline__ void tile4(const float* __restrict__ Aj, const float* __restrict__ Ak, int R,
                                      int lo, int hi, int lane, int jbase, int kbase, const RedOut& out,
                                      int W) {
    typedef typename std::conditional<EXACT, double, float>::type T;
    T g[4 * KW];
    const float4* xj[4];
    const float4* yk[KW];
#pragma unroll
    for (int a = 0; a < 4; ++a) xj[a] = reinterpret_cast<const float4*>(Aj + (size_t)a * R);
#pragma unroll
    for (int q = 0; q < KW; ++q) yk[q] = reinterpret_cast<const float4*>(Ak + (size_t)q * R);
    if (EXACT) {
#pragma unroll
        for (int e = 0; e < 4 * KW; ++e) g[e] = T(0);
        for (int r4 = (lo >> 2) + lane; r4 < (hi >> 2); r4 += 32) {
            float4 x[4], y[KW];
#pragma unroll
            for (int a = 0; a < 4; ++a) x[a] = xj[a][r4];
#pragma unroll
            for (int q = 0; q < KW; ++q) y[q] = yk[q][r4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int q = 0; q < KW; ++q) {
                    T acc = g[a * KW + q];
                    acc = fma((T)x[a].x, (T)y[q].x, acc);
                    acc = fma((T)x[a].y, (T)y[q].y, acc);
                    acc = fma((T)x[a].z, (T)y[q].z, acc);
                    acc = fma((T)x[a].w, (T)y[q].w, acc);
                    g[a * KW + q] = acc;
                }
        }
    } else {  // packed: rows (r, r+1) and (r+2, r+3) of a lane's 4-row group in FFMA2 halves
        float2 g2[4 * KW];
#pragma unroll
        for (int e = 0; e < 4 * KW; ++e) g2[e] = make_float2(0.f, 0.f);
#ifdef DUHL_EXP_NOFMA  // developer timing experiment only: no tile arithmetic
        hi = lo;
#endif
        for (int r4 = (lo >> 2) + lane; r4 < (hi >> 2); r4 += 32) {
            float4 x[4], y[KW];
#pragma unroll
            for (int a = 0; a < 4; ++a) x[a] = xj[a][r4];
#pragma unroll
            for (int q = 0; q < KW; ++q) y[q] = yk[q][r4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int q = 0; q < KW; ++q) {
                    ffma2(g2[a * KW + q], x[a].x, x[a].y, y[q].x, y[q].y);
                    ffma2(g2[a * KW + q], x[a].z, x[a].w, y[q].z, y[q].w);
                }
        }
#pragma unroll
        for (int e = 0; e < 4 * KW; ++e) g[e] = (T)(g2[e].x + g2[e].y);
    }
    const double v = (double)reduce_scatter<T, 4 * KW>(g, lane);
    if (lane < 4 * KW) {
        const int j = jbase + lane / KW, k = kbase + lane % KW;
        if (LOWER) {
            if (k < j) out.add(XL ? W + k * W + j : scd_off_G(W) + j * (j - 1) / 2 + k, v);
        } else {
            out.add(XL ? W + W * W + k * W + j : scd_off_C(W) + j * W + k, v);
        }
    }
}

// u tile: 4 x 1 against the fp64 v slice (always fp64)
__device__ __forceinline__ void utile(const float* __restrict__ Aj, const double* __restrict__ vs, int R,
                                      int lo, int hi, int lane, int jbase, const RedOut& out) {
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    const double2* v2 = reinterpret_cast<const double2*>(vs);
    for (int r4 = (lo >> 2) + lane; r4 < (hi >> 2); r4 += 32) {
        const double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float4 x = reinterpret_cast<const float4*>(Aj + (size_t)a * R)[r4];
            double t = g[a];
            t = fma((double)x.x, v01.x, t);
            t = fma((double)x.y, v01.y, t);
            t = fma((double)x.z, v23.x, t);
            t = fma((double)x.w, v23.y, t);
            g[a] = t;
        }
    }
    const double v = reduce_scatter<double, 4>(g, lane);
    if (lane < 4) out.add(jbase + lane, v);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Bounded spin-waits: a wait that cannot be satisfied (e.g. a profiler that
// serialises the copy stream behind this kernel) sets ScdParams::err and lets
// the kernel drain instead of hanging the device; the host reports DUHL_E_CUDA.
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;  // 4 s

// Stage the CTA's row slice of block blk's columns into shared memory with the
// TMA engine.  Called by a whole warp: lane j fetches the slot of column j (one
// parallel L2 round trip instead of W dependent ones) and issues its own bulk
// copy; lane 0 arms the stage's mbarrier with the total byte count first.
// Stage the CTA's row slice of block blk's columns into shared memory with the
// TMA engine.  Called by a whole warp: lane j issues the bulk copy of column j
// (slot / staging sequence number prefetched by the caller); lane 0 arms the
// stage's mbarrier with the total byte count first.  A column still in flight
// host -> HBM is waited for on the copy-progress counter (cached per lane).
__device__ __forceinline__ void scd_issue(const ScdParams& p, float* Abuf, uint64_t* mbar, int64_t blk,
                                          int64_t r0, int rows, int lane, int slot, unsigned need,
                                          unsigned& seen) {
    const int W = p.W;
    const int64_t base = blk * W;
    const int Wb = (int)imin64(W, p.L - base);
    const int st = (int)(blk % kScdStages);
    float* dst = Abuf + (size_t)st * W * p.R;
    const unsigned bytes = (unsigned)rows * 4u;
    if (lane < Wb) wait_staged(p.progress, p.stage_ctas, need, seen, p.err, kSpinTimeoutNs);  // never hangs
    // (the stage's last generic accesses are reads, completed before the CTA barrier
    // that precedes this refill: no proxy fence is needed for that order)
    if (lane == 0) mbar_arrive_expect_tx(&mbar[st], bytes * (unsigned)Wb);
    __syncwarp();
    if (lane < Wb) bulk_g2s(dst + (size_t)lane * p.R, p.pool + (int64_t)slot * p.ld_dev + r0, bytes, &mbar[st]);
}

// =====================================================================================
// k_scd_gram: exact sequential SCD epoch, Gram-block form, warp-specialised.
// Per block b of W coordinates (in visiting order):
//   compute warps (6): v_slice += A_{b-1} delta^{(b-1)} (the previous block's
//      update), then the partials of block b+1 over the CTA's rows -- G_{b+1}
//      (lower), the cross Gram C_{b+1,b} = A_{b+1}^T A_b and u_{b+1} = A_{b+1}^T v_b
//      (v_b = v at the start of block b) -- REDed straight from the tile registers
//      into red[(b+1) % 6]; the last warp done ARRIVEs(b+1) on the grid barrier.
//   control warp: WAIT(b) (arrived while block b-1 was being solved) -> reads the
//      reduced block -> runs the W closed-form steps in order with
//        s_j = u_j + sum_k C_jk delta^{(b-1)}_k + sum_{k<j} G_jk delta_k
//      (== a_j^T v at the moment coordinate j is visited: exactly sequential SCD)
//      -> publishes delta^{(b)} (mbarrier dfull[b & 1]).
//   producer warp: streams block b+3 into the stage block b freed (mbarrier
//      empty[] per stage, TMA bulk copies completing on full[]).
// The control chain (read + steps) and the compute chain (update + tiles) of
// consecutive blocks overlap; the grid barrier's latency hides behind both.
// Zeroing rule: CTA 0's control warp zeroes red[(b+4) % 6] right after WAIT(b).
// All reads of it (control(b-2), every CTA) precede every CTA's ARRIVE(b)
// (compute warps arrive only after consuming delta^{(b-2)}); its next writer
// (partials of block b+4, iteration b+3) waits on delta^{(b+2)}, which needs
// CTA 0's ARRIVE(b+2), issued after CTA 0 consumed delta^{(b)} (after the zeroing).
// =====================================================================================
// Warp layout (warps w and w+4 share SMSP w % 4): control = warp 3 (its SMSP
// otherwise holds only the mostly-waiting producer, warp 7); compute = 0,1,2,4,5,6.
constexpr int kCompute = kScdWarps - 2;
constexpr int kCtrlWarp = 3;
constexpr int kProdWarp = kScdWarps - 1;
constexpr int kBarCompute = 1;  // named barrier id: compute warps only

template <bool EXACT, int MODEL>
__global__ void __launch_bounds__(kScdThreads, 1) k_scd_gram(const __grid_constant__ ScdParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = p.W, R = p.R, T = W / 4;
    const int NRED = scd_nred(W);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [3] stage data landed
    uint64_t* empty = full + kScdStages;                 // [3] stage consumed
    uint64_t* dfull = empty + kScdStages;                // [2] delta of a block published
    size_t off = 128;
    float* Abuf = reinterpret_cast<float*>(smem + off);
    off += align_up_dev((size_t)kScdStages * W * R * sizeof(float));
    double* vs = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)R * sizeof(double));
    double* sG = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)NRED * sizeof(double));
    double* delta = reinterpret_cast<double*>(smem + off);  // [2][16]
    __shared__ double sT[16], sP[16], sA[16], sS[16], sC[16 * 16];
    __shared__ int sZ[16];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = (int64_t)c * R;
    const int rows = (int)imin64(R, p.d4 - r0);
    const double lam_dn = MODEL != kSvm ? p.lambda * (double)p.d : p.lambda * (double)p.n;
    const size_t bufsz = (size_t)NRED * kRedGroups * kRedStride;
    const int grp = c % kRedGroups;

    for (int q = tid; q < kScdStages * W * R; q += kScdThreads) Abuf[q] = 0.0f;
    for (int r = tid; r < R; r += kScdThreads) vs[r] = r < rows ? p.vt[r0 + r] : 0.0;
    if (tid == 0) {
        for (int q = 0; q < kScdStages; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kCompute);
        }
        mbar_init(&dfull[0], 1);
        mbar_init(&dfull[1], 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();

    // developer trace (ScdParams::trace): per-phase cycle counts of CTA 0 / CTA G-1
    // (control warp lane 0: slots 0-4; compute warp 0 lane 0: slots 5-7)
    const bool trc_cta = p.trace && (c == 0 || c == p.G - 1);
    const bool tr = trc_cta && (tid == kCtrlWarp * 32 || tid == 0);
    unsigned long long trc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // registers; written once at the end
    unsigned long long tprev = tr ? (unsigned long long)clock64() : 0;
    auto stamp = [&](int k) {
        if (tr) {
            unsigned long long t = (unsigned long long)clock64();
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q == k) trc[q] += t - tprev;
            tprev = t;
        }
    };
    const int64_t nblk = (p.L + W - 1) / W;
    auto stage = [&](int64_t blk) { return Abuf + (size_t)(blk % kScdStages) * W * R; };
    const bool ctrl = warp == kCtrlWarp, prod = warp == kProdWarp;
    const int cw = warp < kCtrlWarp ? warp : (warp > kCtrlWarp && warp < kProdWarp ? warp - 1 : -1);

    // per-compute-warp tile lists, built once: item = kind | jt << 2 | k0 << 6 | kw << 11 | part << 15
    __shared__ int witems[kCompute][24];
    __shared__ int wcount[kCompute];
    if (tid == 0) {
        for (int w = 0; w < kCompute; ++w) wcount[w] = 0;
        int item = 0;
        for (int cost = 2; cost >= 0; --cost)          // 2: kw 8 tiles, 1: kw 4 tiles, 0: u tiles
            for (int kind = 0; kind < 3; ++kind) {
                if ((kind == 2) != (cost == 0)) continue;
                for (int jt = 0; jt < T; ++jt) {
                    const int kend = kind == 0 ? 4 * jt + 4 : (kind == 1 ? W : 1);
                    for (int k0 = 0; k0 < kend; k0 += 8) {
                        const int kw = kind == 2 ? 1 : (kend - k0 >= 8 ? 8 : 4);
                        if ((kw == 8) != (cost == 2) && kind != 2) continue;
                        const int nparts = kw == 8 ? 2 : 1;  // split the big tiles by rows
                        for (int part = 0; part < nparts; ++part) {
                            const int rnd = item / kCompute, pos = item % kCompute;
                            const int owner = (rnd & 1) ? kCompute - 1 - pos : pos;
                            ++item;
                            if (wcount[owner] < 24)
                                witems[owner][wcount[owner]++] = kind | jt << 2 | k0 << 6 | kw << 11 | part << 15;
                        }
                    }
                }
            }
    }
    __syncthreads();
    const int half = ((rows >> 2) + 1) / 2 * 4;  // row split point (multiple of 4)

    if (prod) {
        // ---------------------------------------------------------------- producer
        int pf_slot = 0;
        unsigned pf_need = 0, seen = 0;
        auto prefetch_slot = [&](int64_t blk) {
            const int64_t t = blk * W + lane;
            if (lane < W && t < p.L) {
                pf_slot = p.order_slot[t];
                pf_need = p.order_batch ? p.order_batch[t] : 0u;
            }
        };
        prefetch_slot(0);
        for (int64_t q = 0; q < nblk; ++q) {
            const int slot = pf_slot;
            const unsigned need = pf_need;
            if (q + 1 < nblk) prefetch_slot(q + 1);
            if (q >= kScdStages)  // block q-3 consumed: its stage is free
                mbar_wait_bounded(&empty[q % kScdStages], (unsigned)((q / kScdStages - 1) & 1), p.err, 4,
                                  kSpinTimeoutNs);
            scd_issue(p, Abuf, full, q, r0, rows, lane, slot, need, seen);
        }
    } else if (ctrl) {
        // ---------------------------------------------------------------- control
        int64_t pf_j = 0;
        double pf_a = 0, pf_inv = 0, pf_y = 0;
        auto prefetch_coords = [&](int64_t blk) {
            const int64_t t = blk * W + lane;
            if (lane < W && t < p.L) {
                pf_j = p.order_j[t];
                pf_a = p.order_a[t];
                pf_inv = p.order_inv[t];
                pf_y = p.order_y[t];
            }
        };
        prefetch_coords(0);
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t base = b * W;
            const int Wb = (int)imin64(W, p.L - base);
            // this block's inputs (prefetched one block ahead), then start the next block's loads
            const int64_t jg = pf_j;
            const double a_in = pf_a, inv_in = pf_inv, y_in = pf_y;
            if (b + 1 < nblk) prefetch_coords(b + 1);
            stamp(0);
#ifdef DUHL_EXP_ALLPOLL
            if (true) {
#else
            if (lane == 0) {
#endif
                // A CTA may ARRIVE(b+1) before another has ARRIVEd(b), but never ARRIVE(b+2)
                // before WAIT(b) completed everywhere: one counter per block parity counts
                // exactly the arrivals of blocks b, b-2, b-4, ...
                const unsigned target = (unsigned)((b / 2 + 1) * (int64_t)p.G);
                const unsigned long long t0 = gtimer();
                while (ld_acquire_u32(&p.bar[b & 1]) < target) {
                    __nanosleep(32);
                    if (gtimer() - t0 > kSpinTimeoutNs) {
                        atomicOr(p.err, 2);
#ifdef DUHL_DEBUG_WAITS
                        printf("WAIT timeout CTA %d b %lld bar %u target %u G %d nblk %lld\n", c, (long long)b,
                               ld_acquire_u32(&p.bar[b & 1]), target, p.G, (long long)nblk);
#endif
                        break;
                    }
                }
#ifndef DUHL_EXP_ALLPOLL
                __threadfence();
#endif
            }
            __syncwarp();
            stamp(2);
            if (c == 0)
                for (int q = lane; q < NRED * kRedGroups; q += 32)
                    p.red[(size_t)((b + 4) % kRedBufs) * bufsz + (size_t)q * kRedStride] = 0.0;
#ifdef DUHL_EXP_CTRLTRACE
            stamp(5);
#endif
            {   // all loads of the reduced block in flight at once (8 entries per lane per batch)
                const double* red_b = p.red + (size_t)(b % kRedBufs) * bufsz;
                const int nq = b > 0 ? NRED : scd_off_C(W);
                for (int q0 = 0; q0 < nq; q0 += 8 * 32) {
                    double v[8][kRedGroups];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        // unconditional loads (index clamped, store predicated) so all of them
                        // are in flight together: one L2 round trip instead of one per entry
                        const int q = min(q0 + u * 32 + lane, nq - 1);
#pragma unroll
                        for (int g = 0; g < kRedGroups; ++g)
                            v[u][g] = ld_cg_f64(&red_b[((size_t)q * kRedGroups + g) * kRedStride]);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int q = q0 + u * 32 + lane;
                        double s = 0.0;
#pragma unroll
                        for (int g = 0; g < kRedGroups; ++g) s += v[u][g];
                        if (q < nq) sG[q] = s;
                    }
                }
            }
            __syncwarp();
            stamp(3);
            const double* dprev = delta + (size_t)((b & 1) ^ 1) * 16;
            // Lane j < Wb owns coordinate j.  Keep the step's pre-activation t_j and
            // fold every correction into it with one DFMA:
            //   Lasso: t = gamma = a - s/||a||^2,  alpha' = soft(t, lambda d/||a||^2)
            //   SVM:   t = y a + (lambda n - y s)/||a||^2,  alpha' = y clip(t, 0, 1)
            // s_j <- s_j + G_jk delta_k  becomes  t_j <- t_j + c_jk delta_k with
            // c_jk = -G_jk/||a_j||^2 (Lasso) or -y_j G_jk/||a_j||^2 (SVM).
            double a = 0, t = 0, tau = 0, cy_ = 0, scale = 0, afin = 0;
            bool zero = true;
            if (lane < Wb) {
                a = a_in;
                double inv = inv_in;
                zero = inv < 0.0;
                if (zero) inv = 0.0;
                const double yy = y_in;
                double sj = sG[lane];
                if (b > 0)  // u was taken at the start of block b-1: add its effect
                    for (int k2 = 0; k2 < W; ++k2) sj = fma(sG[scd_off_C(W) + lane * W + k2], dprev[k2], sj);
                if (MODEL == kLasso) {
                    t = a - sj * inv;
                    tau = lam_dn * inv;
                    scale = -inv;
                } else if (MODEL == kRidge) {  // ridge / elastic net: inv = 1/(||a||^2 + lambda eta d)
                    t = a - (sj + p.lam_q * a) * inv;
                    tau = p.lam_l1 * inv;
                    scale = -inv;
                } else {
                    t = fma(lam_dn - yy * sj, inv, yy * a);
                    cy_ = yy;
                    scale = -yy * inv;
                }
            }
#ifdef DUHL_EXP_CTRLTRACE
            __syncwarp();
            stamp(6);
#endif
            double* dcur = delta + (size_t)(b & 1) * 16;
            // Stage every coordinate's t_j and scaled Gram row in shared memory, then let
            // every lane run all Wb steps redundantly: no per-step cross-lane traffic.
            if (lane < 16) {
                sT[lane] = t;
                sP[lane] = MODEL != kSvm ? tau : cy_;
                sZ[lane] = zero ? 1 : 0;
                sA[lane] = a;
                sS[lane] = scale;
            }
            __syncwarp();
            // scaled Gram rows, written entry-by-lane (consecutive doubles: no bank conflicts)
#pragma unroll
            for (int e0 = 0; e0 < 256; e0 += 32) {
                const int e = e0 + lane, q = e >> 4, j = e & 15;
                sC[e] = (j < q && q < Wb) ? sS[q] * sG[scd_off_G(W) + q * (q - 1) / 2 + j] : 0.0;
            }
            __syncwarp();
            double tq[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) tq[q] = sT[q];
#ifdef DUHL_EXP_CTRLTRACE
            stamp(7);
#endif
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j >= Wb) break;
                const double aj = sA[j], pj = sP[j];
                double an;
                if (MODEL != kSvm) {
                    const double mag = fabs(tq[j]) - pj;
                    an = mag > 0.0 ? copysign(mag, tq[j]) : 0.0;
                    if (sZ[j]) an = 0.0;
                } else {
                    const double u = tq[j] < 0.0 ? 0.0 : (tq[j] > 1.0 ? 1.0 : tq[j]);
                    an = sZ[j] ? pj : pj * u;
                }
                const double dl = an - aj;
                if (lane == j) afin = an;
                if (lane == 0) dcur[j] = dl;
#pragma unroll
                for (int q = j + 1; q < 16; ++q) tq[q] = fma(sC[q * 16 + j], dl, tq[q]);
            }
            if (lane >= Wb && lane < 16) dcur[lane] = 0.0;
            __syncwarp();
            if (lane == 0) mbar_arrive(&dfull[b & 1]);  // publish delta^{(b)} to the compute warps
#ifdef DUHL_DEBUG_WAITS
            if (lane == 0 && c == 0 && b < 4) printf("ctrl CTA0 published delta %lld\n", (long long)b);
#endif
            if (lane < Wb && c == 0) p.alpha[jg] = afin;
            stamp(4);
        }
    } else {
        // ---------------------------------------------------------------- compute
        const int ctid = cw * 32 + lane;
        const bool tr0 = trc_cta && tid == 0;
        unsigned long long tc = tr0 ? (unsigned long long)clock64() : 0;
        auto cstamp = [&](int k) {
#ifdef DUHL_EXP_CTRLTRACE
            return;
#endif
            if (tr0) {
                unsigned long long t = (unsigned long long)clock64();
#pragma unroll
                for (int q = 5; q < 8; ++q)
                    if (q == k) trc[q] += t - tc;
                tc = t;
            }
        };
        auto tiles = [&](int64_t blk, bool with_c) {  // partials of block blk -> red[blk % 6]
            const float* A1 = stage(blk);
            const float* A0 = with_c ? stage(blk - 1) : nullptr;
            const RedOut out{p.red + (size_t)(blk % kRedBufs) * bufsz, grp};
            const int cnt = wcount[cw];
            for (int it = 0; it < cnt; ++it) {
                const int code = witems[cw][it];
                const int kind = code & 3, jt = (code >> 2) & 15, k0 = (code >> 6) & 31, kw = (code >> 11) & 15,
                          part = (code >> 15) & 1;
                if (kind == 1 && !with_c) continue;
                const int lo = kw == 8 ? (part == 0 ? 0 : half) : 0;
                const int hi = kw == 8 ? (part == 0 ? half : rows) : rows;
                const float* Aj = A1 + (size_t)(4 * jt) * R;
                if (kind == 0) {
                    if (kw == 8) tile4<EXACT, 8, true>(Aj, A1 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
                    else tile4<EXACT, 4, true>(Aj, A1 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
                } else if (kind == 1) {
                    if (kw == 8) tile4<EXACT, 8, false>(Aj, A0 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
                    else tile4<EXACT, 4, false>(Aj, A0 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
                } else {
                    utile(Aj, vs, R, lo, hi, lane, 4 * jt, out);
                }
            }
            // ARRIVE(blk): the compute warps' REDs are ordered before one cumulative fence
            named_sync(kBarCompute, kCompute * 32);
            if (ctid == 0) {
                __threadfence();
                atomicAdd(&p.bar[blk & 1], 1u);
#ifdef DUHL_DEBUG_WAITS
                if (blk < 2) printf("arrive CTA %d blk %lld\n", c, (long long)blk);
#endif
            }
        };
        auto vupdate = [&](int64_t b) {  // v slice += A_b delta_b (rows split over the compute warps)
            const int Wb = (int)imin64(W, p.L - b * W);
            const float* A = stage(b);
            const double* dcur = delta + (size_t)(b & 1) * 16;
            double2* v2 = reinterpret_cast<double2*>(vs);
            for (int r4 = ctid; r4 < (rows >> 2); r4 += kCompute * 32) {
                double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
                for (int j = 0; j < Wb; ++j) {
                    const float4 x = reinterpret_cast<const float4*>(A + (size_t)j * R)[r4];
                    const double dj = dcur[j];
                    v01.x = fma(dj, (double)x.x, v01.x);
                    v01.y = fma(dj, (double)x.y, v01.y);
                    v23.x = fma(dj, (double)x.z, v23.x);
                    v23.y = fma(dj, (double)x.w, v23.y);
                }
                v2[2 * r4] = v01;
                v2[2 * r4 + 1] = v23;
            }
        };
        auto wait_data = [&](int64_t blk) {
            mbar_wait_bounded(&full[blk % kScdStages], (unsigned)((blk / kScdStages) & 1), p.err, 8,
                              kSpinTimeoutNs);
        };
        auto wait_delta = [&](int64_t blk) {
            mbar_wait_bounded(&dfull[blk & 1], (unsigned)((blk >> 1) & 1), p.err, 16, kSpinTimeoutNs);
        };
        if (nblk > 0) {
            wait_data(0);
            tiles(0, false);
        }
        for (int64_t b = 0; b < nblk; ++b) {
            named_sync(kBarCompute, kCompute * 32);  // every warp is done reading v for block b's u
            if (b >= 1) {
                cstamp(7);
#ifdef DUHL_DEBUG_WAITS
                if (lane == 0 && c == 0 && b < 4) printf("cmp CTA0 warp %d waits delta %lld\n", warp, (long long)(b - 1));
#endif
                wait_delta(b - 1);
#ifdef DUHL_DEBUG_WAITS
                if (lane == 0 && c == 0 && b < 4) printf("cmp CTA0 warp %d got delta %lld\n", warp, (long long)(b - 1));
#endif
                cstamp(5);
                vupdate(b - 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[(b - 1) % kScdStages]);  // block b-1's stage is free
                named_sync(kBarCompute, kCompute * 32);  // v_b complete before the u tiles read it
                cstamp(6);
            }
            if (b + 1 < nblk) {
                wait_data(b + 1);
#ifdef DUHL_DEBUG_WAITS
                if (lane == 0 && c == 0 && b < 4) printf("cmp CTA0 warp %d got data %lld\n", warp, (long long)(b + 1));
#endif
                tiles(b + 1, true);
            }
        }
        if (nblk > 0) {
            cstamp(7);
            wait_delta(nblk - 1);
            cstamp(5);
            vupdate(nblk - 1);
            cstamp(6);
        }
    }
    __syncthreads();
    for (int r = tid; r < rows; r += kScdThreads) p.vt[r0 + r] = vs[r];
    if (tr)
        for (int q = 0; q < 8; ++q)
            if (trc[q]) atomicAdd(&p.trace[(c == 0 ? 0 : 8) + q], trc[q]);
}

cudaError_t launch_scd_gram(const ScdParams& p, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    size_t smem = scd_smem_bytes(p.W, p.R, kScdStages);
    const void* fn = p.model == kLasso
                         ? (p.exact ? (const void*)k_scd_gram<true, kLasso> : (const void*)k_scd_gram<false, kLasso>)
                     : (p.model == kRidge || p.model == kElastic)
                         ? (p.exact ? (const void*)k_scd_gram<true, kRidge> : (const void*)k_scd_gram<false, kRidge>)
                         : (p.exact ? (const void*)k_scd_gram<true, kSvm> : (const void*)k_scd_gram<false, kSvm>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ScdParams q = p;
    void* args[] = {&q};
    e = cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(kScdThreads), args, smem, st);
    ++*launches;
    return e;
}

#include "scd_pipe.cuh"
#include "scd_ser.cuh"

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

// out[0] += sum_i x_i
__global__ void k_sum(const double* x, int64_t n, double* out) {
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += x[i];
    s = warp_sum(s);
    __shared__ double sh[8];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += sh[w];
        atomicAdd(out, a);
    }
}
cudaError_t launch_sum(const double* x, int64_t n, double* out, cudaStream_t st, int64_t* launches) {
    k_sum<<<(unsigned)imin64(cdiv(n, 256), 296), 256, 0, st>>>(x, n, out);
    ++*launches;
    return cudaGetLastError();
}

// ---- CoCoA-style aggregation helpers ------------------------------
// out[q] = x[idx[q]]
__global__ void k_gather_f64(const double* x, const int64_t* idx, int64_t k, double* out) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < k) out[q] = x[idx[q]];
}
// dv = v - v0 ; sums[0] += v0^T dv, sums[1] += dv^T dv
__global__ void k_delta_v(const double* v, const double* v0, int64_t d4, double* dv, double* sums) {
    double s0 = 0, s1 = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d4; r += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[r] - v0[r];
        dv[r] = x;
        s0 = fma(v0[r], x, s0);
        s1 = fma(x, x, s1);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if ((threadIdx.x & 31) == 0) { atomicAdd(&sums[0], s0); atomicAdd(&sums[1], s1); }
}
// SVM: sums[0] += sum_q y_j (alpha_j - aold_q),  j = P[q]
__global__ void k_ydalpha(const double* alpha, const double* y, const int64_t* P, const double* aold, int64_t k,
                          double* sums) {
    double s = 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x)
        s += y[P[q]] * (alpha[P[q]] - aold[q]);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) atomicAdd(&sums[0], s);
}
__global__ void k_ridge_sums(const double* alpha, const int64_t* P, const double* aold, int64_t k, double* sums) {
    double s0 = 0, s1 = 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x) {
        const double da = alpha[P[q]] - aold[q];
        s0 += aold[q] * da;
        s1 += da * da;
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[0], s0);
        atomicAdd(&sums[1], s1);
    }
}
cudaError_t launch_ridge_sums(const double* alpha, const int64_t* P, const double* aold, int64_t k, double* sums,
                              cudaStream_t st, int64_t* launches) {
    if (k <= 0) return cudaSuccess;
    k_ridge_sums<<<(unsigned)imin64(cdiv(k, 256), 148), 256, 0, st>>>(alpha, P, aold, k, sums);
    ++*launches;
    return cudaGetLastError();
}
// Lasso: out[g] += sum_q da_q sgn+(aold_q + gam[g] da_q), da_q = alpha_j - aold_q  (g < ng,
// gam ascending), sgn+(x) = sign(x), and sign(da) at x = 0 (the right derivative).  Along the
// grid x_q(g) = fma(g, da, aold) is monotone, so coordinate q contributes -|da_q| below its
// switch index j*_q (the first grid point where x_q has reached da's side of 0, by the same
// fma predicate the direct evaluation uses) and +|da_q| from j*_q on:
//   out[g] = sum_q |da_q| - 2 sum_{q: j*_q > g} |da_q|.
// One binary search and one shared-memory atomic per coordinate instead of ng.
__global__ void k_lasso_dgrid(const double* alpha, const int64_t* P, const double* aold, int64_t k,
                              const double* gam, int ng, double* out) {
    __shared__ double sg[64], cnt[65], sbase[8];
    for (int g = threadIdx.x; g < ng; g += blockDim.x) sg[g] = gam[g];
    for (int g = threadIdx.x; g <= ng; g += blockDim.x) cnt[g] = 0.0;
    __syncthreads();
    double base = 0.0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x) {
        const double a0 = aold[q], da = alpha[P[q]] - a0;
        if (da == 0.0) continue;
        const double w = fabs(da);
        base += w;
        int lo = 0, hi = ng;  // first j in [0, ng] with the predicate true (ng: never)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const double x = fma(sg[mid], da, a0);
            const bool reached = da > 0.0 ? x >= 0.0 : x <= 0.0;
            if (reached) hi = mid;
            else lo = mid + 1;
        }
        if (lo > 0) atomicAdd(&cnt[lo], w);  // j* = lo: grid points 0..lo-1 lie below the switch
    }
    base = warp_sum(base);
    if ((threadIdx.x & 31) == 0) sbase[threadIdx.x >> 5] = base;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += sbase[w];
        double suffix = 0.0;  // sum of cnt[j'] for j' > g, walking g downwards
        for (int g = ng - 1; g >= 0; --g) {
            suffix += cnt[g + 1];
            atomicAdd(&out[g], b - 2.0 * suffix);
        }
    }
}
// v = v0 + gamma dv ; alpha_P = aold + gamma (alpha_P - aold)
__global__ void k_apply_gamma(double* v, const double* v0, const double* dv, int64_t d4, double* alpha,
                              const int64_t* P, const double* aold, int64_t k, double gamma) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d4; r += stride) v[r] = fma(gamma, dv[r], v0[r]);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += stride) {
        const int64_t j = P[q];
        alpha[j] = fma(gamma, alpha[j] - aold[q], aold[q]);
    }
}
cudaError_t launch_gather_f64(const double* x, const int64_t* idx, int64_t k, double* out, cudaStream_t st,
                              int64_t* launches) {
    if (k <= 0) return cudaSuccess;
    k_gather_f64<<<(unsigned)cdiv(k, 256), 256, 0, st>>>(x, idx, k, out);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_delta_v(const double* v, const double* v0, int64_t d4, double* dv, double* sums,
                           cudaStream_t st, int64_t* launches) {
    k_delta_v<<<(unsigned)imin64(cdiv(d4, 256), 296), 256, 0, st>>>(v, v0, d4, dv, sums);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_ydalpha(const double* alpha, const double* y, const int64_t* P, const double* aold, int64_t k,
                           double* sums, cudaStream_t st, int64_t* launches) {
    k_ydalpha<<<(unsigned)imin64(cdiv(k, 256), 148), 256, 0, st>>>(alpha, y, P, aold, k, sums);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_lasso_dgrid(const double* alpha, const int64_t* P, const double* aold, int64_t k,
                               const double* gam, int ng, double* out, cudaStream_t st, int64_t* launches) {
    k_lasso_dgrid<<<(unsigned)imin64(cdiv(k, 256), 148), 256, 0, st>>>(alpha, P, aold, k, gam, ng, out);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_apply_gamma(double* v, const double* v0, const double* dv, int64_t d4, double* alpha,
                               const int64_t* P, const double* aold, int64_t k, double gamma, cudaStream_t st,
                               int64_t* launches) {
    k_apply_gamma<<<(unsigned)imin64(cdiv(d4 > k ? d4 : k, 256), 296), 256, 0, st>>>(v, v0, dv, d4, alpha, P,
                                                                                     aold, k, gamma);
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


// =====================================================================================
// Sparse (CSC) path, SURVEY 8 C5.  One warp per column; the shared vector is
// gathered by row index (fp64, L2-resident: 8 d bytes), the column streamed once.
// =====================================================================================
__device__ __forceinline__ int ld_stream_i32(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(256) k_csc_norms(CscMat A, int64_t n, double* norms) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        const int64_t k0 = A.col_ptr[i], k1 = A.col_ptr[i + 1];
        double s = 0.0;
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const double x = (double)ld_stream_f32(A.vals + k);
            s = fma(x, x, s);
        }
        s = warp_sum(s);
        if (lane == 0) norms[i] = s;
    }
}

// s_i = sum_k a_ki (wscale vt_k) over the column's nonzeros, then the gap (as k_gap_tile).
__global__ void __launch_bounds__(256) k_csc_gap(GapParams p, CscMat A) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    SumAcc acc;
    int flag = 0;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < p.k; t += nw) {
        const int64_t i = p.cols ? p.cols[t] : t;
        const int64_t k0 = A.col_ptr[i], k1 = A.col_ptr[i + 1];
        double s0 = 0.0, s1 = 0.0;
        int64_t k = k0 + lane;
        for (; k + 32 < k1; k += 64) {  // two independent gathers in flight per lane
            const int r0 = ld_stream_i32(A.rows + k), r1 = ld_stream_i32(A.rows + k + 32);
            const float x0 = ld_stream_f32(A.vals + k), x1 = ld_stream_f32(A.vals + k + 32);
            s0 = fma((double)x0, __ldg(p.vt + r0) * p.wscale, s0);
            s1 = fma((double)x1, __ldg(p.vt + r1) * p.wscale, s1);
        }
        if (k < k1) s0 = fma((double)ld_stream_f32(A.vals + k), __ldg(p.vt + ld_stream_i32(A.rows + k)) * p.wscale, s0);
        const double s = warp_sum(s0 + s1);
        if (lane == 0) gap_finish_one(p, t, i, s, acc, flag);
    }
    block_flush_sums(p, acc, flag);
}

__global__ void __launch_bounds__(256) k_csc_scd(CscScdParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double dd = (double)p.d, nn = (double)p.n;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < p.L; t += nw) {
        const int64_t j = p.order_j[t];
        const int64_t k0 = p.A.col_ptr[j], k1 = p.A.col_ptr[j + 1];
        double s = 0.0;
        for (int64_t k = k0 + lane; k < k1; k += 32)  // v is being updated by other warps: read it at L2
            s = fma((double)p.A.vals[k], __ldcg(p.vt + p.A.rows[k]), s);
        s = warp_sum(s);
        const double a = p.alpha[j];
        const double an = coord_step(p.model, a, s, p.norms[j], p.y ? p.y[j] : 0.0, p.lambda, dd, nn, p.eta);
        const double dl = an - a;
        if (dl != 0.0)
            for (int64_t k = k0 + lane; k < k1; k += 32) atomicAdd(p.vt + p.A.rows[k], dl * (double)p.A.vals[k]);
        if (lane == 0) p.alpha[j] = an;
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_csc_matvec(CscMat A, const double* alpha, int64_t n, double* vt) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        const double a = alpha[i];
        if (a == 0.0) continue;
        for (int64_t k = A.col_ptr[i] + lane; k < A.col_ptr[i + 1]; k += 32)
            atomicAdd(vt + A.rows[k], a * (double)A.vals[k]);
    }
}

static unsigned csc_grid(int64_t work_warps) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t full = (int64_t)nsm * 8;  // 8 CTAs x 8 warps per SM
    const int64_t need = (work_warps + 7) / 8;
    return (unsigned)(need < full ? (need > 0 ? need : 1) : full);
}

cudaError_t launch_csc_norms(const CscMat& A, int64_t n, double* norms, cudaStream_t st, int64_t* launches) {
    if (n <= 0) return cudaSuccess;
    k_csc_norms<<<csc_grid(n), 256, 0, st>>>(A, n, norms);
    ++*launches;
    return cudaGetLastError();
}

// The same pass with the head of the shared vector in shared memory: one 1024-thread CTA per
// SM stages w_r = wscale vt_r for rows r < Rs (fp64, up to DUHL_CSC_SMEM_KB, default 160 KB)
// and gathers those rows from shared memory, the rest through L1 / L2 as above.  A warp's 32
// row indices of one column are ~100 rows apart (uniform rows, 1 % density), so a global
// gather touches ~32 L1 lines -- the L1 tag rate, ~1 line per clock per SM, bounds
// k_csc_gap at ~1 nonzero per clock per SM; a shared-memory gather costs a few bank
// wavefronts instead.  Same products (vt_r wscale rounded once); four partial sums per lane
// (fp64; k_csc_gap keeps two).  Measured (C5s, gap pass GB/s): k_csc_gap 2274; this kernel
// with 64 / 96 / 128 / 160 / 192 KB of rows in shared memory 2443 / 2548 / 2607 / 2624 /
// 2568; two partial sums at 200 KB 1737; eight (predicated tails, next column's extent
// prefetched) 2024-2189 -- register-limited at 1024 threads; the index / value loads of the
// next 128-nonzero window software-pipelined across the warp's column stream 2313 (1024
// threads, spills) / 2235 (768) / 1618 (512), against 2629 for this loop in the same run.
constexpr int kCscSmemThreads = 1024;
__global__ void __launch_bounds__(kCscSmemThreads, 1) k_csc_gap_smem(GapParams p, CscMat A, int Rs) {
    extern __shared__ double sw[];
    for (int r = threadIdx.x; r < Rs; r += kCscSmemThreads) sw[r] = p.vt[r] * p.wscale;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    SumAcc acc;
    int flag = 0;
    auto wget = [&](int r) { return r < Rs ? sw[r] : __ldg(p.vt + r) * p.wscale; };
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < p.k; t += nw) {
        const int64_t i = p.cols ? p.cols[t] : t;
        const int64_t k0 = A.col_ptr[i], k1 = A.col_ptr[i + 1];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t k = k0 + lane;
        for (; k + 96 < k1; k += 128) {  // four independent gathers in flight per lane
            const int r0 = ld_stream_i32(A.rows + k), r1 = ld_stream_i32(A.rows + k + 32);
            const int r2 = ld_stream_i32(A.rows + k + 64), r3 = ld_stream_i32(A.rows + k + 96);
            const float x0 = ld_stream_f32(A.vals + k), x1 = ld_stream_f32(A.vals + k + 32);
            const float x2 = ld_stream_f32(A.vals + k + 64), x3 = ld_stream_f32(A.vals + k + 96);
            s0 = fma((double)x0, wget(r0), s0);
            s1 = fma((double)x1, wget(r1), s1);
            s2 = fma((double)x2, wget(r2), s2);
            s3 = fma((double)x3, wget(r3), s3);
        }
        for (; k < k1; k += 32) s0 = fma((double)ld_stream_f32(A.vals + k), wget(ld_stream_i32(A.rows + k)), s0);
        const double s = warp_sum((s0 + s1) + (s2 + s3));
        if (lane == 0) gap_finish_one(p, t, i, s, acc, flag);
    }
    block_flush_sums<kCscSmemThreads>(p, acc, flag);
}

cudaError_t launch_csc_gap(const GapParams& p, const CscMat& A, int max_ctas, cudaStream_t st, int64_t* launches) {
    if (p.k <= 0) return cudaSuccess;
    static const int smem_kb = [] {
        const char* e = std::getenv("DUHL_CSC_SMEM_KB");  // developer A/B; 0 = k_csc_gap
        return e ? std::atoi(e) : 160;
    }();
    if (smem_kb > 0 && p.k >= 4096) {
        const int Rs = (int)std::min<int64_t>(p.d, (int64_t)smem_kb * 1024 / 8);
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int g = nsm;
        if (max_ctas > 0 && g > max_ctas) g = max_ctas;
        const size_t smem = (size_t)Rs * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_csc_gap_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_csc_gap_smem<<<g, kCscSmemThreads, smem, st>>>(p, A, Rs);
        ++*launches;
        return cudaGetLastError();
    }
    unsigned g = csc_grid(p.k);
    if (max_ctas > 0 && g > (unsigned)max_ctas) g = (unsigned)max_ctas;
    k_csc_gap<<<g, 256, 0, st>>>(p, A);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_csc_scd(const CscScdParams& p, int warps, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    if (warps == 1) k_csc_scd<<<1, 32, 0, st>>>(p);
    else k_csc_scd<<<csc_grid(warps > 0 ? warps : p.L), 256, 0, st>>>(p);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_csc_matvec(const CscMat& A, const double* alpha, int64_t n, double* vt, cudaStream_t st,
                              int64_t* launches) {
    if (n <= 0) return cudaSuccess;
    k_csc_matvec<<<csc_grid(n), 256, 0, st>>>(A, alpha, n, vt);
    ++*launches;
    return cudaGetLastError();
}

// Resident working set (no slot pool): slot of P[q] = P[q], no staging; count the
// coordinates not selected last time (stamp[j] == sel - 1) and, for CSC, the
// algorithmic bytes of a pass over P; stamp the new members with sel.
__global__ void k_resident_select(const int64_t* P, int64_t m, int* stamp, int sel, int* P_slot,
                                  unsigned* P_batch, const int64_t* col_ptr, unsigned long long* out) {
    unsigned long long sw = 0, by = 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = P[q];
        P_slot[q] = (int)j;
        P_batch[q] = 0u;
        sw += stamp[j] != sel - 1;
        stamp[j] = sel;
        if (col_ptr) by += (unsigned long long)(col_ptr[j + 1] - col_ptr[j]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        sw += __shfl_xor_sync(~0u, sw, o);
        by += __shfl_xor_sync(~0u, by, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sw) atomicAdd(&out[0], sw);
        if (by) atomicAdd(&out[1], by);
    }
}

cudaError_t launch_resident_select(const int64_t* P, int64_t m, int* stamp, int sel, int* P_slot,
                                   unsigned* P_batch, const int64_t* col_ptr, unsigned long long* out,
                                   cudaStream_t st, int64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess || m <= 0) return e;
    k_resident_select<<<(unsigned)imin64(cdiv(m, 256), 1184), 256, 0, st>>>(P, m, stamp, sel, P_slot, P_batch,
                                                                           col_ptr, out);
    ++*launches;
    return cudaGetLastError();
}

// Load every kernel of the library now.  Under lazy module loading (the CUDA 12
// default) the first launch of a kernel loads it, and that load can wait for the
// device to go idle -- fatal while the SCD kernel waits on staging copies the
// host has yet to enqueue (the refresh kernel is launched in between).
cudaError_t preload_kernels() {
    const void* fns[] = {
        (const void*)k_gap_tile<false>, (const void*)k_gap_tile<true>, (const void*)k_gap_finalize, (const void*)k_col_norms,
        (const void*)k_topm,        (const void*)k_perm_order,   (const void*)k_order_info,
        (const void*)k_scd_gram<true, kLasso>, (const void*)k_scd_gram<false, kLasso>,
        (const void*)k_scd_gram<true, kSvm>,   (const void*)k_scd_gram<false, kSvm>,
        (const void*)k_scd_pipe<true, kLasso>, (const void*)k_scd_pipe<false, kLasso>,
        (const void*)k_scd_pipe<true, kSvm>,   (const void*)k_scd_pipe<false, kSvm>,
        (const void*)k_scd_gram<true, kRidge>, (const void*)k_scd_gram<false, kRidge>,
        (const void*)k_scd_pipe<true, kRidge>, (const void*)k_scd_pipe<false, kRidge>, (const void*)k_ridge_sums,
        (const void*)k_scd_ser<true, kLasso>, (const void*)k_scd_ser<false, kLasso>,
        (const void*)k_scd_ser<true, kSvm>,   (const void*)k_scd_ser<false, kSvm>,
        (const void*)k_scd_ser<true, kRidge>, (const void*)k_scd_ser<false, kRidge>,
        (const void*)k_matvec,      (const void*)k_set_slots,    (const void*)k_sum,
        (const void*)k_gather_f64,  (const void*)k_delta_v,      (const void*)k_ydalpha,
        (const void*)k_lasso_dgrid, (const void*)k_apply_gamma,  (const void*)k_vec_sums,
        (const void*)k_csc_norms,   (const void*)k_csc_gap,      (const void*)k_csc_gap_smem,      (const void*)k_csc_scd,
        (const void*)k_csc_matvec,  (const void*)k_topm_hist,    (const void*)k_topm_pick,
        (const void*)k_topm_count,  (const void*)k_topm_offsets, (const void*)k_topm_write,
        (const void*)k_resident_select, (const void*)k_stage_gather};
    for (const void* f : fns) {
        cudaFuncAttributes a;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace duhl
