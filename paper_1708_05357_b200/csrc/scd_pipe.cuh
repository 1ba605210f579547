// scd_pipe.cuh -- pipelined exact SCD epoch (App. D closed forms in the exact
// sequential order).  Included by kernels.cu (uses its
// tile4 / utile helpers, the RED layout constants and the bounded waits).
//
// Why a second kernel: in k_scd_gram every CTA runs the W sequential steps in a
// control warp that shares the SM's shared-memory / shuffle pipe with six
// compute warps saturating it, and a block's Gram tiles wait for delta_{b-1}.
// Measured (DUHL_SCD_TRACE, C4 / C3 shapes): ~7.8 us per block, of which the
// control chain (barrier wait + read-back + steps) is ~7.6 us and the tiles ~6 us,
// against 1.5 us (C4) / 0.3 us (C3) of HBM time.  This kernel
//   * gives the sequential part its own CTA (the control CTA, blockIdx.x == G):
//     it waits for block b's reduction, reads it back with all of its threads,
//     runs the W steps on one warp (lane j owns coordinate j; delta_j is
//     broadcast by one shuffle per step) and publishes delta_b to global memory
//     with a release flag;
//   * lets the G compute CTAs build block b+1's delta-independent partials
//     (G_{b+1} and the cross Gram C_{b+1,b}) as soon as the TMA engine has
//     landed the columns, and only then wait for delta_{b-1} to apply
//     v += A_{b-1} delta_{b-1} and take u_{b+1} = A_{b+1}^T v_b;
//   * allows W <= 32 coordinates per block where shared memory holds 3 stages.
// Per block the control CTA computes, for coordinate j of block b (visiting order),
//   s_j = u_j + sum_k C_jk delta^{(b-1)}_k + sum_{k<j} G_jk delta^{(b)}_k  (== a_j^T v at its visit)
// exactly as k_scd_gram does; the result is sequential SCD up to summation order.
//
// Synchronisation (all global, K = kPipeRot rotating buffers):
//   red[b % K]   fp64 REDs of block b's partials by every compute CTA, then
//                cnt[b % K] += 1 per CTA (after a gpu-scope fence);
//   control:     waits cnt[b % K] == G (acquire), reads red[b % K] into shared
//                memory, zeroes red[b % K] and cnt[b % K], runs the steps, writes
//                dbuf[b % K] and releases flg[b % K] = b + 1;
//   compute:     before applying delta_b, waits flg[b % K] >= b + 1 (acquire).
// Reuse of red/cnt[b % K] by block b + K: its first RED is issued (compute
// iteration b + K - 1) after that CTA acquired delta_{b+K-3} >= delta_b, which the
// control CTA released after zeroing -- safe for K >= 3.  dbuf[b % K] is
// rewritten for block b + K only after every CTA arrived for block b + K, i.e.
// after each consumed delta_b (iteration b + 1 <= b + K - 1) -- safe for K >= 2.
#pragma once

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

static_assert(kRedGroups == 1, "the pipelined kernel assumes one reduction group");
constexpr int kPipeWMax = 32;
constexpr int kPipeRot = 6;
constexpr int kPipeThreads = 256;
constexpr int kPipeCompute = 7;   // compute warps 0..6 of a compute CTA
constexpr int kPipeProd = 7;      // producer warp (TMA)
constexpr int kGcWarps = 4;       // Gram group: warps 0..3 (FFMA2); v group: warps 4..6 (fp64)
constexpr int kGcWarpsMax = kGcWarps;
// (3 Gram warps: C4 W = 12 6.97 vs 7.59 ms; 4: C3 W = 32 12.0 vs 16.2 ms -- C3 is the shape that
// runs this kernel by default)
constexpr int kBarGc = 1, kBarV = 2;              // named barriers of the two groups

// Reduction entries of one block (expanded layout, see tile4<..., XL>):
//   u_j [0, W),  G_jk (k < j) at W + k W + j,  C_jk at W + W^2 + k W + j.
__host__ __device__ __forceinline__ int pipe_ne(int W) { return W + 2 * W * W; }
size_t pipe_red_doubles(int W) {
    return (size_t)kPipeRot * pipe_ne(W) * kRedStride + (size_t)kPipeRot * kPipeWMax;  // + delta buffers
}
// Column stride of a stage in shared memory: R rounded so that R/4 is odd -- the
// 16-byte chunks of 8 consecutive columns at one row then fall in 8 distinct bank groups.
__host__ __device__ __forceinline__ int pipe_stride(int R) { return ((R >> 2) & 1) ? R : R + 4; }
size_t pipe_smem_bytes(int W, int R, int NS) {
    const size_t compute = 128 + align_up_dev((size_t)NS * W * pipe_stride(R) * sizeof(float)) +
                           align_up_dev((size_t)R * sizeof(double)) +
                           align_up_dev((size_t)kGcWarpsMax * 2 * W * W * sizeof(float)) +
                           align_up_dev((size_t)kPipeCompute * kPipeWMax * sizeof(double)) +
                           (R <= 512 ? align_up_dev((size_t)3 * R * sizeof(double)) : 0);
    const size_t control = 128 + align_up_dev((size_t)pipe_ne(W) * sizeof(double));
    return compute > control ? compute : control;
}

// One warp's share of a block's Gram partials: the W x 2W block M = A1^T [A1 | A0]
// (M_jk = G_jk for k < W, C_j,k-W for k >= W; global entry W + k W + j) over rows
// [4 r4lo, 4 r4hi).  Lane (jg, kg) = (lane & 3, lane >> 2) owns rows j = jg + 4a and
// columns k = kg + 8b (a, b < T = W/4): one 16-byte load per owned column and 4-row
// step feeds 4 T^2 FMAs, and the 4 (8) distinct columns a load instruction touches are
// consecutive, i.e. conflict-free with the padded stride.  Fast mode: fp32 FMA (FFMA2
// over row pairs), the partial of every lane-entry written to `part` (slot (a T + b) 32
// + lane) for the cross-warp sum; exact mode: fp64 products, REDs straight from here.
template <bool EXACT, int T, int B0, int NBK>  // columns k = kg + 8 b, b in [B0, B0 + NBK)
__device__ __forceinline__ void gc_warp_part(const float* __restrict__ A1, const float* __restrict__ A0, int Rs,
                                             int W, int r4lo, int r4hi, int lane, float* __restrict__ part,
                                             const RedOut& out) {
    const int jg = lane & 3, kg = lane >> 2;
    // (a, b) pairs whose every lane-entry is strictly upper G (k >= 8b > 4a + 3 >= j, k < W): skipped
    auto upper = [](int a, int b) { return 8 * b + 7 < 4 * T && a < 2 * b; };
    // 32-bit shared-window addresses
    uint32_t xa[T], ya[NBK];
#pragma unroll
    for (int a = 0; a < T; ++a) xa[a] = smem_addr(A1 + (size_t)(jg + 4 * a) * Rs);
#pragma unroll
    for (int b = 0; b < NBK; ++b) {
        const int k = kg + 8 * (B0 + b);
        ya[b] = smem_addr(k < W ? A1 + (size_t)k * Rs : A0 + (size_t)(k - W) * Rs);
    }
    if (EXACT) {
        double acc[T][NBK];
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) acc[a][b] = 0.0;
#pragma unroll 2
        for (int r4 = r4lo; r4 < r4hi; ++r4) {
            float4 x[T];
#pragma unroll
            for (int a = 0; a < T; ++a) x[a] = lds_f4(xa[a] + 16u * r4);
#pragma unroll
            for (int b = 0; b < NBK; ++b) {
                const float4 y = lds_f4(ya[b] + 16u * r4);
#pragma unroll
                for (int a = 0; a < T; ++a) {
                    if (upper(a, B0 + b)) continue;
                    double t = acc[a][b];
                    t = fma((double)x[a].x, (double)y.x, t);
                    t = fma((double)x[a].y, (double)y.y, t);
                    t = fma((double)x[a].z, (double)y.z, t);
                    t = fma((double)x[a].w, (double)y.w, t);
                    acc[a][b] = t;
                }
            }
        }
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) {
                const int j = jg + 4 * a, k = kg + 8 * (B0 + b);
                if (k >= W || k < j) out.add(W + k * W + j, acc[a][b]);
            }
    } else if (T + NBK <= 8) {
        // small tiles (W <= 16): loads of row group r4 + 1 in flight while r4's FMAs issue
        float2 acc[T][NBK];
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) acc[a][b] = make_float2(0.f, 0.f);
        float4 xn[T], yn[NBK];
        const int r4c = r4lo < r4hi ? r4lo : 0;
#pragma unroll
        for (int a = 0; a < T; ++a) xn[a] = lds_f4(xa[a] + 16u * r4c);
#pragma unroll
        for (int b = 0; b < NBK; ++b) yn[b] = lds_f4(ya[b] + 16u * r4c);
        for (int r4 = r4lo; r4 < r4hi; ++r4) {
            float4 x[T], y[NBK];
#pragma unroll
            for (int a = 0; a < T; ++a) x[a] = xn[a];
#pragma unroll
            for (int b = 0; b < NBK; ++b) y[b] = yn[b];
            const uint32_t nx = 16u * (uint32_t)(r4 + 1 < r4hi ? r4 + 1 : r4);
#pragma unroll
            for (int a = 0; a < T; ++a) xn[a] = lds_f4(xa[a] + nx);
#pragma unroll
            for (int b = 0; b < NBK; ++b) yn[b] = lds_f4(ya[b] + nx);
#pragma unroll
            for (int b = 0; b < NBK; ++b)
#pragma unroll
                for (int a = 0; a < T; ++a) {
                    if (upper(a, B0 + b)) continue;
                    ffma2(acc[a][b], x[a].x, x[a].y, y[b].x, y[b].y);
                    ffma2(acc[a][b], x[a].z, x[a].w, y[b].z, y[b].w);
                }
        }
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) part[(a * T + B0 + b) * 32 + lane] = acc[a][b].x + acc[a][b].y;
    } else {
        float2 acc[T][NBK];
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) acc[a][b] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int r4 = r4lo; r4 < r4hi; ++r4) {
            float4 x[T];
#pragma unroll
            for (int a = 0; a < T; ++a) x[a] = lds_f4(xa[a] + 16u * r4);
#pragma unroll
            for (int b = 0; b < NBK; ++b) {
                const float4 y = lds_f4(ya[b] + 16u * r4);
#pragma unroll
                for (int a = 0; a < T; ++a) {
                    if (upper(a, B0 + b)) continue;
                    ffma2(acc[a][b], x[a].x, x[a].y, y.x, y.y);
                    ffma2(acc[a][b], x[a].z, x[a].w, y.z, y.w);
                }
            }
        }
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < NBK; ++b) part[(a * T + B0 + b) * 32 + lane] = acc[a][b].x + acc[a][b].y;
    }
}
template <bool EXACT, int T>
__device__ __forceinline__ void gc_warp(const float* A1, const float* A0, int Rs, int W, int r4lo, int r4hi,
                                        int lane, float* part, const RedOut& out) {
    if (T <= 4) {
        gc_warp_part<EXACT, T, 0, T>(A1, A0, Rs, W, r4lo, r4hi, lane, part, out);
    } else {
        gc_warp_part<EXACT, T, 0, 4>(A1, A0, Rs, W, r4lo, r4hi, lane, part, out);
        gc_warp_part<EXACT, T, 4, (T > 4 ? T - 4 : 1)>(A1, A0, Rs, W, r4lo, r4hi, lane, part, out);
    }
}

// Tensor-core form of gc_warp in fast mode (p.gram_tc; default at W = 32, the case described
// here -- gc_warp_tc<T> below generalises it to W = 4 T): the warp's 32 x 64 block
// M = A1^T [A1 | A0] over its rows [4 r4lo, 4 r4hi) as 2 x 8 tiles of mma.sync m16n8k8 TF32
// (M index j = column of A1, N index k = column of [A1 | A0], K index = row).  Each fp32
// operand x is split x = hi + lo with hi = tf32(x), lo = tf32(x - hi), and every tile takes
// hi*lo + lo*hi + hi*hi (3xTF32: the product error of plain TF32 would be ~1e-3, the split
// keeps it near fp32's), accumulated in fp32 like the FFMA2 path.  Fragments are single
// 32-bit shared loads at (column g, row t) -- lane = 4 g + t, the column stride Rs = 4 x odd,
// so the 32 lanes of a load hit 32 distinct banks.  The two all-upper tiles of G (j < 16,
// 16 <= k < 32) are skipped; results go to the same `part` slots as gc_warp_part's
// (slot ((j/4) 8 + k/8) 32 + (j%4) + 4 (k%8)) for gc_sum<8>.
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    const float r = x - __uint_as_float(hi);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// General W = 4 T (T <= 8): MT = ceil(W / 16) row tiles (rows j >= W load zeros), NT = T column
// tiles of 8 over [A1 | A0] (lane g's column k = 8 nt + g is in A1 for k < W, else A0 at k - W,
// so a tile may straddle the two blocks when W % 8 = 4).  A tile is skipped when every entry
// of it is an upper-G entry (16 mt + 15 < 8 nt <= k < W).
template <int T>
__device__ __forceinline__ void gc_warp_tc(const float* __restrict__ A1, const float* __restrict__ A0, int Rs,
                                           int r4lo, int r4hi, int lane, float* __restrict__ part) {
    constexpr int W = 4 * T, MT = (W + 15) / 16, NT = T;
    const int g = lane >> 2, t = lane & 3;
    auto skip = [](int mt, int nt) { return 8 * nt + 7 < W && 16 * mt + 15 < 8 * nt; };
    float acc[MT][NT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.f;
    uint32_t aa[MT][2];   // lane's A rows j = 16 mt + g (+ 8); valid flags
    bool av[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 16 * mt + g + 8 * h;
            av[mt][h] = j < W;
            aa[mt][h] = smem_addr(A1 + (size_t)(j < W ? j : 0) * Rs + t);
        }
    uint32_t ba[NT];      // lane's B column k = 8 nt + g of [A1 | A0]
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int k = 8 * nt + g;
        ba[nt] = smem_addr((k < W ? A1 + (size_t)k * Rs : A0 + (size_t)(k - W) * Rs) + t);
    }
    const int r_lo = 4 * r4lo, r_hi = 4 * r4hi;
    for (int r = r_lo; r < r_hi; r += 8) {
        const bool full = r + 8 <= r_hi;   // else rows r .. r + 3 only (4-row tail)
        const uint32_t ro = 4u * (uint32_t)r;
        uint32_t ah[MT][4], al[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const float x0 = av[mt][0] ? lds_f32(aa[mt][0] + ro) : 0.f;
            const float x1 = av[mt][1] ? lds_f32(aa[mt][1] + ro) : 0.f;
            const float x2 = (av[mt][0] && full) ? lds_f32(aa[mt][0] + ro + 16u) : 0.f;
            const float x3 = (av[mt][1] && full) ? lds_f32(aa[mt][1] + ro + 16u) : 0.f;
            tf32_split(x0, ah[mt][0], al[mt][0]);
            tf32_split(x1, ah[mt][1], al[mt][1]);
            tf32_split(x2, ah[mt][2], al[mt][2]);
            tf32_split(x3, ah[mt][3], al[mt][3]);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float y0 = lds_f32(ba[nt] + ro), y1 = full ? lds_f32(ba[nt] + ro + 16u) : 0.f;
            uint32_t bh0, bl0, bh1, bl1;
            tf32_split(y0, bh0, bl0);
            tf32_split(y1, bh1, bl1);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                if (skip(mt, nt)) continue;
                mma_tf32(acc[mt][nt], al[mt], bh0, bh1);
                mma_tf32(acc[mt][nt], ah[mt], bl0, bl1);
                mma_tf32(acc[mt][nt], ah[mt], bh0, bh1);
            }
        }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (skip(mt, nt)) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 16 * mt + g + 8 * (q >> 1), k = 8 * nt + 2 * t + (q & 1);
                if (j < W) part[(((j >> 2) * T + (k >> 3)) << 5) + (j & 3) + 4 * (k & 7)] = acc[mt][nt][q];
            }
        }
}

// Cross-warp sum of the fast-mode partials (fp32 within the CTA, fp64 REDs across CTAs).
template <int T>
__device__ __forceinline__ void gc_sum(const float* __restrict__ part, int W, int tid, int nwarps,
                                       const RedOut& out) {
    constexpr int nslot = 32 * T * T;
    for (int sl = tid; sl < nslot; sl += nwarps * 32) {
        const int ln = sl & 31, e = sl >> 5, a = e / T, bb = e - a * T;
        const int j = (ln & 3) + 4 * a, k = (ln >> 2) + 8 * bb;
        if (k >= W || k < j) {
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < kGcWarpsMax; ++w)
                if (w < nwarps) sum += part[w * 2 * 16 * T * T + sl];
            out.add(W + k * W + j, (double)sum);
        }
    }
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stage block blk's row slice (W column slices of `rows` floats, stride R) into
// stage blk % NS.  Whole producer warp; lane j copies column j.
__device__ __forceinline__ void pipe_issue(const ScdParams& p, float* Abuf, uint64_t* full, int64_t blk,
                                           int64_t r0, int rows, int lane, int slot, unsigned need,
                                           unsigned& seen, int Rs) {
    const int W = p.W;
    const int Wb = (int)imin64(W, p.L - blk * W);
    const int st = (int)(blk % p.NB);
    float* dst = Abuf + (size_t)st * W * Rs;
    const unsigned bytes = (unsigned)rows * 4u;
    if (lane < Wb) wait_staged(p.progress, p.stage_ctas, need, seen, p.err, kSpinTimeoutNs);
    if (lane == 0) mbar_arrive_expect_tx(&full[st], bytes * (unsigned)Wb);
    __syncwarp();
    if (lane < Wb) bulk_g2s(dst + (size_t)lane * Rs, p.pool + (int64_t)slot * p.ld_dev + r0, bytes, &full[st]);
}

template <bool EXACT, int MODEL>
__global__ void __launch_bounds__(kPipeThreads, 1) k_scd_pipe(const __grid_constant__ ScdParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = p.W, R = p.R, NS = p.NB, G = p.G;
    const int NE = pipe_ne(W);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t nblk = (p.L + W - 1) / W;
    unsigned* cnt = p.bar;       // [kPipeRot]
    unsigned* flg = p.bar + 8;   // [kPipeRot]
    const size_t rbsz = (size_t)NE * kRedStride;
    double* dbuf = p.red + (size_t)kPipeRot * rbsz;  // [kPipeRot][kPipeWMax]
    const double lam_dn = MODEL != kSvm ? p.lambda * (double)p.d : p.lambda * (double)p.n;
    const bool tr = p.trace != nullptr && (tid == 0) && (c == G || c == 0);
    unsigned long long trc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tprev = tr ? (unsigned long long)clock64() : 0;
    auto stamp = [&](int k) {
        if (tr) {
            const unsigned long long t = (unsigned long long)clock64();
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q == k) trc[q] += t - tprev;
            tprev = t;
        }
    };

    if (c == G) {
        // ============================================================ control CTA
        double* sRed = reinterpret_cast<double*>(smem + 128);  // [NE]
        __shared__ double sDprev[kPipeWMax];
        if (tid < kPipeWMax) sDprev[tid] = 0.0;
        int64_t pf_j = 0;
        double pf_a = 0, pf_inv = 0, pf_y = 0;
        auto prefetch = [&](int64_t blk) {
            const int64_t t = blk * W + lane;
            if (warp == 0 && lane < W && t < p.L) {
                pf_j = p.order_j[t];
                pf_a = p.order_a[t];
                pf_inv = p.order_inv[t];
                pf_y = p.order_y[t];
            }
        };
        prefetch(0);
        __syncthreads();
        for (int64_t b = 0; b < nblk; ++b) {
            const int rb = (int)(b % kPipeRot);
            const int Wb = (int)imin64(W, p.L - b * W);
            const int64_t jg = pf_j;
            const double a_in = pf_a, inv_in = pf_inv, y_in = pf_y;
            if (b + 1 < nblk) prefetch(b + 1);
            stamp(3);
            if (tid == 0) {
                const unsigned long long t0 = gtimer();
                while (ld_acquire_u32(&cnt[rb]) < (unsigned)(2 * G)) {  // both groups of every CTA
                    if (gtimer() - t0 > kSpinTimeoutNs) { atomicOr(p.err, 2); break; }
                }
            }
            __syncthreads();
            stamp(0);
            {   // read back (all loads in flight), then zero the buffer for block b + K
                double* red_b = p.red + (size_t)rb * rbsz;
                double v[(kPipeWMax + 2 * kPipeWMax * kPipeWMax + kPipeThreads - 1) / kPipeThreads];
                constexpr int kPer = (kPipeWMax + 2 * kPipeWMax * kPipeWMax + kPipeThreads - 1) / kPipeThreads;
#pragma unroll
                for (int u = 0; u < kPer; ++u) {
                    const int q = tid + u * kPipeThreads;
                    v[u] = q < NE ? ld_cg_f64(&red_b[(size_t)q * kRedStride]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kPer; ++u) {
                    const int q = tid + u * kPipeThreads;
                    if (q < NE) {
                        sRed[q] = v[u];
                        __stcg(&red_b[(size_t)q * kRedStride], 0.0);
                    }
                }
                if (tid == 0) cnt[rb] = 0u;
            }
            __syncthreads();
            stamp(1);
            if (warp == 0) {
                double a = 0, t = 0, tau = 0, cy = 0, scale = 0;
                bool zero = true;
                if (lane < Wb) {
                    a = a_in;
                    double inv = inv_in;
                    zero = inv < 0.0;
                    if (zero) inv = 0.0;
                    double sj = sRed[lane];
                    if (b > 0)
                        for (int k = 0; k < W; ++k) sj = fma(sRed[W + W * W + k * W + lane], sDprev[k], sj);
                    if (MODEL == kLasso) {
                        t = a - sj * inv;
                        tau = lam_dn * inv;
                        scale = -inv;
                    } else if (MODEL == kRidge) {  // ridge / elastic net: inv = 1/(||a||^2 + lambda eta d)
                        t = a - (sj + p.lam_q * a) * inv;
                        tau = p.lam_l1 * inv;
                        scale = -inv;
                    } else {
                        t = fma(lam_dn - y_in * sj, inv, y_in * a);
                        cy = y_in;
                        scale = -y_in * inv;
                    }
                }
                // lane j's scaled Gram row: t_j += scale_j G_jk delta_k for k < j (G_jk = 0 for k >= j;
                // scale = 0 on lanes >= Wb), read from shared memory as the steps go (no register copy)
                double afin = a;
                double* dout = dbuf + (size_t)rb * kPipeWMax;
#pragma unroll
                for (int j = 0; j < kPipeWMax; ++j) {
                    if (j >= Wb) break;
                    double an;
                    if (MODEL != kSvm) {
                        const double mag = fabs(t) - tau;
                        an = mag > 0.0 ? copysign(mag, t) : 0.0;
                        if (zero) an = 0.0;
                    } else {
                        const double u = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                        an = zero ? cy : cy * u;
                    }
                    double dl = an - a;
                    if (lane == j) afin = an;
                    dl = __shfl_sync(0xffffffffu, dl, j);
                    t = fma(scale * sRed[W + j * W + lane], dl, t);
                    if (lane == 0) {  // every lane has delta_j: lane 0 publishes (its own stores, then release)
                        __stcg(&dout[j], dl);
                        sDprev[j] = dl;
                    }
                }
                if (lane == 0)
                    for (int j = Wb; j < W; ++j) {
                        __stcg(&dout[j], 0.0);
                        sDprev[j] = 0.0;
                    }
                stamp(2);
                if (lane == 0) st_release_u32(&flg[rb], (unsigned)(b + 1));
                if (lane < Wb) p.alpha[jg] = afin;
                __syncwarp();
                stamp(4);
            }
        }
    } else {
        // ============================================================ compute CTA c
        // Shared memory: mbarriers | NS stages of W column slices (stride Rs) | v slice (fp64) |
        // per-warp fp32 partials of the Gram block (fast mode) | per-warp u partials.
        uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NS]
        uint64_t* empty = full + 4;                          // [NS]
        const int Rs = pipe_stride(R);
        float* Abuf = reinterpret_cast<float*>(smem + 128);
        size_t off = 128 + align_up_dev((size_t)NS * W * Rs * sizeof(float));
        double* vs = reinterpret_cast<double*>(smem + off);
        off += align_up_dev((size_t)R * sizeof(double));
        float* part = reinterpret_cast<float*>(smem + off);  // [ngc][2 W^2]
        off += align_up_dev((size_t)kGcWarpsMax * 2 * W * W * sizeof(float));
        double* upart = reinterpret_cast<double*>(smem + off);  // [kPipeCompute][32]
        off += align_up_dev((size_t)kPipeCompute * kPipeWMax * sizeof(double));
        double* vpart = reinterpret_cast<double*>(smem + off);  // [3][R] partial v updates
        __shared__ double sDelta[2][kPipeWMax];
        const int64_t r0 = (int64_t)c * R;
        const int rows = (int)imin64(R, p.d4 - r0);
        for (int q = tid; q < NS * W * Rs; q += kPipeThreads) Abuf[q] = 0.0f;
        for (int r = tid; r < R; r += kPipeThreads) vs[r] = r < rows ? p.vt[r0 + r] : 0.0;
        if (tid == 0) {
            for (int q = 0; q < NS; ++q) {
                mbar_init(&full[q], 1);
                mbar_init(&empty[q], kPipeCompute);
            }
            fence_mbar_init();
        }
        fence_proxy_async();
        __syncthreads();

        if (warp == kPipeProd) {
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
                if (q >= NS)
                    mbar_wait_bounded(&empty[q % NS], (unsigned)((q / NS - 1) & 1), p.err, 4, kSpinTimeoutNs);
                pipe_issue(p, Abuf, full, q, r0, rows, lane, slot, need, seen, Rs);
            }
        } else {
            // Two warp groups on different pipes, each with its own named barrier and arrival:
            //   Gram group (warps 0 .. ngc-1, FFMA2): G_{b+1}, C_{b+1,b} as soon as block b+1
            //     has landed -- needs no delta;
            //   v group (the other compute warps, fp64): wait delta_{b-1}, v += A_{b-1} delta_{b-1},
            //     u_{b+1} = A_{b+1}^T v_b.
            // Each group REDs its entries, fences and adds 1 to cnt[(b+1) % K] (the control CTA
            // waits for 2 G arrivals).  A stage is released when every compute warp is done with
            // it: the Gram warps after G/C of the next block (its last read, as the C partner),
            // the v warps after the v update.
            const int n4 = rows >> 2;
            auto stage = [&](int64_t blk) { return Abuf + (size_t)(blk % NS) * W * Rs; };
            auto wait_data = [&](int64_t blk) {
                mbar_wait_bounded(&full[blk % NS], (unsigned)((blk / NS) & 1), p.err, 8, kSpinTimeoutNs);
            };
            auto out_of = [&](int64_t blk) { return RedOut{p.red + (size_t)(blk % kPipeRot) * rbsz, 0}; };
            auto arrive_cnt = [&](int64_t blk) {  // after the group's named barrier
#ifndef DUHL_EXP_NOFENCE
                __threadfence();
#endif
                atomicAdd(&cnt[blk % kPipeRot], 1u);
            };
            constexpr int ngc = kGcWarps, nvw = kPipeCompute - kGcWarps;
            if (warp < ngc) {
                // ---------------------------------------------------------- Gram group
                const int gw = warp, gtid = tid;
                const int w4lo = (gw * n4) / ngc, w4hi = ((gw + 1) * n4) / ngc;
                float* mypart = part + (size_t)gw * 2 * W * W;
                for (int64_t b = -1; b + 1 < nblk; ++b) {
                    stamp(7);
                    wait_data(b + 1);
                    stamp(0);
                    const float* A1 = stage(b + 1);
                    const float* A0 = b >= 0 ? stage(b) : A1;  // block 0: C is never read
                    const RedOut out = out_of(b + 1);
                    if (!EXACT && p.gram_tc && (W == 32 || (p.gram_tc > 1 && (W == 12 || W == 16 || W == 24)))) {
                        switch (W >> 2) {
                            case 3: gc_warp_tc<3>(A1, A0, Rs, w4lo, w4hi, lane, mypart); break;
                            case 4: gc_warp_tc<4>(A1, A0, Rs, w4lo, w4hi, lane, mypart); break;
                            case 6: gc_warp_tc<6>(A1, A0, Rs, w4lo, w4hi, lane, mypart); break;
                            default: gc_warp_tc<8>(A1, A0, Rs, w4lo, w4hi, lane, mypart); break;
                        }
                    } else switch (W >> 2) {
                        case 1: gc_warp<EXACT, 1>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 2: gc_warp<EXACT, 2>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 3: gc_warp<EXACT, 3>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 4: gc_warp<EXACT, 4>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 5: gc_warp<EXACT, 5>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 6: gc_warp<EXACT, 6>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        case 7: gc_warp<EXACT, 7>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                        default: gc_warp<EXACT, 8>(A1, A0, Rs, W, w4lo, w4hi, lane, mypart, out); break;
                    }
                    __syncwarp();
                    if (b >= 0 && lane == 0) mbar_arrive(&empty[b % NS]);  // last Gram read of block b
                    stamp(1);
                    if (!EXACT) {  // sum the warps' partials and add one (fp64) RED per entry
                        named_sync(kBarGc, ngc * 32);
                        switch (W >> 2) {
                            case 1: gc_sum<1>(part, W, gtid, ngc, out); break;
                            case 2: gc_sum<2>(part, W, gtid, ngc, out); break;
                            case 3: gc_sum<3>(part, W, gtid, ngc, out); break;
                            case 4: gc_sum<4>(part, W, gtid, ngc, out); break;
                            case 5: gc_sum<5>(part, W, gtid, ngc, out); break;
                            case 6: gc_sum<6>(part, W, gtid, ngc, out); break;
                            case 7: gc_sum<7>(part, W, gtid, ngc, out); break;
                            default: gc_sum<8>(part, W, gtid, ngc, out); break;
                        }
                    }
                    named_sync(kBarGc, ngc * 32);  // partials consumed, every RED issued
                    if (gtid == 0) arrive_cnt(b + 1);
                    stamp(2);
                }
            } else {
                // ---------------------------------------------------------- v group
                const int vw = warp - ngc, vtid = tid - ngc * 32;
                constexpr int kVThreads = nvw * 32;
                const int w4lo = (vw * n4) / nvw, w4hi = ((vw + 1) * n4) / nvw;
                const int vq = n4 > 0 ? kVThreads / n4 : 1;
                const int vparts = vq < 1 ? 1 : (vq > 4 ? 4 : vq);
                auto wait_delta = [&](int64_t blk) {  // delta_blk -> sDelta[blk & 1]
                    if (vw == 0) {
                        const unsigned* f = &flg[blk % kPipeRot];
                        const unsigned long long t0 = gtimer();
                        while (ld_acquire_u32(f) < (unsigned)(blk + 1)) {
                            if (gtimer() - t0 > kSpinTimeoutNs) { atomicOr(p.err, 16); break; }
                        }
                        if (lane < W) sDelta[blk & 1][lane] = ld_cg_f64(&dbuf[(size_t)(blk % kPipeRot) * kPipeWMax + lane]);
                    }
                    named_sync(kBarV, kVThreads);
                };
                // v slice += A_blk delta_blk (delta = 0 beyond the block); short slices split the
                // columns over `vparts` thread groups, partials of groups >= 1 via shared memory
                auto vupdate = [&](int64_t blk) {
                    const double* dl = sDelta[blk & 1];
                    double2* v2 = reinterpret_cast<double2*>(vs);
                    const uint32_t a0 = smem_addr(stage(blk));
                    const int span = n4 * vparts;
                    for (int it = vtid; it < span; it += kVThreads) {
                        const int r4 = it % n4, part_ = it / n4;
                        const int jlo = (W / 4 * part_) / vparts * 4, jhi = (W / 4 * (part_ + 1)) / vparts * 4;
                        double2 p01 = make_double2(0.0, 0.0), p23 = p01, q01 = p01, q23 = p01;
                        for (int j = jlo; j < jhi; j += 4) {  // W % 4 == 0: two independent chains
#pragma unroll
                            for (int u = 0; u < 4; u += 2) {
                                const float4 x = lds_f4(a0 + 4u * (uint32_t)((j + u) * Rs) + 16u * r4);
                                const float4 y = lds_f4(a0 + 4u * (uint32_t)((j + u + 1) * Rs) + 16u * r4);
                                const double dx = dl[j + u], dy = dl[j + u + 1];
                                p01.x = fma(dx, (double)x.x, p01.x);
                                p01.y = fma(dx, (double)x.y, p01.y);
                                p23.x = fma(dx, (double)x.z, p23.x);
                                p23.y = fma(dx, (double)x.w, p23.y);
                                q01.x = fma(dy, (double)y.x, q01.x);
                                q01.y = fma(dy, (double)y.y, q01.y);
                                q23.x = fma(dy, (double)y.z, q23.x);
                                q23.y = fma(dy, (double)y.w, q23.y);
                            }
                        }
                        p01.x += q01.x; p01.y += q01.y; p23.x += q23.x; p23.y += q23.y;
                        if (part_ == 0) {
                            double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
                            v01.x += p01.x; v01.y += p01.y; v23.x += p23.x; v23.y += p23.y;
                            v2[2 * r4] = v01;
                            v2[2 * r4 + 1] = v23;
                        } else {
                            double2* vp = reinterpret_cast<double2*>(vpart) + 2 * ((size_t)(part_ - 1) * n4 + r4);
                            vp[0] = p01;
                            vp[1] = p23;
                        }
                    }
                    if (vparts > 1) {
                        named_sync(kBarV, kVThreads);
                        for (int r4 = vtid; r4 < n4; r4 += kVThreads) {
                            double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
                            for (int q = 1; q < vparts; ++q) {
                                const double2* vp = reinterpret_cast<const double2*>(vpart) + 2 * ((size_t)(q - 1) * n4 + r4);
                                v01.x += vp[0].x; v01.y += vp[0].y; v23.x += vp[1].x; v23.y += vp[1].y;
                            }
                            v2[2 * r4] = v01;
                            v2[2 * r4 + 1] = v23;
                        }
                    }
                };
                // u_blk = A_blk^T v (v = v_{blk-1}) over this warp's rows, fp64, summed across the group
                auto u_block = [&](int64_t blk) {
                    const float* A1 = stage(blk);
                    const double2* v2 = reinterpret_cast<const double2*>(vs);
                    if (W > 16) {  // lane j = column j (no cross-lane reduction; two chains)
                        if (lane < W) {
                            const uint32_t ca = smem_addr(A1 + (size_t)lane * Rs);
                            double acc0 = 0.0, acc1 = 0.0;
                            for (int r4 = w4lo; r4 < w4hi; ++r4) {
                                const float4 a4 = lds_f4(ca + 16u * r4);
                                const double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
                                acc0 = fma((double)a4.x, v01.x, acc0);
                                acc1 = fma((double)a4.y, v01.y, acc1);
                                acc0 = fma((double)a4.z, v23.x, acc0);
                                acc1 = fma((double)a4.w, v23.y, acc1);
                            }
                            upart[vw * kPipeWMax + lane] = acc0 + acc1;
                        }
                    } else {  // lane (jq, rs) = (lane & 3, lane >> 2): columns jq + 4a, rows rs mod 8
                        const int jq = lane & 3, rs = lane >> 2, T = W >> 2;
                        double acc[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) acc[a] = 0.0;
                        double acc2[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) acc2[a] = 0.0;
                        for (int r4 = w4lo + rs; r4 < w4hi; r4 += 8) {
                            const double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
#pragma unroll
                            for (int a = 0; a < 4; ++a) {
                                if (a >= T) break;
                                const float4 x = lds_f4(smem_addr(A1 + (size_t)(jq + 4 * a) * Rs) + 16u * r4);
                                acc[a] = fma((double)x.x, v01.x, acc[a]);   // two chains per column
                                acc2[a] = fma((double)x.y, v01.y, acc2[a]);
                                acc[a] = fma((double)x.z, v23.x, acc[a]);
                                acc2[a] = fma((double)x.w, v23.y, acc2[a]);
                            }
                        }
#pragma unroll
                        for (int a = 0; a < 4; ++a) acc[a] += acc2[a];
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            if (a >= T) break;
                            double t = acc[a];
                            t += __shfl_xor_sync(0xffffffffu, t, 4);
                            t += __shfl_xor_sync(0xffffffffu, t, 8);
                            t += __shfl_xor_sync(0xffffffffu, t, 16);
                            if (rs == 0) upart[vw * kPipeWMax + jq + 4 * a] = t;
                        }
                    }
                    named_sync(kBarV, kVThreads);
                    if (vtid < W) {
                        double sum = 0.0;
#pragma unroll
                        for (int w = 0; w < kPipeCompute; ++w)
                            if (w < nvw) sum += upart[w * kPipeWMax + vtid];
                        out_of(blk).add(vtid, sum);
                    }
                };
                // b = -1: u_0 against the initial v; b = nblk: the last v update
                const bool trv = p.trace != nullptr && c == 0 && vtid == 0;
                unsigned long long tv = trv ? (unsigned long long)clock64() : 0;
                auto vstamp = [&](int k) {
                    if (trv) {
                        const unsigned long long t = (unsigned long long)clock64();
#pragma unroll
                        for (int q = 3; q < 7; ++q)
                            if (q == k) trc[q] += t - tv;
                        tv = t;
                    }
                };
                for (int64_t b = -1; b <= nblk; ++b) {
                    vstamp(6);
                    if (b >= 1) {
                        wait_delta(b - 1);
                        vstamp(3);
                        vupdate(b - 1);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[(b - 1) % NS]);
                        named_sync(kBarV, kVThreads);  // v_b complete before the u tiles read it
                        vstamp(4);
                    }
                    if (b + 1 < nblk) {
                        wait_data(b + 1);
                        u_block(b + 1);
                        named_sync(kBarV, kVThreads);
                        if (vtid == 0) arrive_cnt(b + 1);
                        vstamp(5);
                    }
                }
                if (trv)
                    for (int q = 3; q < 7; ++q)
                        if (trc[q]) atomicAdd(&p.trace[8 + q], trc[q]);
            }
        }
        __syncthreads();
        for (int r = tid; r < rows; r += kPipeThreads) p.vt[r0 + r] = vs[r];
    }
    if (tr)
        for (int q = 0; q < 8; ++q)
            if (trc[q]) atomicAdd(&p.trace[(c == G ? 0 : 8) + q], trc[q]);
}

cudaError_t launch_scd_pipe(const ScdParams& p, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    const size_t smem = pipe_smem_bytes(p.W, p.R, p.NB);
    const void* fn = p.model == kLasso
                         ? (p.exact ? (const void*)k_scd_pipe<true, kLasso> : (const void*)k_scd_pipe<false, kLasso>)
                     : (p.model == kRidge || p.model == kElastic)
                         ? (p.exact ? (const void*)k_scd_pipe<true, kRidge> : (const void*)k_scd_pipe<false, kRidge>)
                         : (p.exact ? (const void*)k_scd_pipe<true, kSvm> : (const void*)k_scd_pipe<false, kSvm>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ScdParams q = p;
    void* args[] = {&q};
    e = cudaLaunchCooperativeKernel(fn, dim3(p.G + 1), dim3(kPipeThreads), args, smem, st);
    ++*launches;
    return e;
}
