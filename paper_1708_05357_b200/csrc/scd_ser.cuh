// scd_ser.cuh -- exact sequential SCD epoch, Gram-block form WITHOUT the cross
// Gram (App. D closed forms in the exact sequential order).
// Included by kernels.cu (uses its tile4 helper, the RED layout, the bounded waits
// and k_scd_gram's warp layout).
//
// k_scd_gram overlaps block b's control chain with block b+1's partials, which
// forces u_{b+1} to be taken against v_b (before block b's update) and the cross
// Gram C_{b+1,b} = A_{b+1}^T A_b to correct it: 144 of the 222 reduced entries
// per block at W = 12 and ~60 % of the compute warps' FMAs, which bind that
// kernel (C4: compute warps 7.8 us per block).  Here u_{b+1} = a^T v at the start
// of block b+1 is assembled by the compute warps themselves:
//     u_{b+1} = A_{b+1}^T v_b            (fp64, before delta_b is known: off the chain)
//             + A_{b+1}^T (A_b delta_b)  (after delta_b: the only work on the chain)
// so the control warp needs only u and G:  s_j = u_j + sum_{k<j} G_jk delta_k
// (== a_j^T v at coordinate j's visit).  The correction term is the cross-Gram
// term of k_scd_gram in another order (C delta = A_{b+1}^T (A_b delta)); like
// the Gram entries it is taken in fp32 in fast mode (delta rounded to fp32,
// fp32 products and row sums inside a thread, fp64 from the thread sums on) and
// in fp64 in exact mode.  The exact fp64 update v += A_b delta_b runs after the
// arrival (fast mode) or is the correction sweep itself (exact mode: v += dv,
// dv = A_b delta_b in fp64).
//
// Per block b, compute warps (6):
//   off the chain: G_{b+1} tiles -> red[(b+1) % 6]; u'_{b+1} = A_{b+1}^T v_b (registers)
//   wait delta_b; correction sweep; warp reduce-scatter -> shared memory -> warp 0
//     REDs u_{b+1} (one RED per entry per CTA) and ARRIVEs(b+1)
//   off the chain: fast mode v += A_b delta_b (fp64); free stage b (mbarrier empty)
// control warp: WAIT(b) -> zero red[(b+5) % 6] (CTA 0) -> read red[b % 6] ->
//     the W steps -> publish delta_b (mbarrier dfull[b & 1]).
// producer warp: block q into stage q % 3 once block q-3's stage is free.
// Zeroing rule: CTA 0 zeroes red[(b+5) % 6] (block b-1's, next block b+5's) right
// after WAIT(b).  Every CTA read block b-1 before consuming delta_{b-1}, i.e. before
// its ARRIVE(b).  Block b+5's first writes (G tiles, iteration b+4) follow that
// CTA's consumption of delta_{b+3}, which needs CTA 0's ARRIVE(b+3), issued after
// CTA 0 consumed delta_{b+2} -- published by CTA 0's control after the zeroing.
// Arrival counters: bar[b & 1] counts the arrivals of blocks b, b-2, ...; a CTA
// ARRIVEs(b+1) only after its own WAIT(b) completed, so no CTA can ARRIVE(b+2)
// before every WAIT(b) saw its target.
// Measured variants (C4 fast mode, 140 CTAs, 4.65 ms per pass as built): fusing the v update
// with u'_{b+2} in one sweep 4.91 ms (u' then waits on the update's 12-deep DFMA chains);
// warp 7 taking a double share of the sweeps (TMA issue moved into it) 4.65 ms -- the
// compute warps are bound by their per-lane latency chains, not by sub-partition issue.
#pragma once

static_assert(kRedBufs == 6, "the zeroing rule of k_scd_ser assumes 6 reduction buffers");

// Warps: control = 3, producer = the last, compute = the others (k_scd_gram's layout at 8).
// Measured (C4, 140 CTAs, fast / exact ms per pass): 8 warps 4.69 / 6.46, 12 warps 4.96 / 6.67,
// 16 warps 5.30 / 8.94 (register spills) -- the compute warps' per-block work (~540 KB of
// shared-memory reads: G tiles 230, u' 81, correction 138, v update 92) does not shrink with
// more warps.  Taking u' inside the k0 = 0 Gram tiles (x slices already in registers, no u'
// sweep) and sharing the x loads of diagonal tiles: 7.49 ms -- the fp64 u' work then sits on
// the five tile warps unevenly and the kernel needs a 168-byte local frame.  Sharing the x
// loads of diagonal tiles alone (12 of 40 loads per row group): fast 4.79 vs 4.68 ms, exact
// 6.25 vs 6.47 -- not kept.  The fast-mode v update with two half-depth chains per component
// 4.58 ms, or with the thread's two row groups interleaved 4.61, against 4.59-4.63: noise.
// Warps 1-5 only arriving at the u-publish barrier (bar.arrive) and going on to their v update
// while warp 0 sums and releases: 4.74-4.78 vs 4.66-4.69 -- slower.
#ifndef DUHL_SER_WARPS
#define DUHL_SER_WARPS 8
#endif
constexpr int kSerThreads = DUHL_SER_WARPS * 32;
constexpr int kSerCompute = DUHL_SER_WARPS - 2;
constexpr int kSerProd = DUHL_SER_WARPS - 1;


// u'_j = a_j^T v over the thread's 4-row groups (fp64), NW = W columns unrolled.
template <int NW>
__device__ __forceinline__ void ser_uprime(const float* __restrict__ An, int R, const double2* v2, int r4_0,
                                           int nr4, double (&u)[16]) {
    for (int r4 = r4_0; r4 < nr4; r4 += kSerCompute * 32) {
        const double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
        float4 y[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) y[j] = reinterpret_cast<const float4*>(An + (size_t)j * R)[r4];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            double acc = u[j];
            acc = fma((double)y[j].x, v01.x, acc);
            acc = fma((double)y[j].y, v01.y, acc);
            acc = fma((double)y[j].z, v23.x, acc);
            acc = fma((double)y[j].w, v23.y, acc);
            u[j] = acc;
        }
    }
}

// The correction sweep (on the chain): dv = A_b delta_b per 4-row group, u_j += a_{b+1,j}^T dv
// (nxt).  EXACT: fp64, and v += dv (the exact update itself).  Fast: fp32 (FFMA2), thread
// sums converted to fp64 once.  A ragged block needs no masking: delta_j = 0 past its last
// coordinate, and u_j past it is never REDed (stage columns there hold finite earlier data).
template <int NW, bool EXACT>
__device__ __forceinline__ void ser_corr(const float* __restrict__ A, const float* __restrict__ An, int R,
                                         const double* __restrict__ dcur, double2* v2, int r4_0, int nr4,
                                         bool nxt, double (&u)[16]) {
    if (EXACT) {
        double d[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) d[j] = dcur[j];
        for (int r4 = r4_0; r4 < nr4; r4 += kSerCompute * 32) {
            float4 x[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) x[j] = reinterpret_cast<const float4*>(A + (size_t)j * R)[r4];
            double2 d01 = make_double2(0.0, 0.0), d23 = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                d01.x = fma(d[j], (double)x[j].x, d01.x);
                d01.y = fma(d[j], (double)x[j].y, d01.y);
                d23.x = fma(d[j], (double)x[j].z, d23.x);
                d23.y = fma(d[j], (double)x[j].w, d23.y);
            }
            double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
            v01.x += d01.x;
            v01.y += d01.y;
            v23.x += d23.x;
            v23.y += d23.y;
            v2[2 * r4] = v01;
            v2[2 * r4 + 1] = v23;
            if (nxt) {
                float4 y[NW];
#pragma unroll
                for (int j = 0; j < NW; ++j) y[j] = reinterpret_cast<const float4*>(An + (size_t)j * R)[r4];
#pragma unroll
                for (int j = 0; j < NW; ++j) {
                    double acc = u[j];
                    acc = fma((double)y[j].x, d01.x, acc);
                    acc = fma((double)y[j].y, d01.y, acc);
                    acc = fma((double)y[j].z, d23.x, acc);
                    acc = fma((double)y[j].w, d23.y, acc);
                    u[j] = acc;
                }
            }
        }
    } else {
        if (!nxt) return;
        float d[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) d[j] = (float)dcur[j];
        float2 c[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) c[j] = make_float2(0.f, 0.f);
        for (int r4 = r4_0; r4 < nr4; r4 += kSerCompute * 32) {
            float4 x[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) x[j] = reinterpret_cast<const float4*>(A + (size_t)j * R)[r4];
            float2 d01 = make_float2(0.f, 0.f), d23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                ffma2(d01, d[j], d[j], x[j].x, x[j].y);
                ffma2(d23, d[j], d[j], x[j].z, x[j].w);
            }
            float4 y[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) y[j] = reinterpret_cast<const float4*>(An + (size_t)j * R)[r4];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                ffma2(c[j], y[j].x, y[j].y, d01.x, d01.y);
                ffma2(c[j], y[j].z, y[j].w, d23.x, d23.y);
            }
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) u[j] += (double)c[j].x + (double)c[j].y;
    }
}

// Fast mode, off the chain: v += A_b delta_b in fp64, the oracle's column order.
template <int NW>
__device__ __forceinline__ void ser_vupdate(const float* __restrict__ A, int R, const double* __restrict__ dcur,
                                            double2* v2, int r4_0, int nr4) {
    double d[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) d[j] = dcur[j];
    for (int r4 = r4_0; r4 < nr4; r4 += kSerCompute * 32) {
        double2 v01 = v2[2 * r4], v23 = v2[2 * r4 + 1];
        float4 x[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) x[j] = reinterpret_cast<const float4*>(A + (size_t)j * R)[r4];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            v01.x = fma(d[j], (double)x[j].x, v01.x);
            v01.y = fma(d[j], (double)x[j].y, v01.y);
            v23.x = fma(d[j], (double)x[j].z, v23.x);
            v23.y = fma(d[j], (double)x[j].w, v23.y);
        }
        v2[2 * r4] = v01;
        v2[2 * r4 + 1] = v23;
    }
}

#define SER_DISPATCH(W, CALL)                 \
    switch (W) {                              \
        case 4: { constexpr int NW = 4; CALL; break; }   \
        case 8: { constexpr int NW = 8; CALL; break; }   \
        case 12: { constexpr int NW = 12; CALL; break; } \
        default: { constexpr int NW = 16; CALL; break; } \
    }

template <bool EXACT, int MODEL>
__global__ void __launch_bounds__(kSerThreads, 1) k_scd_ser(const __grid_constant__ ScdParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = p.W, R = p.R, T = W / 4;
    const int NQ = scd_off_C(W);  // reduced entries per block: u [0, W), G lower after
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [3] stage data landed
    uint64_t* empty = full + kScdStages;                 // [3] stage consumed
    uint64_t* dfull = empty + kScdStages;                // [2] delta of a block published
    size_t off = 128;
    float* Abuf = reinterpret_cast<float*>(smem + off);
    off += align_up_dev((size_t)kScdStages * W * R * sizeof(float));
    double* vs = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)R * sizeof(double));
    double* sG = reinterpret_cast<double*>(smem + off);
    off += align_up_dev((size_t)scd_nred(W) * sizeof(double));
    double* delta = reinterpret_cast<double*>(smem + off);  // [2][16]
    __shared__ double sT[16], sP[16], sA[16], sS[16], sC[16 * 16];
    __shared__ int sZ[16];
    __shared__ double su[kSerCompute * 16];  // per-compute-warp u partials

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = (int64_t)c * R;
    const int rows = (int)imin64(R, p.d4 - r0);
    const double lam_dn = MODEL != kSvm ? p.lambda * (double)p.d : p.lambda * (double)p.n;
    const size_t bufsz = (size_t)scd_nred(W) * kRedGroups * kRedStride;
    const int grp = c % kRedGroups;

    for (int q = tid; q < kScdStages * W * R; q += kSerThreads) Abuf[q] = 0.0f;
    for (int r = tid; r < R; r += kSerThreads) vs[r] = r < rows ? p.vt[r0 + r] : 0.0;
    if (tid == 0) {
        for (int q = 0; q < kScdStages; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kSerCompute);
        }
        mbar_init(&dfull[0], 1);
        mbar_init(&dfull[1], 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();

    // developer trace (ScdParams::trace, DUHL_SCD_TRACE): per-phase cycle counts of CTA 0 /
    // CTA G-1 -- control lane 0: 0 WAIT, 1 zero + read-back, 2 steps + publish, 3 other;
    // compute thread 0: 4 data + G tiles + u', 5 wait delta, 6 correction sweep,
    // 7 reduce + REDs + arrive + (fast) v update
    const bool trc_cta = p.trace && (c == 0 || c == p.G - 1);
    const bool tr = trc_cta && (tid == kCtrlWarp * 32 || tid == 0);
    unsigned long long trc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
    const bool ctrl = warp == kCtrlWarp, prod = warp == kSerProd;
    const int cw = warp < kCtrlWarp ? warp : (warp > kCtrlWarp && warp < kSerProd ? warp - 1 : -1);

    // per-compute-warp G tile lists, built once: item = jt | k0 << 4 | kw << 9 | part << 13
    // (4 x 8 tiles split by rows into two items, so W = 12's four tiles are six equal items)
    __shared__ int witems[kSerCompute][12];
    __shared__ int wcount[kSerCompute];
    if (tid == 0) {
        for (int w = 0; w < kSerCompute; ++w) wcount[w] = 0;
        int item = 0;
        for (int cost = 2; cost >= 1; --cost)
            for (int jt = 0; jt < T; ++jt)
                for (int k0 = 0; k0 < 4 * jt + 4; k0 += 8) {
                    const int kw = 4 * jt + 4 - k0 >= 8 ? 8 : 4;
                    if ((kw == 8) != (cost == 2)) continue;
                    for (int part = 0; part < (kw == 8 ? 2 : 1); ++part) {
                        const int rnd = item / kSerCompute, pos = item % kSerCompute;
                        const int owner = (rnd & 1) ? kSerCompute - 1 - pos : pos;
                        ++item;
                        if (wcount[owner] < 12) witems[owner][wcount[owner]++] = jt | k0 << 4 | kw << 9 | part << 13;
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
            if (q >= kScdStages)  // block q-3 done: its stage is free
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
            const int64_t jg = pf_j;
            const double a_in = pf_a, inv_in = pf_inv, y_in = pf_y;
            if (b + 1 < nblk) prefetch_coords(b + 1);
            stamp(3);
            {   // WAIT(b): every lane polls with acquire (no separate fence on the critical path)
                const unsigned target = (unsigned)((b / 2 + 1) * (int64_t)p.G);
                const unsigned long long t0 = gtimer();
                while (ld_acquire_u32(&p.bar[b & 1]) < target) {
                    __nanosleep(32);
                    if (gtimer() - t0 > kSpinTimeoutNs) {
                        atomicOr(p.err, 2);
                        break;
                    }
                }
            }
            __syncwarp();
            stamp(0);
            if (c == 0)
                for (int q = lane; q < NQ * kRedGroups; q += 32)
                    p.red[(size_t)((b + 5) % kRedBufs) * bufsz + (size_t)q * kRedStride] = 0.0;
            {   // all loads of the reduced block in flight at once
                const double* red_b = p.red + (size_t)(b % kRedBufs) * bufsz;
                for (int q0 = 0; q0 < NQ; q0 += 4 * 32) {
                    double v[4][kRedGroups];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = min(q0 + u * 32 + lane, NQ - 1);
#pragma unroll
                        for (int g = 0; g < kRedGroups; ++g)
                            v[u][g] = ld_cg_f64(&red_b[((size_t)q * kRedGroups + g) * kRedStride]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = q0 + u * 32 + lane;
                        double s = 0.0;
#pragma unroll
                        for (int g = 0; g < kRedGroups; ++g) s += v[u][g];
                        if (q < NQ) sG[q] = s;
                    }
                }
            }
            __syncwarp();
            stamp(1);
            // lane j < Wb owns coordinate j: pre-activation t_j with every correction
            // folded in by one DFMA (see k_scd_gram)
            double a = 0, t = 0, tau = 0, cy_ = 0, scale = 0, afin = 0;
            bool zero = true;
            if (lane < Wb) {
                a = a_in;
                double inv = inv_in;
                zero = inv < 0.0;
                if (zero) inv = 0.0;
                const double yy = y_in;
                const double sj = sG[lane];  // u_j = a_j^T v at the start of block b
                if (MODEL == kLasso) {
                    t = a - sj * inv;
                    tau = lam_dn * inv;
                    scale = -inv;
                } else if (MODEL == kRidge) {
                    t = a - (sj + p.lam_q * a) * inv;
                    tau = p.lam_l1 * inv;
                    scale = -inv;
                } else {
                    t = fma(lam_dn - yy * sj, inv, yy * a);
                    cy_ = yy;
                    scale = -yy * inv;
                }
            }
            double* dcur = delta + (size_t)(b & 1) * 16;
            if (lane < 16) {
                sT[lane] = t;
                sP[lane] = MODEL != kSvm ? tau : cy_;
                sZ[lane] = zero ? 1 : 0;
                sA[lane] = a;
                sS[lane] = scale;
            }
            __syncwarp();
#pragma unroll
            for (int e0 = 0; e0 < 256; e0 += 32) {
                const int e = e0 + lane, q = e >> 4, j = e & 15;
                sC[e] = (j < q && q < Wb) ? sS[q] * sG[scd_off_G(W) + q * (q - 1) / 2 + j] : 0.0;
            }
            __syncwarp();
            double tq[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) tq[q] = sT[q];
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
            stamp(2);
            if (lane < Wb && c == 0) p.alpha[jg] = afin;
        }
    } else {
        // ---------------------------------------------------------------- compute
        const int ctid = cw * 32 + lane, nr4 = rows >> 2;
        const double2* v2c = reinterpret_cast<const double2*>(vs);
        double2* v2 = reinterpret_cast<double2*>(vs);
        auto gtiles = [&](int64_t blk) {  // G_blk (lower) -> red[blk % 6]
            const float* A1 = stage(blk);
            const RedOut out{p.red + (size_t)(blk % kRedBufs) * bufsz, grp};
            const int cnt = wcount[cw];
            for (int it = 0; it < cnt; ++it) {
                const int code = witems[cw][it];
                const int jt = code & 15, k0 = (code >> 4) & 31, kw = (code >> 9) & 15, part = (code >> 13) & 1;
                const int lo = kw == 8 ? (part == 0 ? 0 : half) : 0;
                const int hi = kw == 8 ? (part == 0 ? half : rows) : rows;
                const float* Aj = A1 + (size_t)(4 * jt) * R;
                if (kw == 8) tile4<EXACT, 8, true>(Aj, A1 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
                else tile4<EXACT, 4, true>(Aj, A1 + (size_t)k0 * R, R, lo, hi, lane, 4 * jt, k0, out, W);
            }
        };
        // warp reduce-scatter of the u partials -> one row per warp in shared memory -> warp 0
        // sums the rows, one RED per entry (same-address REDs serialise at the L2 slice: G per
        // entry and block, not 6 G), then ARRIVE(blk) with a release add (the G-tile REDs of
        // every compute warp precede the barrier; the release is cumulative over them)
        auto publish_u = [&](int64_t blk, double (&u)[16]) {
            const int Wn = (int)imin64(W, p.L - blk * W);
            const double s = reduce_scatter<double, 16>(u, lane);
            if (lane < 16) su[cw * 16 + lane] = s;
            named_sync(kBarCompute, kSerCompute * 32);
            if (cw == 0) {
                if (lane < Wn) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < kSerCompute; ++w) t += su[w * 16 + lane];
                    const RedOut out{p.red + (size_t)(blk % kRedBufs) * bufsz, grp};
                    out.add(lane, t);
                }
                __syncwarp();
                if (lane == 0) {
#ifdef DUHL_EXP_SER_SCFENCE  // developer A/B: sequentially consistent fence + relaxed add
                    __threadfence();
                    atomicAdd(&p.bar[blk & 1], 1u);
#else
                    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&p.bar[blk & 1]), "r"(1u)
                                 : "memory");
#endif
                }
            }
        };
        auto wait_data = [&](int64_t blk) {
            mbar_wait_bounded(&full[blk % kScdStages], (unsigned)((blk / kScdStages) & 1), p.err, 8,
                              kSpinTimeoutNs);
        };
        auto wait_delta = [&](int64_t blk) {
            mbar_wait_bounded(&dfull[blk & 1], (unsigned)((blk >> 1) & 1), p.err, 16, kSpinTimeoutNs);
        };
        double u[16];
        auto zero_u = [&]() {
#pragma unroll
            for (int j = 0; j < 16; ++j) u[j] = 0.0;
        };
        if (nblk > 0) {
            wait_data(0);
            gtiles(0);
            zero_u();
            SER_DISPATCH(W, (ser_uprime<NW>(stage(0), R, v2c, ctid, nr4, u)));
            publish_u(0, u);  // u_0 = A_0^T v at the start of the epoch; ARRIVE(0)
        }
        for (int64_t b = 0; b < nblk; ++b) {
            const bool nxt = b + 1 < nblk;
            stamp(7);
            zero_u();
            if (nxt) {
                wait_data(b + 1);
                gtiles(b + 1);
                SER_DISPATCH(W, (ser_uprime<NW>(stage(b + 1), R, v2c, ctid, nr4, u)));  // against v_b
                stamp(4);
            }
            wait_delta(b);
            stamp(5);
            const double* dcur = delta + (size_t)(b & 1) * 16;
            SER_DISPATCH(W, (ser_corr<NW, EXACT>(stage(b), nxt ? stage(b + 1) : nullptr, R, dcur, v2, ctid, nr4,
                                                 nxt, u)));
            stamp(6);
            if (nxt) publish_u(b + 1, u);
            if (!EXACT) SER_DISPATCH(W, (ser_vupdate<NW>(stage(b), R, dcur, v2, ctid, nr4)));
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b % kScdStages]);  // block b's stage is free
        }
        stamp(7);
    }
    __syncthreads();
    for (int r = tid; r < rows; r += kSerThreads) p.vt[r0 + r] = vs[r];
    if (tr)
        for (int q = 0; q < 8; ++q)
            if (trc[q]) atomicAdd(&p.trace[(c == 0 ? 0 : 8) + q], trc[q]);
}

cudaError_t launch_scd_ser(const ScdParams& p, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    if (p.W > 16) return cudaErrorInvalidValue;
    size_t smem = scd_smem_bytes(p.W, p.R, kScdStages);
    const void* fn = p.model == kLasso
                         ? (p.exact ? (const void*)k_scd_ser<true, kLasso> : (const void*)k_scd_ser<false, kLasso>)
                     : (p.model == kRidge || p.model == kElastic)
                         ? (p.exact ? (const void*)k_scd_ser<true, kRidge> : (const void*)k_scd_ser<false, kRidge>)
                         : (p.exact ? (const void*)k_scd_ser<true, kSvm> : (const void*)k_scd_ser<false, kSvm>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ScdParams q = p;
    void* args[] = {&q};
    e = cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(kSerThreads), args, smem, st);
    ++*launches;
    return e;
}
