// device.cuh -- sm_100a device helpers for the DuHL kernels (no host code).
//
// PTX wrappers for the Blackwell async-copy path (mbarrier + cp.async.bulk,
// SASS UBLKCP / SYNCS), acquire/release global accesses for the grid barrier,
// warp reductions in fp64, and the closed-form coordinate/gap arithmetic of the
// paper (App. D, App. E).  Independent of oracle/ (shares nothing with it).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace duhl {

constexpr int kLasso = 0;

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
constexpr int kSvm = 1;
constexpr int kRidge = 2;  // ridge regression: the regression structure of Lasso, g = (lambda/2) a^2
constexpr int kElastic = 3;  // elastic net: g = lambda (eta/2 a^2 + (1-eta)|a|), 0 < eta < 1

// ---------------------------------------------------------------- counter RNG
// splitmix64 finaliser; permutation key(seed, round, pass, j) (DESIGN.md
// "Randomness").  Written independently of the oracle's copy of the same
// documented generator.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t perm_key(uint64_t seed, int64_t round, int64_t pass,
                                                      int64_t j) {
    uint64_t h = mix64(seed);
    h = mix64(h ^ (uint64_t)round);
    h = mix64(h ^ (uint64_t)pass);
    return mix64(h ^ (uint64_t)j);
}

// ---------------------------------------------------------------- closed forms
// Exact coordinate step (App. D).  s = a_j^T v~ (Lasso, v~ = A alpha - b) or
// a_j^T v^ (SVM, v^ = A alpha); nrm = ||a_j||^2.
//   Lasso, eta = 0: gamma = (alpha nrm - s)/nrm, tau = lambda d/nrm,
//                               alpha' = sign(gamma) max(|gamma| - tau, 0)
//   Ridge (eta = 1): alpha' = (alpha nrm - s) / (nrm + lambda d)
//   SVM: Delta = (y - s/(lambda n)) / (nrm/(lambda n)),
//                    alpha' = y clip(y (alpha + Delta), 0, 1)
// Zero column: the exact 1-D minimiser (Lasso 0, SVM y) -- reading R5.
__device__ __forceinline__ double coord_step(int model, double alpha, double s, double nrm,
                                             double y, double lambda, double dd, double nn, double eta = 0.0) {
    if (model == kRidge) return (alpha * nrm - s) / (nrm + lambda * dd);  // P:808-813, eta = 1
    if (model == kElastic) {  // gamma and tau over ||a||^2 + lambda eta d
        const double den = nrm + lambda * eta * dd;
        const double gamma = (alpha * nrm - s) / den, tau = lambda * dd * (1.0 - eta) / den;
        const double mag = fabs(gamma) - tau;
        return mag > 0.0 ? copysign(mag, gamma) : 0.0;
    }
    if (model == kLasso) {
        if (nrm == 0.0) return 0.0;
        double gamma = (alpha * nrm - s) / nrm;
        double tau = lambda * dd / nrm;
        double mag = fabs(gamma) - tau;
        if (mag <= 0.0) return 0.0;
        return gamma > 0.0 ? mag : -mag;
    }
    if (nrm == 0.0) return y;
    double ln = lambda * nn;
    double delta = (y - s / ln) / (nrm / ln);
    double u = y * (alpha + delta);
    u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
    return y * u;
}

// Per-coordinate gap, Eq. 4 with the App. E closed forms; s = a_i^T w.
//   Lasso: (1/d)[alpha s + B max(|s| - lambda d, 0) + lambda d |alpha|]
//   Ridge: (1/d)[alpha s + s^2/(2 lambda d) + (lambda d/2) alpha^2]
//   SVM: (1/n)[alpha s + max(0, 1 - y s) - y alpha]
// Returns the raw gap; *scale receives the magnitude of its terms (for the
// negative-gap check, reading R17); *aux receives the conjugate / loss term
// used by the certificate: Lasso B max(|s|/d - lambda, 0), SVM max(0, 1 - y s).
__device__ __forceinline__ double coord_gap(int model, double alpha, double s, double y,
                                            double lambda, double B, double dd, double nn,
                                            double* scale, double* aux, double eta = 0.0) {
    if (model == kElastic) {  // Eq. 4 with the conjugate g*(x) = [|x| - lambda(1-eta)]_+^2/(2 lambda eta)
        const double x = fabs(s) / dd - lambda * (1.0 - eta);
        const double t1 = alpha * s / dd;
        const double t2 = lambda * (0.5 * eta * alpha * alpha + (1.0 - eta) * fabs(alpha));
        const double t3 = x > 0.0 ? x * x / (2.0 * lambda * eta) : 0.0;
        *scale = fabs(t1) + t2 + t3;
        *aux = t3;  // g*(a^T u), u = w/d: the dual's penalty term
        return t1 + t2 + t3;
    }
    if (model == kRidge) {  // P:841; aux = g*(-a^T u) = (s/d)^2/(2 lambda) for the dual
        const double lam_d = lambda * dd;
        const double t1 = alpha * s, t2 = s * s / (2.0 * lam_d), t3 = 0.5 * lam_d * alpha * alpha;
        *scale = (fabs(t1) + t2 + t3) / dd;
        const double x = s / dd;
        *aux = x * x / (2.0 * lambda);
        return (t1 + t2 + t3) / dd;
    }
    if (model == kLasso) {
        double lam_d = lambda * dd;
        double thr = fabs(s) - lam_d;
        double t1 = alpha * s, t2 = B * (thr > 0.0 ? thr : 0.0), t3 = lam_d * fabs(alpha);
        *scale = (fabs(t1) + t2 + t3) / dd;
        double x = fabs(s / dd) - lambda;
        *aux = B * (x > 0.0 ? x : 0.0);
        return (t1 + t2 + t3) / dd;
    }
    double h = 1.0 - y * s;
    double t1 = alpha * s, t2 = (h > 0.0 ? h : 0.0), t3 = y * alpha;
    *scale = (fabs(t1) + t2 + fabs(t3)) / nn;
    *aux = t2;
    return (t1 + t2 - t3) / nn;
}

// ---------------------------------------------------------------- packed fp32 (sm_100 FFMA2)
// c += a * b on two fp32 lanes with one instruction (fma.rn.f32x2).
__device__ __forceinline__ void ffma2(float2& c, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%0, %1};\n\t"
        "fma.rn.f32x2 rc, ra, rb, rc;\n\tmov.b64 {%0, %1}, rc;\n\t}"
        : "+f"(c.x), "+f"(c.y)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- memory model
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
#ifndef DUHL_STAGE_SLEEP_NS
#define DUHL_STAGE_SLEEP_NS 128
#endif
// staging counter c of the gather lives at progress[c * kProgressStride] (own 128-byte line:
// the polls of the SCD grid and the releases of the other gather CTAs do not share it)
constexpr int kProgressStride = 32;

// Wait until a staged column has landed in HBM (the SCD kernels' producer warps).
// need = 0: resident.  stage_ctas = 0: copy-engine staging, one monotone sequence
// counter progress[0] (need = the copy's sequence number; seen caches the last value
// read).  stage_ctas = G > 0: the gather kernel k_stage_gather, plan entry q = need - 1
// landed once progress[(q % G) * kProgressStride] > q / G; a token with the high bit set is a
// column the copy engine stages beside the gather (sequence number on progress[16 * stride]).  After the acquire, a proxy fence orders the
// generic-proxy stores of the gather before this thread's async-proxy (TMA) reads.
// Bounded: after timeout_ns the wait gives up and sets *err (bit 0).
__device__ __forceinline__ bool wait_staged(const unsigned* progress, int stage_ctas, unsigned need,
                                            unsigned& seen, int* err, unsigned long long timeout_ns) {
    if (!progress || need == 0) return true;
    const unsigned* c = progress;
    unsigned thr = need;
    if (stage_ctas > 0 && (need & 0x80000000u)) {  // a column the copy engine stages (sequence number)
        c = progress + (size_t)16 * kProgressStride;
        thr = need & 0x7fffffffu;
    } else if (stage_ctas > 0) {
        c = progress + (size_t)((need - 1) % (unsigned)stage_ctas) * kProgressStride;
        thr = (need - 1) / (unsigned)stage_ctas + 1;
    } else if (need <= seen) {
        return true;
    }
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned v;
    while ((v = ld_acquire_u32(c)) < thr) {
        __nanosleep(DUHL_STAGE_SLEEP_NS);
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > timeout_ns) { atomicOr(err, 1); return false; }
    }
    if (stage_ctas == 0) seen = v;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    return true;
}

__device__ __forceinline__ double ld_cg_f64(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {  // streamed once: no L1 allocate
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  `bar` is
// a monotone counter zeroed before the launch; generation g waits for
// (g+1)*nblocks arrivals.  __syncthreads + gpu-scope fence make every prior
// write of the CTA visible before the arrival (fence cumulativity).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) { __nanosleep(32); }
        __threadfence();
    }
    __syncthreads();
}

// ---------------------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release.cta
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: after `timeout_ns` sets bit `bit` of *err and returns (never hang the GPU).
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, unsigned parity, int* err, int bit,
                                                  unsigned long long timeout_ns) {
    if (mbar_try(bar, parity)) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (!mbar_try(bar, parity)) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) { atomicOr(err, bit); return; }
    }
}
// Named CTA barrier over `n` threads (multiple of 32).
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine), completion on mbarrier.
// bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

}  // namespace duhl
