// scd_tpa.cu -- asynchronous (TPA-SCD style) SCD epoch on a dense working set, sm_100a.
//
// The paper's own GPU design (TPA-SCD; App. D, "the shared vector ... is
// updated atomically"): many coordinates are processed concurrently, each reads the shared
// vector as it is (stale by the updates in flight), takes the closed-form step (P:804-815
// Lasso / ridge / elastic net, P:824-827 SVM) and adds delta_j a_j to the shared vector with
// atomics.  B200 form ("TPA-style bounded-W async"):
//   * W = number of thread-block clusters = coordinates in flight (the staleness bound); a
//     cluster of C CTAs splits one coordinate's column by rows (C chosen so a CTA's slice of
//     the column fits in shared memory: C4's 803-KB columns take C = 4..8), so all SMs stream
//     while only W coordinates are concurrent;
//   * per coordinate: each CTA's slice of a_j arrives in shared memory by one TMA bulk copy,
//     double-buffered (the next coordinate's slice streams in while this one is reduced and
//     REDed); the CTA accumulates its part of a_j^T v~ in fp64; the C partial dots meet in the
//     leader's shared memory
//     (distributed shared memory) behind one cluster barrier; every CTA then takes the same
//     closed-form step and adds delta_j a_j to its rows of v~f with red.global.add.v4.f32
//     (one 16-byte RED per 4 rows; App. D's atomic update);
//   * the shared vector during the epoch is v~0 + dvf: v~0 = the exact fp64 vector at epoch
//     start, dvf = an fp32 shadow of the epoch's own updates (zero at start, REDed).
//     s_j = a_j^T v~0 + a_j^T dvf: the first term for every j in P by one gap pass before the
//     epoch (fp64, u0), the second in fp64 accumulation here: the fp32 rounding touches only
//     the epoch's change, which vanishes near the optimum (an fp32 copy of v~ itself held
//     C3's Lasso above 1e-5: its gap is sensitive to s through B = ||b||^2/(2 lambda d));
//   * the epoch ends with the exact resync v~ = v~0 + A_P (alpha_P - alpha_P0) in fp64
//     (k_tpa_resync, SURVEY 8 a6 "Delta v exact"), so the state the gaps and certificates use
//     is exact to rounding whatever the interleaving was.
// Pinned by P7s/P8s (disjoint-support orthogonal designs: any interleaving is the sequential
// epoch) and by convergence to the oracle's optimum (tests/test_gpu_tpa.py).
#include <cooperative_groups.h>

#include "device.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace duhl {

constexpr int kTpaThreads = 512;
constexpr int kTpaMaxCluster = 8;

__device__ __forceinline__ void red_add_v4_f32(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__global__ void __launch_bounds__(kTpaThreads, 1) k_scd_tpa(const __grid_constant__ TpaParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* bufs = reinterpret_cast<float*>(smem);   // [2][Rc]: this CTA's slices of two coordinates
    __shared__ __align__(8) uint64_t mbar[2];        // slice landed (TMA bulk copy, tx bytes)
    __shared__ double part[2][kTpaMaxCluster];      // partial dots (read through the leader's copy)
    __shared__ double wsum[kTpaThreads / 32];
    __shared__ double s_delta;
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t cid = blockIdx.x / C, ncl = gridDim.x / C;
    const int64_t r0 = (int64_t)rank * p.Rc;
    const int64_t rows = r0 < p.d4 ? (p.d4 - r0 < p.Rc ? p.d4 - r0 : p.Rc) : 0;  // multiple of 4
    const int n4 = (int)(rows >> 2);
    double* lead = cl.map_shared_rank(&part[0][0], 0);
    const double dd = (double)p.d, nn = (double)p.n;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // the TMA engine streams the next coordinate's slice into the other buffer while this one's
    // dot, cluster reduction and REDs run (one thread issues one bulk copy of rows x 4 bytes)
    auto issue = [&](int64_t it) {
        const int64_t t = cid + it * ncl;
        if (t >= p.L || n4 == 0) return;
        const int b = (int)(it & 1);
        fence_proxy_async();  // the buffer's last generic reads (two iterations ago) before the async write
        mbar_arrive_expect_tx(&mbar[b], (unsigned)rows * 4u);
        bulk_g2s(bufs + (size_t)b * p.Rc, p.pool + (int64_t)p.order_slot[t] * p.ld_dev + r0, (unsigned)rows * 4u,
                 &mbar[b]);
    };
    if (tid == 0) issue(0);
    int it = 0;
    for (int64_t t = cid; t < p.L; t += ncl, ++it) {
        const int64_t j = p.order_j[t];
        if (tid == 0) issue(it + 1);  // its buffer was released by the __syncthreads closing it - 1
        const int b = it & 1;
        if (n4 > 0) mbar_wait(&mbar[b], (unsigned)((it >> 1) & 1));
        const float4* col = reinterpret_cast<const float4*>(bufs + (size_t)b * p.Rc);
        const float4* vf4 = reinterpret_cast<const float4*>(p.vf + r0);
        // a_j^T v~0 was taken for every j in P before the epoch (p.u0): only the epoch's own
        // updates dvf are read here (4 bytes per row from L2, not 12)
        double acc0 = 0.0, acc1 = 0.0;
        for (int q = tid; q < n4; q += kTpaThreads) {
            const float4 a = col[q];
            const float4 dv = __ldcg(vf4 + q);  // dvf is being updated by the other clusters: read at L2
            acc0 = fma((double)a.x, (double)dv.x, acc0);
            acc1 = fma((double)a.y, (double)dv.y, acc1);
            acc0 = fma((double)a.z, (double)dv.z, acc0);
            acc1 = fma((double)a.w, (double)dv.w, acc1);
        }
        double s = warp_sum(acc0 + acc1);
        if (lane == 0) wsum[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < kTpaThreads / 32; ++w) tot += wsum[w];
            lead[(it & 1) * kTpaMaxCluster + rank] = tot;  // distributed shared memory store
        }
        cl.sync();  // all C partials of coordinate t are in the leader's part[it & 1]
        if (tid == 0) {
            double sj = p.u0[j];
            for (int r = 0; r < C; ++r) sj += lead[(it & 1) * kTpaMaxCluster + r];  // rank order: same on every CTA
            const double a_old = p.order_a[t];
            const double an = coord_step(p.model, a_old, sj, p.norms[j], p.y ? p.y[j] : 0.0, p.lambda, dd, nn, p.eta);
            s_delta = an - a_old;
            if (rank == 0) p.alpha[j] = an;
        }
        __syncthreads();
        const float dl = (float)s_delta;
        if (s_delta != 0.0) {
            float* vrow = p.vf + r0;
            for (int q = tid; q < n4; q += kTpaThreads) {
                const float4 a = col[q];
                red_add_v4_f32(vrow + 4 * q, dl * a.x, dl * a.y, dl * a.z, dl * a.w);
            }
        }
        __syncthreads();  // the slice buffer is refilled two coordinates later
    }
    cl.sync();  // no CTA leaves while another may still read the leader's partials
}

// v~ += A_P (alpha_P - alpha_P0), fp64 (the exact resync after an asynchronous epoch; v~ was
// reset to v~0 first).  Grid (row groups, column chunks): CTA (x, y) takes 512 rows (one 4-row
// group per thread) and kResyncChunk columns of P, accumulates in fp64 and adds its partial with
// fp64 atomics -- enough CTAs to stream A_P at HBM rate (one CTA per 512 rows alone left C3's 40k
// rows on 79 SMs).
constexpr int kResyncThreads = 128;
constexpr int kResyncChunk = 512;
__global__ void __launch_bounds__(kResyncThreads) k_tpa_resync(const float* pool, int64_t ld_dev, const int* P_slot,
                                                               const int64_t* P, const double* alpha,
                                                               const double* a0, int64_t m, double* vt, int64_t d4) {
    __shared__ double sda[kResyncChunk];
    __shared__ int sslot[kResyncChunk];
    const int64_t r4 = (int64_t)blockIdx.x * kResyncThreads + threadIdx.x;
    const int64_t q0 = (int64_t)blockIdx.y * kResyncChunk;
    const int nq = (int)(m - q0 < kResyncChunk ? m - q0 : kResyncChunk);
    int nz = 0;
    for (int q = threadIdx.x; q < nq; q += kResyncThreads) {
        sda[q] = alpha[P[q0 + q]] - a0[q0 + q];
        sslot[q] = P_slot[q0 + q];
    }
    __syncthreads();
    if (4 * r4 >= d4) return;
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
    for (int q = 0; q < nq; ++q) {
        const double da = sda[q];
        if (da == 0.0) continue;
        ++nz;
        const float4 a = ld_stream_f4(reinterpret_cast<const float4*>(pool + (int64_t)sslot[q] * ld_dev) + r4);
        x0 = fma(da, (double)a.x, x0);
        x1 = fma(da, (double)a.y, x1);
        x2 = fma(da, (double)a.z, x2);
        x3 = fma(da, (double)a.w, x3);
    }
    if (nz == 0) return;
    const int64_t r = 4 * r4;
    atomicAdd(vt + r, x0);
    atomicAdd(vt + r + 1, x1);
    atomicAdd(vt + r + 2, x2);
    atomicAdd(vt + r + 3, x3);
}

// u0[P[q]] = s[q] * scale (a_j^T v~0 of the working set, from a gap pass's s_out)
__global__ void k_scatter_scaled(const double* s, const int64_t* P, int64_t m, double scale, double* u0) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < m) u0[P[q]] = s[q] * scale;
}
cudaError_t launch_scatter_scaled(const double* s, const int64_t* P, int64_t m, double scale, double* u0,
                                  cudaStream_t st, int64_t* launches) {
    if (m <= 0) return cudaSuccess;
    k_scatter_scaled<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(s, P, m, scale, u0);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_f64_to_f32(const double* x, float* y, int64_t k) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) y[i] = (float)x[i];
}

size_t tpa_smem_bytes(int64_t Rc, bool v0_smem) { (void)v0_smem; return (size_t)Rc * 8; }  // 2 slices

cudaError_t launch_scd_tpa(const TpaParams& p, int W, cudaStream_t st, int64_t* launches) {
    if (p.L <= 0) return cudaSuccess;
    const size_t smem = tpa_smem_bytes(p.Rc, p.v0_smem != 0);
    cudaError_t e = cudaFuncSetAttribute(k_scd_tpa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (p.C > 8) {
        e = cudaFuncSetAttribute(k_scd_tpa, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(W * p.C));
    cfg.blockDim = dim3(kTpaThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_scd_tpa, p);
    ++*launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_tpa_resync(const float* pool, int64_t ld_dev, const int* P_slot, const int64_t* P,
                              const double* alpha, const double* a0, int64_t m, const double* v0, double* vt,
                              int64_t d4, cudaStream_t st, int64_t* launches) {
    cudaError_t e = cudaMemcpyAsync(vt, v0, d4 * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess || m <= 0) return e;
    const int64_t n4 = d4 / 4;
    const dim3 grid((unsigned)((n4 + kResyncThreads - 1) / kResyncThreads), (unsigned)((m + kResyncChunk - 1) / kResyncChunk));
    k_tpa_resync<<<grid, kResyncThreads, 0, st>>>(pool, ld_dev, P_slot, P, alpha, a0, m, vt, d4);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* x, float* y, int64_t k, cudaStream_t st, int64_t* launches) {
    k_f64_to_f32<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(x, y, k);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t preload_tpa_kernels() {
    const void* fns[] = {(const void*)k_scd_tpa, (const void*)k_tpa_resync, (const void*)k_f64_to_f32,
                         (const void*)k_scatter_scaled};
    for (const void* f : fns) {
        cudaFuncAttributes a;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace duhl
