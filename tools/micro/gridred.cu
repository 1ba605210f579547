// Microbenchmark: per-iteration cost of a 148-CTA fp64 reduction + grid barrier + read-back,
// the synchronisation step of k_scd_gram.  mode 0: full; 1: barrier only; 2: RED + barrier;
// 3: barrier + read.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ double ld_cg(const double* p) {
    double v; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v;
}
__global__ void k(double* red, unsigned* bar, int nred, int groups, int iters, int mode, double* sink) {
    __shared__ double sg[1024];
    const int tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        double* rb = red + (size_t)(it % 6) * nred * groups * 32;
        if (mode == 0 || mode == 2 || mode == 4 || mode == 5)
            for (int q = tid; q < nred; q += blockDim.x) atomicAdd(&rb[((size_t)q * groups + c % groups) * 32], 1.0);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(&bar[it & 1], 1u);
            unsigned target = (unsigned)((it / 2 + 1) * G);
            while (ld_acq(&bar[it & 1]) < target) __nanosleep(32);
            __threadfence();
        }
        __syncthreads();
        if (mode == 4) {  // whole CTA reads, one entry per thread
            for (int q = tid; q < nred; q += blockDim.x) {
                double v = 0;
                for (int g = 0; g < groups; ++g) v += ld_cg(&rb[((size_t)q * groups + g) * 32]);
                sg[q] = v;
            }
        }
        if (mode == 5 && tid < 32) {  // one warp, all loads first (padded, unconditional)
            double v[8][2];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    int q = u * 32 + tid; if (q >= nred) q = nred - 1;
                    v[u][g] = g < groups ? ld_cg(&rb[((size_t)q * groups + (g < groups ? g : 0)) * 32]) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < 8; ++u) { int q = u * 32 + tid; if (q < nred) sg[q] = v[u][0] + v[u][1]; }
        }
        if (mode == 0 || mode == 3)
            if (tid < 32)
                for (int q = tid; q < nred; q += 32) {
                    double v = 0;
                    for (int g = 0; g < groups; ++g) v += ld_cg(&rb[((size_t)q * groups + g) * 32]);
                    sg[q] = v;
                }
        __syncthreads();
        acc += sg[tid % nred];
    }
    sink[c * blockDim.x + tid] = acc;
}
int main() {
    const int G = 148, T = 256, iters = 2000;
    double *red, *sink; unsigned* bar;
    cudaMalloc(&red, 6ull * 1024 * 8 * 32 * 8); cudaMalloc(&sink, G * T * 8); cudaMalloc(&bar, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode : {0, 4, 5})
        for (int nred : {100, 222}) for (int groups : {1, 2}) {
            cudaMemset(bar, 0, 64);
            int it = iters, md = mode, nr = nred, gr = groups;
            void* args[] = {&red, &bar, &nr, &gr, &it, &md, &sink};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k, G, T, args, 0, 0);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("mode %d nred %3d groups %d: %.2f us/iter  %s\n", mode, nred, groups, 1e3 * ms / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
