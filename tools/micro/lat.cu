// Microbenchmark: dependent-chain latencies (DFMA, DADD, FFMA, SHFL.f64, DMNMX, fp64 select) on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, long long* cyc, double x0, int iters) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    float f = (float)x0, g = 1.0000001f;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-12);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = x + 1e-13;
    t1 = clock64(); cyc[1] = t1 - t0;
    // FFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) f = fmaf(f, g, 1e-7f);
    t1 = clock64(); cyc[2] = t1 - t0;
    // SHFL f64 chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(~0u, x, (threadIdx.x + 1) & 31) + 1e-14;
    t1 = clock64(); cyc[3] = t1 - t0;
    // fmin/fmax (clamp) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fmin(fmax(x, 0.25), 0.75) + 1e-14;
    t1 = clock64(); cyc[4] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = x * y;
    t1 = clock64(); cyc[5] = t1 - t0;
    out[threadIdx.x] = x; outf[threadIdx.x] = f;
}
int main() {
    double* o; float* of; long long* c;
    cudaMalloc(&o, 32 * 8); cudaMalloc(&of, 32 * 4); cudaMallocManaged(&c, 8 * 8);
    const int iters = 4096;
    k<<<1, 32>>>(o, of, c, 1.0, iters);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(o, of, c, 1.0, iters);
    cudaDeviceSynchronize();
    const char* nm[6] = {"DFMA", "DADD", "FFMA", "SHFL.f64+DADD", "fmin(fmax)+DADD", "DMUL"};
    for (int i = 0; i < 6; ++i) printf("%-18s %.1f cycles/iter\n", nm[i], (double)c[i] / iters);
    return 0;
}
