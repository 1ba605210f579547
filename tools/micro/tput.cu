// Microbenchmark: per-SM throughput of F2F.F64.F32 (float -> double), DFMA, FFMA2 and the
// integer-ALU float->double bit conversion, 8 warps per SM, independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void k(const float* in, double* out, long long* cyc, int iters) {
    float f[8];
    double d[8];
    for (int q = 0; q < 8; ++q) { f[q] = in[threadIdx.x + q]; d[q] = 0.0; }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (K == 0) d[q] += (double)f[q];                       // F2F + DADD
            if (K == 1) d[q] = fma(d[q], 1.0000001, 1e-9);          // DFMA
            if (K == 2) { f[q] = fmaf(f[q], 1.0000001f, 1e-7f); }   // FFMA
            if (K == 3) {                                           // ALU conversion + DADD
                unsigned b = __float_as_uint(f[q]);
                unsigned hi = (b & 0x80000000u) | (((b >> 3) & 0x0FFFFFFFu) + 0x38000000u);
                unsigned lo = b << 29;
                d[q] += __hiloint2double((int)((b & 0x7FFFFFFFu) ? hi : (b & 0x80000000u)), (int)lo);
            }
            if (K == 4) d[q] += 1e-9;                               // DADD only
        }
        if (K != 2) f[0] += 1e-7f;
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int q = 0; q < 8; ++q) s += d[q] + f[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* in; double* out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    const char* nm[5] = {"F2F.F64.F32+DADD", "DFMA", "FFMA", "ALU f32->f64 + DADD", "DADD"};
    for (int kk = 0; kk < 5; ++kk) {
        for (int rep = 0; rep < 2; ++rep) {
            if (kk == 0) k<0><<<148, 256>>>(in, out, cyc, iters);
            if (kk == 1) k<1><<<148, 256>>>(in, out, cyc, iters);
            if (kk == 2) k<2><<<148, 256>>>(in, out, cyc, iters);
            if (kk == 3) k<3><<<148, 256>>>(in, out, cyc, iters);
            if (kk == 4) k<4><<<148, 256>>>(in, out, cyc, iters);
        }
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = 256.0 * iters * 8;  // per SM
        printf("%-22s %.2f results/clk/SM\n", nm[kk], ops / c);
    }
    return 0;
}
