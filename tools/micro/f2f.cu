// Throughput of fp32 -> fp64 conversion on sm_100a: F2F.F64.F32 vs an integer bit
// construction, and DFMA, per SM per clock (one CTA per SM, 8 independent chains per thread).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double cvt_int(float x) {
    const unsigned u = __float_as_uint(x);
    const unsigned t = (u << 1) >> 4;                 // exponent + mantissa >> 3, sign dropped
    const unsigned hi = (t + 0x38000000u) | (u & 0x80000000u);
    const unsigned lo = u << 29;
    return __hiloint2double((int)hi, (int)lo);
}

template <int MODE>
__global__ void k(const float* in, double* out, int iters) {
    float x[8];
    double acc[8];
    for (int i = 0; i < 8; ++i) { x[i] = in[(threadIdx.x + i) & 255]; acc[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) acc[i] += (double)x[i];                          // F2F + DADD
            else if (MODE == 1) acc[i] += cvt_int(x[i]);                    // int cvt + DADD
            else if (MODE == 2) acc[i] = fma(acc[i], 1.0000001, (double)i);  // DFMA only
            else acc[i] += (i & 1) ? cvt_int(x[i]) : (double)x[i];          // half / half
            x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);                // keep the input live
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* in; double* out;
    cudaMalloc(&in, 256 * 4); cudaMalloc(&out, 148 * 1024 * 8);
    float h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0f + i * 0.37f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* nm[4] = {"F2F+DADD", "intcvt+DADD", "DFMA", "half/half+DADD"};
    for (int mode = 0; mode < 4; ++mode)
        for (int thr : {256, 512, 1024}) {
            const int iters = 4096;
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) k<0><<<148, thr>>>(in, out, iters);
                if (mode == 1) k<1><<<148, thr>>>(in, out, iters);
                if (mode == 2) k<2><<<148, thr>>>(in, out, iters);
                if (mode == 3) k<3><<<148, thr>>>(in, out, iters);
                cudaEventRecord(b); cudaEventSynchronize(b);
            }
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = 148.0 * thr * iters * 8;
            printf("%-16s thr %4d: %.1f ops/clk/SM (at %d MHz)\n", nm[mode], thr, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
        }
    return 0;
}
