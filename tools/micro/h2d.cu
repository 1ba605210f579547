// H2D copy throughput: registered malloc vs cudaHostAlloc; one big copy vs many column copies.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
static double run(const char* what, char* h, char* dv, size_t col, int ncol, int chunk, int nstreams, bool scatter) {
    std::vector<cudaStream_t> s(nstreams);
    for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, s[0]));
        for (int k = 1; k < nstreams; ++k) CK(cudaStreamWaitEvent(s[k], a));
        for (int c = 0, q = 0; c < ncol; c += chunk, ++q) {
            int nc = c + chunk <= ncol ? chunk : ncol - c;
            size_t src = scatter ? ((size_t)(c * 7919) % (size_t)ncol) : (size_t)c;
            if (scatter && src + nc > (size_t)ncol) src = 0;
            CK(cudaMemcpyAsync(dv + c * col, h + src * col, nc * col, cudaMemcpyHostToDevice, s[q % nstreams]));
        }
        for (int k = 1; k < nstreams; ++k) { cudaEvent_t ev; CK(cudaEventCreate(&ev)); CK(cudaEventRecord(ev, s[k])); CK(cudaStreamWaitEvent(s[0], ev)); }
        CK(cudaEventRecord(b, s[0])); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        double gbs = (double)ncol * col / ms / 1e6;
        if (gbs > best) best = gbs;
    }
    printf("%-28s chunk %4d cols, %d streams: %.1f GB/s\n", what, chunk, nstreams, best);
    return best;
}
__global__ void zc_read(const float4* __restrict__ h, size_t n4, float* out) {
    float acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        float4 a = h[i], b = h[i + stride], c = h[i + 2 * stride], d = h[i + 3 * stride];
        acc += a.x + b.y + c.z + d.w;
    }
    for (; i < n4; i += stride) acc += h[i].x;
    if (acc == 12345.f) *out = acc;
}
// concurrent: stream 0 = 1-column copies of cols [0,nc); stream 1 = big copy or zero-copy kernel over other bytes
static void concurrent(const char* what, char* h, char* dv, size_t col, int nc, char* h2, char* dv2, size_t bytes2, int mode, int ctas = 148 * 4) {
    cudaStream_t s0, s1; CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t a, b, e0, e1; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float* out; CK(cudaMalloc(&out, 4));
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, s0)); CK(cudaStreamWaitEvent(s1, a));
        if (mode == 0) CK(cudaMemcpyAsync(dv2, h2, bytes2, cudaMemcpyHostToDevice, s1));
        else if (mode == 1) zc_read<<<ctas, 256, 0, s1>>>((const float4*)h2, bytes2 / 16, out);
        CK(cudaEventRecord(e1, s1));
        for (int c = 0; c < nc; ++c) CK(cudaMemcpyAsync(dv + c * col, h + (size_t)((c * 7919) % nc) * col, col, cudaMemcpyHostToDevice, s0));
        CK(cudaEventRecord(e0, s0));
        CK(cudaStreamWaitEvent(s0, e1)); CK(cudaEventRecord(b, s0)); CK(cudaEventSynchronize(b));
        float ms, ms0, ms1; CK(cudaEventElapsedTime(&ms, a, b)); CK(cudaEventElapsedTime(&ms0, a, e0)); CK(cudaEventElapsedTime(&ms1, a, e1));
        if (rep) printf("%-34s total %.1f GB/s (%.1f ms); cols done at %.1f ms, other at %.1f ms\n", what,
                        ((double)nc * col + (mode >= 0 ? bytes2 : 0)) / ms / 1e6, ms, ms0, ms1);
    }
}
int main() {
    const size_t col = 200704 * 4;  // C4 column
    const int ncol = 3000;
    const size_t bytes = col * ncol;
    char* dv; CK(cudaMalloc(&dv, bytes));
    char* hr = (char*)aligned_alloc(4096, bytes); memset(hr, 1, bytes);
    CK(cudaHostRegister(hr, bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly));
    char* ha; CK(cudaHostAlloc(&ha, bytes, cudaHostAllocMapped)); memset(ha, 1, bytes);
    for (int w = 0; w < 2; ++w) {
        char* h = w ? ha : hr;
        const char* nm = w ? "cudaHostAlloc" : "registered malloc";
        run(nm, h, dv, col, ncol, ncol, 1, false);
        run(nm, h, dv, col, ncol, 1, 1, false);
        run(nm, h, dv, col, ncol, 1, 2, false);
        run(nm, h, dv, col, ncol, 4, 1, false);
        run(nm, h, dv, col, ncol, 1, 1, true);
    }
    // madvise hugepages variant
    char* hh = (char*)aligned_alloc(1 << 21, bytes);
    madvise(hh, bytes, 14 /*MADV_HUGEPAGE*/);
    memset(hh, 1, bytes);
    CK(cudaHostRegister(hh, bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly));
    run("registered THP", hh, dv, col, ncol, ncol, 1, false);
    run("registered THP", hh, dv, col, ncol, 1, 1, false);
    // zero-copy alone
    {
        float* out; CK(cudaMalloc(&out, 4)); cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
        for (int g = 1; g <= 8; g *= 2) {
            zc_read<<<148 * g, 256>>>((const float4*)ha, bytes / 16, out);
            CK(cudaEventRecord(a)); zc_read<<<148 * g, 256>>>((const float4*)ha, bytes / 16, out); CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b));
            printf("zero-copy read alone, %d CTAs/SM: %.1f GB/s\n", g, bytes / ms / 1e6);
        }
    }
    size_t half = bytes / 2;
    concurrent("1-col copies + big DMA", ha, dv, col, 1500, ha + half, dv + half, half, 0);
    concurrent("1-col copies + zero-copy kernel", ha, dv, col, 1500, ha + half, dv + half, half, 1);
    for (int g : {8, 16, 32, 64, 148}) {
        char nm[64]; snprintf(nm, 64, "1-col + zero-copy %d CTAs", g);
        concurrent(nm, ha, dv, col, 1500, ha + half, dv + half, half / 4, 1, g);
    }
    concurrent("1-col copies alone", ha, dv, col, 1500, ha + half, dv + half, 0, -1);
    return 0;
}
