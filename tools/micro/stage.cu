// Staging micro-benchmark (C4 columns, 803 KB): H2D throughput of per-column copies vs the
// number of streams (copy engines), a zero-copy gather kernel, and cudaHostRegister cost
// (one call vs chunked calls from several threads).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void gather(const float4* __restrict__ h, const int* cols, int ncol, size_t col4, float4* dv) {
    for (int c = blockIdx.y; c < ncol; c += gridDim.y) {
        const float4* src = h + (size_t)cols[c] * col4;
        float4* dst = dv + (size_t)c * col4;
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < col4; i += (size_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
    }
}

int main() {
    const size_t col = 200704 * 4;
    const int ncol = 2400, nsrc = 8000;
    char* dv; CK(cudaMalloc(&dv, col * ncol));
    char* h; CK(cudaHostAlloc(&h, col * nsrc, cudaHostAllocMapped));
    memset(h, 1, col * nsrc);
    std::vector<int> cols(ncol);
    for (int c = 0; c < ncol; ++c) cols[c] = (int)(((long)c * 7919) % nsrc);
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    for (int ns : {1, 2, 3, 4, 8}) {
        std::vector<cudaStream_t> s(ns);
        for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(a, s[0]));
            for (int k = 1; k < ns; ++k) CK(cudaStreamWaitEvent(s[k], a));
            for (int c = 0; c < ncol; ++c)
                CK(cudaMemcpyAsync(dv + c * col, h + (size_t)cols[c] * col, col, cudaMemcpyHostToDevice, s[c % ns]));
            for (int k = 1; k < ns; ++k) { cudaEvent_t ev; CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)); CK(cudaEventRecord(ev, s[k])); CK(cudaStreamWaitEvent(s[0], ev)); }
            CK(cudaEventRecord(b, s[0])); CK(cudaEventSynchronize(b));
            float ms; CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, (double)ncol * col / ms / 1e6);
        }
        printf("per-column copies, %d streams: %.1f GB/s\n", ns, best);
    }
    {   // one big copy: the PCIe ceiling
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a)); CK(cudaMemcpyAsync(dv, h, col * ncol, cudaMemcpyHostToDevice)); CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, (double)ncol * col / ms / 1e6);
        }
        printf("one %zu MB copy: %.1f GB/s\n", ncol * col >> 20, best);
    }
    int* dcols; CK(cudaMalloc(&dcols, ncol * sizeof(int)));
    CK(cudaMemcpy(dcols, cols.data(), ncol * sizeof(int), cudaMemcpyHostToDevice));
    float4* hal; CK(cudaHostGetDevicePointer((void**)&hal, h, 0));
    for (int gx : {1, 2, 4, 8}) for (int gy : {8, 16, 32, 64, 148}) {
        double best = 0;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(a));
            gather<<<dim3(gx, gy), 512>>>(hal, dcols, ncol, col / 16, (float4*)dv);
            CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
            float ms; CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, (double)ncol * col / ms / 1e6);
        }
        printf("zero-copy gather kernel grid (%d x %d) x 512: %.1f GB/s\n", gx, gy, best);
    }
    CK(cudaFreeHost(h));
    // cudaHostRegister cost: 32 GB malloc'ed (touched), one call vs chunked from T threads
    const size_t big = (size_t)32 << 30;
    char* m = (char*)aligned_alloc(4096, big);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < 16; ++t) th.emplace_back([=] { memset(m + big / 16 * t, 1, big / 16); });
        for (auto& x : th) x.join();
    }
    for (int T : {1, 4, 8, 16}) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        std::vector<cudaError_t> err(T);
        for (int t = 0; t < T; ++t)
            th.emplace_back([=, &err] { err[t] = cudaHostRegister(m + big / T * t, big / T, cudaHostRegisterMapped | cudaHostRegisterReadOnly); });
        for (auto& x : th) x.join();
        double reg = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto e : err) if (e != cudaSuccess) printf("register error %s\n", cudaGetErrorString(e));
        void* dp = nullptr;
        cudaHostGetDevicePointer(&dp, m, 0);
        int same = dp == (void*)m;
        t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < T; ++t) CK(cudaHostUnregister(m + big / T * t));
        double unreg = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("cudaHostRegister 32 GB in %d chunk(s)/threads: %.2f s (unregister %.2f s), device ptr == host ptr: %d\n", T, reg, unreg, same);
    }
    int attr = 0; cudaDeviceGetAttribute(&attr, cudaDevAttrCanUseHostPointerForRegisteredMem, 0);
    printf("CanUseHostPointerForRegisteredMem = %d\n", attr);
    return 0;
}
