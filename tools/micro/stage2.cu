// Gather (zero-copy) and per-column copy-engine staging from three kinds of pinned host memory:
// cudaHostAlloc, malloc + cudaHostRegister (4 KB pages), THP malloc + cudaHostRegister.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__global__ void gather(const float4* __restrict__ h, const int* cols, int ncol, size_t col4, float4* dv) {
    for (int c = blockIdx.x; c < ncol; c += gridDim.x) {
        const float4* src = h + (size_t)cols[c] * col4;
        float4* dst = dv + (size_t)c * col4;
        size_t i = threadIdx.x;
        for (; i + 7 * 256 < col4; i += 8 * 256) {
            float4 x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = src[i + u * 256];
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[i + u * 256] = x[u];
        }
        for (; i < col4; i += 256) dst[i] = src[i];
    }
}
int main() {
    const size_t col = 200704 * 4;
    const int ncol = 2400;
    const int nsrc = getenv("NSRC") ? atoi(getenv("NSRC")) : 12000;
    const size_t bytes = col * nsrc;
    char* dv; CK(cudaMalloc(&dv, col * ncol));
    std::vector<int> cols(ncol);
    for (int c = 0; c < ncol; ++c) cols[c] = (int)(((long)c * 7919) % nsrc);
    int* dcols; CK(cudaMalloc(&dcols, ncol * sizeof(int)));
    CK(cudaMemcpy(dcols, cols.data(), ncol * sizeof(int), cudaMemcpyHostToDevice));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    for (int kind = 0; kind < 3; ++kind) {
        char* h = nullptr;
        const char* nm[3] = {"cudaHostAlloc", "malloc+register (4K)", "THP malloc+register"};
        if (kind == 0) CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
        else {
            h = (char*)aligned_alloc(1 << 21, bytes);
            if (kind == 2) madvise(h, bytes, MADV_HUGEPAGE);
            else madvise(h, bytes, MADV_NOHUGEPAGE);
        }
        memset(h, 1, bytes);
        if (kind) CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
        for (int g : {16, 32, 64}) {
            double best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaEventRecord(a));
                gather<<<g, 256>>>((const float4*)h, dcols, ncol, col / 16, (float4*)dv);
                CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
                float ms; CK(cudaEventElapsedTime(&ms, a, b));
                best = std::max(best, (double)ncol * col / ms / 1e6);
            }
            printf("%-24s gather %d CTAs x 256: %.1f GB/s\n", nm[kind], g, best);
        }
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a));
            for (int c = 0; c < ncol; ++c) CK(cudaMemcpyAsync(dv + c * col, h + (size_t)cols[c] * col, col, cudaMemcpyHostToDevice));
            CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
            float ms; CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, (double)ncol * col / ms / 1e6);
        }
        printf("%-24s per-column copies: %.1f GB/s\n", nm[kind], best);
        if (kind == 0) CK(cudaFreeHost(h)); else { CK(cudaHostUnregister(h)); free(h); }
    }
    return 0;
}
