// Host DRAM bandwidth on the GPU box: multi-threaded read (dot) and gather-memcpy of 800 KB columns.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t col = 200704 * 4, ncol = 4000, bytes = col * ncol;
    float* A = (float*)aligned_alloc(4096, bytes);
    char* B = (char*)aligned_alloc(4096, bytes / 2);
    memset(A, 0, bytes); memset(B, 0, bytes / 2);
    std::vector<float> w(200704, 1.0f);
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    for (int T : {1, 2, 4, 8, 16}) {
        double best = 0, bestc = 0;
        for (int rep = 0; rep < 3; ++rep) {
            std::vector<double> acc(T);
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
                double s = 0;
                for (size_t c = t; c < ncol; c += T) {
                    const float* a = A + c * 200704;
                    float p0 = 0, p1 = 0, p2 = 0, p3 = 0, p4 = 0, p5 = 0, p6 = 0, p7 = 0;
                    for (size_t r = 0; r < 200704; r += 8) {
                        p0 += a[r] * w[r]; p1 += a[r + 1] * w[r + 1]; p2 += a[r + 2] * w[r + 2]; p3 += a[r + 3] * w[r + 3];
                        p4 += a[r + 4] * w[r + 4]; p5 += a[r + 5] * w[r + 5]; p6 += a[r + 6] * w[r + 6]; p7 += a[r + 7] * w[r + 7];
                    }
                    s += p0 + p1 + p2 + p3 + p4 + p5 + p6 + p7;
                }
                acc[t] = s;
            });
            for (auto& x : th) x.join();
            double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = std::max(best, bytes / dt / 1e9);
            th.clear();
            t0 = std::chrono::steady_clock::now();
            for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
                for (size_t c = t; c < ncol / 2; c += T) memcpy(B + c * col, (char*)A + ((c * 7919) % ncol) * col, col);
            });
            for (auto& x : th) x.join();
            dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            bestc = std::max(bestc, bytes / 2 / dt / 1e9);
        }
        printf("threads %2d: dot read %.1f GB/s, gather memcpy %.1f GB/s (bytes copied)\n", T, best, bestc);
    }
}
