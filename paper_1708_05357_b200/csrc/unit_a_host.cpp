// Host-thread share of the unit-A refresh: see unit_a_host.h.
#include "unit_a_host.h"

#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

namespace {

// a^T v over n elements, fp32 data widened to fp64 (exact), fp64 FMAs in 4 chains.
__attribute__((target("avx2,fma"))) double dot_avx2(const float* a, const double* v, int64_t n) {
    __m256d s0 = _mm256_setzero_pd(), s1 = _mm256_setzero_pd(), s2 = _mm256_setzero_pd(),
            s3 = _mm256_setzero_pd();
    int64_t i = 0;
    for (; i + 16 <= n; i += 16) {
        const __m256 f0 = _mm256_loadu_ps(a + i), f1 = _mm256_loadu_ps(a + i + 8);
        s0 = _mm256_fmadd_pd(_mm256_cvtps_pd(_mm256_castps256_ps128(f0)), _mm256_loadu_pd(v + i), s0);
        s1 = _mm256_fmadd_pd(_mm256_cvtps_pd(_mm256_extractf128_ps(f0, 1)), _mm256_loadu_pd(v + i + 4), s1);
        s2 = _mm256_fmadd_pd(_mm256_cvtps_pd(_mm256_castps256_ps128(f1)), _mm256_loadu_pd(v + i + 8), s2);
        s3 = _mm256_fmadd_pd(_mm256_cvtps_pd(_mm256_extractf128_ps(f1, 1)), _mm256_loadu_pd(v + i + 12), s3);
    }
    __m256d s = _mm256_add_pd(_mm256_add_pd(s0, s1), _mm256_add_pd(s2, s3));
    alignas(32) double l[4];
    _mm256_store_pd(l, s);
    double r = (l[0] + l[1]) + (l[2] + l[3]);
    for (; i < n; ++i) r += (double)a[i] * v[i];
    return r;
}

double dot_scalar(const float* a, const double* v, int64_t n) {
    double r0 = 0, r1 = 0;
    int64_t i = 0;
    for (; i + 2 <= n; i += 2) {
        r0 += (double)a[i] * v[i];
        r1 += (double)a[i + 1] * v[i + 1];
    }
    for (; i < n; ++i) r0 += (double)a[i] * v[i];
    return r0 + r1;
}

}  // namespace

struct HostUnitA {
    int dev = 0;
    bool avx2 = false;
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv_job, cv_done;
    uint64_t gen = 0;  // job generation; workers run each generation once
    bool stop = false;
    int active = 0;    // workers still on the current job
    // job
    const float* store = nullptr;
    int64_t ld = 0, d4 = 0, k = 0;
    const int64_t* cols = nullptr;
    const double* vt = nullptr;
    double scale = 1.0;
    cudaEvent_t ready = nullptr;
    double* s_out = nullptr;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> t_ready_ns{0};
    std::chrono::steady_clock::time_point t_end;
    bool posted = false;

    void run_worker() {
        cudaSetDevice(dev);
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_job.wait(lk, [&] { return stop || gen != seen; });
                if (stop) return;
                seen = gen;
            }
            cudaEventSynchronize(ready);
            int64_t expect = 0;
            const int64_t now = std::chrono::steady_clock::now().time_since_epoch().count();
            t_ready_ns.compare_exchange_strong(expect, now);
            for (;;) {
                const int64_t t = next.fetch_add(1, std::memory_order_relaxed);
                if (t >= k) break;
                const float* a = store + cols[t] * ld;
                s_out[t] = scale * (avx2 ? dot_avx2(a, vt, d4) : dot_scalar(a, vt, d4));
            }
            std::lock_guard<std::mutex> lk(mu);
            if (--active == 0) {
                t_end = std::chrono::steady_clock::now();
                cv_done.notify_all();
            }
        }
    }
};

HostUnitA* hua_create(int threads, int dev) {
    if (threads < 1) return nullptr;
    HostUnitA* h = new HostUnitA();
    h->dev = dev;
    __builtin_cpu_init();
    h->avx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
    for (int i = 0; i < threads; ++i) h->workers.emplace_back([h] { h->run_worker(); });
    return h;
}

void hua_destroy(HostUnitA* h) {
    if (!h) return;
    hua_wait(h);
    {
        std::lock_guard<std::mutex> lk(h->mu);
        h->stop = true;
    }
    h->cv_job.notify_all();
    for (auto& w : h->workers) w.join();
    delete h;
}

void hua_post(HostUnitA* h, const float* store, int64_t ld, int64_t d4, const int64_t* cols, int64_t k,
              const double* vt, double scale, cudaEvent_t ready, double* s_out) {
    hua_wait(h);
    std::lock_guard<std::mutex> lk(h->mu);
    h->store = store;
    h->ld = ld;
    h->d4 = d4;
    h->cols = cols;
    h->k = k;
    h->vt = vt;
    h->scale = scale;
    h->ready = ready;
    h->s_out = s_out;
    h->next.store(0);
    h->t_ready_ns.store(0);
    h->active = (int)h->workers.size();
    h->posted = true;
    ++h->gen;
    h->cv_job.notify_all();
}

double hua_wait(HostUnitA* h) {
    if (!h) return 0.0;
    std::unique_lock<std::mutex> lk(h->mu);
    if (!h->posted) return 0.0;
    h->cv_done.wait(lk, [&] { return h->active == 0; });
    h->posted = false;
    const int64_t t0 = h->t_ready_ns.load();
    const int64_t t1 = h->t_end.time_since_epoch().count();
    return t0 > 0 && t1 > t0 ? (double)(t1 - t0) * 1e-9 : 0.0;
}
