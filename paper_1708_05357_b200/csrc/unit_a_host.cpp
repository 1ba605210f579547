// Host-thread share of the unit-A refresh: see unit_a_host.h.
#include "unit_a_host.h"

#include <immintrin.h>

#include <atomic>
#include <cstdlib>
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

// Four columns against one v: each 8-element slice of v is loaded once (a zmm) and used by
// four columns, so v (1.6 MB at C4) streams from L2 a quarter as often; 8 FMA chains.
__attribute__((target("avx512f"))) void dot4_avx512(const float* const* a, const double* v, int64_t n,
                                                    double* out) {
    __m512d s[4][2];
    for (int c = 0; c < 4; ++c) s[c][0] = s[c][1] = _mm512_setzero_pd();
    int64_t i = 0;
    for (; i + 16 <= n; i += 16) {
        const __m512d v0 = _mm512_loadu_pd(v + i), v1 = _mm512_loadu_pd(v + i + 8);
#pragma GCC unroll 4
        for (int c = 0; c < 4; ++c) {
            const __m512 f = _mm512_loadu_ps(a[c] + i);
            s[c][0] = _mm512_fmadd_pd(_mm512_cvtps_pd(_mm512_castps512_ps256(f)), v0, s[c][0]);
            s[c][1] = _mm512_fmadd_pd(
                _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(f), 1))), v1, s[c][1]);
        }
    }
    for (int c = 0; c < 4; ++c) {
        double r = _mm512_reduce_add_pd(_mm512_add_pd(s[c][0], s[c][1]));
        for (int64_t k = i; k < n; ++k) r += (double)a[c][k] * v[k];
        out[c] = r;
    }
}

// Four columns: a^T v and ||a||^2 in one read (duhl_create's ingest share on the host).
__attribute__((target("avx512f"))) void dotnorm4_avx512(const float* const* a, const double* v, int64_t n,
                                                        double* out, double* nrm) {
    __m512d s[4], q[4];
    for (int c = 0; c < 4; ++c) s[c] = q[c] = _mm512_setzero_pd();
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        const __m512d v0 = _mm512_loadu_pd(v + i);
#pragma GCC unroll 4
        for (int c = 0; c < 4; ++c) {
            const __m512d f = _mm512_cvtps_pd(_mm256_loadu_ps(a[c] + i));
            s[c] = _mm512_fmadd_pd(f, v0, s[c]);
            q[c] = _mm512_fmadd_pd(f, f, q[c]);
        }
    }
    for (int c = 0; c < 4; ++c) {
        double r = _mm512_reduce_add_pd(s[c]), w = _mm512_reduce_add_pd(q[c]);
        for (int64_t k = i; k < n; ++k) {
            const double x = (double)a[c][k];
            r += x * v[k];
            w += x * x;
        }
        out[c] = r;
        nrm[c] = w;
    }
}

double norm_scalar(const float* a, int64_t n) {
    double r0 = 0, r1 = 0;
    int64_t i = 0;
    for (; i + 2 <= n; i += 2) {
        r0 += (double)a[i] * a[i];
        r1 += (double)a[i + 1] * a[i + 1];
    }
    for (; i < n; ++i) r0 += (double)a[i] * a[i];
    return r0 + r1;
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
    bool avx2 = false, avx512 = false;
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
    double* norm_out = nullptr;
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
                const int64_t t = next.fetch_add(4, std::memory_order_relaxed);
                if (t >= k) break;
                if (avx512 && t + 4 <= k) {
                    const float* a4[4];
                    double r[4], w[4];
                    for (int c = 0; c < 4; ++c) a4[c] = store + cols[t + c] * ld;
                    if (norm_out) dotnorm4_avx512(a4, vt, d4, r, w);
                    else dot4_avx512(a4, vt, d4, r);
                    for (int c = 0; c < 4; ++c) {
                        s_out[t + c] = scale * r[c];
                        if (norm_out) norm_out[t + c] = w[c];
                    }
                    continue;
                }
                for (int64_t u = t; u < t + 4 && u < k; ++u) {
                    const float* a = store + cols[u] * ld;
                    s_out[u] = scale * (avx2 ? dot_avx2(a, vt, d4) : dot_scalar(a, vt, d4));
                    if (norm_out) norm_out[u] = norm_scalar(a, d4);
                }
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
    h->avx512 = __builtin_cpu_supports("avx512f") && std::getenv("DUHL_HOST_NO_AVX512") == nullptr;
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
              const double* vt, double scale, cudaEvent_t ready, double* s_out, double* norm_out) {
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
    h->norm_out = norm_out;
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
