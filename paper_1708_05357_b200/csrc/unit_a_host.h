// Host-thread share of the unit-A gap refresh (Alg. 2 l.7-10).
//
// In the paper unit A is the slower, larger-memory device that keeps the gap memory
// fresh while unit B runs the epochs.  Out of core on a B200 the refresh reads the
// non-resident columns over PCIe (zero-copy), which it shares with the working-set
// swaps; the host's own DRAM bandwidth is larger than PCIe, so the host cores take
// part of those columns: they compute the partial products s_i = a_i^T v~ straight
// from the pinned host store (v~ = the round-start snapshot, copied to the host on
// the compute stream), and the device finishes gap_i from s_i (k_gap_finalize, the
// same Eq. 4 / App. E code as the GPU refresh).  Only the dot products run here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

struct HostUnitA;

// threads >= 1 workers bound to CUDA device `dev` (they wait on events of it).
HostUnitA* hua_create(int threads, int dev);
void hua_destroy(HostUnitA* h);

// Posts one job: for t in [0, k): s_out[t] = scale * sum_{r < d4} store[cols[t] * ld + r] * vt[r],
// fp64 accumulation of fp32 data, and, if norm_out is not null, norm_out[t] = sum_r a_r^2 (fp64;
// duhl_create's ingest share).  vt becomes valid when `ready` completes (the workers wait on
// it).  cols, vt, s_out and norm_out must stay valid until hua_wait returns.  One job at a time.
void hua_post(HostUnitA* h, const float* store, int64_t ld, int64_t d4, const int64_t* cols, int64_t k,
              const double* vt, double scale, cudaEvent_t ready, double* s_out, double* norm_out = nullptr);

// Blocks until the posted job (if any) completes; returns its wall seconds from the
// moment `ready` completed to the last column (0 with no job).
double hua_wait(HostUnitA* h);
