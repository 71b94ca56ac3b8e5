// sched.cuh — work order of the query kernels (static grid stride or dynamic warp chunks).
//
// Static (DYN = false): the grid-stride order — the unit (lane pair, or lane when QPW = 32)
// with global index U handles queries U, U + units, U + 2 units, ...  Dynamic (DYN = true): each
// warp takes chunks of SC_CHUNK_STEPS groups of QPW * K consecutive queries from a global counter
// (one atomicAdd per chunk, taken while the current group's gathers are in flight), so SMs that
// run faster take more chunks instead of waiting for the slowest at the end of the launch
// (measured 35.0 -> 46.3 Gq/s on the BiRank cluster kernel).  QPW = queries per
// warp per sub-group: 16 for lane-pair kernels, 32 for one lane per query.
#pragma once
#include <stdint.h>

#include "qr_common.cuh"

namespace qr {

constexpr uint32_t SC_CHUNK_STEPS = 8;

struct ScSched {
  uint64_t gb;          // first query index of the warp's current group
  uint64_t stride;      // distance between the K sub-groups of a group
  uint64_t step;        // static: advance per group
  uint32_t r;           // dynamic: group within the chunk
};

template <int K, int QPW>
__device__ __forceinline__ uint64_t sc_grab(unsigned long long* ctr) {
  uint64_t b = 0;
  if ((threadIdx.x & 31u) == 0) b = atomicAdd(ctr, (unsigned long long)(QPW * K * SC_CHUNK_STEPS));
  return __shfl_sync(0xffffffffu, b, 0);
}

template <int K, bool DYN, int QPW>
__device__ __forceinline__ ScSched sc_first(unsigned long long* ctr) {
  ScSched s;
  s.r = 0;
  if (DYN) {
    s.gb = sc_grab<K, QPW>(ctr);
    s.stride = QPW;
    s.step = (uint64_t)QPW * K;
  } else {
    const uint64_t units = ((uint64_t)gridDim.x * blockDim.x) / (32 / QPW);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    s.gb = (tid & ~31ull) / (32 / QPW);
    s.stride = units;
    s.step = units * K;
  }
  return s;
}

template <int K, bool DYN, int QPW>
__device__ __forceinline__ ScSched sc_next(ScSched s, unsigned long long* ctr) {
  if (DYN) {
    if (++s.r == SC_CHUNK_STEPS) { s.gb = sc_grab<K, QPW>(ctr); s.r = 0; }
    else s.gb += s.step;
  } else {
    s.gb += s.step;
  }
  return s;
}

// the lane's unit within its warp's group (0..QPW-1)
template <int QPW>
__device__ __forceinline__ uint32_t sc_unit_in_warp() {
  return (threadIdx.x & 31u) / (32 / QPW);
}

extern int g_rank_dyn;

// The global-memory query kernels take the dynamic order for large batches only: below 2^22
// queries the counter's memset would be a visible share of the launch.
inline bool use_dyn_order(uint64_t m) { return g_rank_dyn != 0 && m >= (1ull << 22); }

// Launch a 256-thread query kernel in the static order (KS, multi-wave grid `grid_static`, null
// counter) or the dynamic one (KD: the resident grid, capped by grid_static, with a leased
// counter).  Both kernels take the counter as their last argument.
template <typename KS, typename KD, typename... Args>
cudaError_t launch_ordered(KS ks, KD kd, bool dyn, int device, int sms, unsigned grid_static, cudaStream_t st,
                           Args... args) {
  if (!dyn) {
    ks<<<grid_static, 256, 0, st>>>(args..., (unsigned long long*)nullptr);
    return cudaGetLastError();
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kd, 256, 0) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  const unsigned res = (unsigned)per_sm * (unsigned)sms;
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e = lease.acquire(device, st, &ctr);
  if (e) return e;
  kd<<<res < grid_static ? res : grid_static, 256, 0, st>>>(args..., ctr);
  e = cudaGetLastError();
  cudaError_t e2 = lease.release(st);
  return e ? e : e2;
}

// As launch_ordered, with `smem` bytes of dynamic shared memory per CTA (<= 48 KB).
template <typename KS, typename KD, typename... Args>
cudaError_t launch_ordered_smem(KS ks, KD kd, bool dyn, int device, int sms, unsigned grid_static, size_t smem,
                                cudaStream_t st, Args... args) {
  if (!dyn) {
    ks<<<grid_static, 256, smem, st>>>(args..., (unsigned long long*)nullptr);
    return cudaGetLastError();
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kd, 256, smem) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  const unsigned res = (unsigned)per_sm * (unsigned)sms;
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e = lease.acquire(device, st, &ctr);
  if (e) return e;
  kd<<<res < grid_static ? res : grid_static, 256, smem, st>>>(args..., ctr);
  e = cudaGetLastError();
  cudaError_t e2 = lease.release(st);
  return e ? e : e2;
}

}  // namespace qr
