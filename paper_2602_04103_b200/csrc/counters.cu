// counters.cu — per-launch work counters for the dynamic work orders (sbcache.cu, fm.cu).
//
// A per-device ring of counters, each with the event of its last use: a launch takes the next
// slot, makes its stream wait for that event (so a slot is never shared by two launches in
// flight, whatever streams they run on), zeroes it stream-ordered and records the event again
// after the kernel.  No allocation per launch: cudaMallocAsync / cudaFreeAsync on the staged
// path's streams added cross-stream dependencies (e2e 5.98 -> 2.64 Gq/s).  The ring lock is held
// from acquire to release (host side only: wait, memset, launch, record).
#include <map>
#include <mutex>

#include "qr_common.cuh"

namespace qr {

constexpr int CTR_SLOTS = 64;
constexpr int CTR_WORDS = 4;          // u64 words per counter slot (zeroed together)
struct CtrRing {
  std::mutex mu;
  unsigned long long* d = nullptr;
  cudaEvent_t ev[CTR_SLOTS] = {};
  uint32_t next = 0;
};

static CtrRing* ctr_ring(int device) {
  static std::mutex mu;
  static std::map<int, CtrRing*> rings;
  std::lock_guard<std::mutex> g(mu);
  CtrRing*& r = rings[device];
  if (!r) {
    CtrRing* n = new CtrRing();
    if (cudaMalloc((void**)&n->d, CTR_SLOTS * 128) != cudaSuccess) { delete n; return nullptr; }
    for (int i = 0; i < CTR_SLOTS; ++i)
      if (cudaEventCreateWithFlags(&n->ev[i], cudaEventDisableTiming) != cudaSuccess) {
        for (int j = 0; j < i; ++j) cudaEventDestroy(n->ev[j]);
        cudaFree(n->d);
        delete n;
        return nullptr;
      }
    r = n;
  }
  return r;
}

cudaError_t CounterLease::acquire(int device, cudaStream_t st, unsigned long long** ctr) {
  // Inside a stream capture (CUDA graphs) the ring's cross-stream event wait is not allowed:
  // the counter is a stream-ordered allocation of the graph instead (memory node; a graph
  // exec never runs concurrently with itself), zeroed and freed inside the same capture.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive) {
    cudaError_t e = cudaMallocAsync((void**)ctr, CTR_WORDS * sizeof(unsigned long long), st);
    if (!e) e = cudaMemsetAsync(*ctr, 0, CTR_WORDS * sizeof(unsigned long long), st);
    if (!e) own = *ctr;
    return e;
  }
  cudaGetLastError();
  CtrRing* r = ctr_ring(device);
  if (!r) return cudaErrorMemoryAllocation;
  r->mu.lock();
  ring = r;
  slot = r->next++ % CTR_SLOTS;
  *ctr = r->d + 16 * slot;                        // one 128-B line per counter
  cudaError_t e = cudaStreamWaitEvent(st, r->ev[slot], 0);
  if (!e) e = cudaMemsetAsync(*ctr, 0, CTR_WORDS * sizeof(unsigned long long), st);
  if (e) { r->mu.unlock(); ring = nullptr; }
  return e;
}

cudaError_t CounterLease::release(cudaStream_t st) {
  if (own) {
    cudaError_t e = cudaFreeAsync(own, st);
    own = nullptr;
    return e;
  }
  if (!ring) return cudaSuccess;
  CtrRing* r = static_cast<CtrRing*>(ring);
  cudaError_t e = cudaEventRecord(r->ev[slot], st);
  ring = nullptr;
  r->mu.unlock();
  return e;
}

CounterLease::~CounterLease() {
  if (ring) static_cast<CtrRing*>(ring)->mu.unlock();
}

// ---- output checksum (qr_checksum) ----------------------------------------------------------
__device__ __forceinline__ uint64_t cks_mix(uint64_t i, uint64_t v) {
  uint64_t z = v ^ (i * 0x9E3779B97F4A7C15ull) ^ 0xD6E8FEB86659FD93ull;
  z = (z ^ (z >> 32)) * 0xD6E8FEB86659FD93ull;
  z = (z ^ (z >> 32)) * 0xD6E8FEB86659FD93ull;
  return z ^ (z >> 32);
}
template <typename T>
__global__ void k_checksum(const T* __restrict__ d, uint64_t n, uint64_t i0, unsigned long long* __restrict__ sum) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += cks_mix(i0 + i, (uint64_t)d[i]);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sum, (unsigned long long)acc);
}

// ---- opt-in range check (QR_ERANGE) ----------------------------------------------------------
__global__ void k_count_gt(const uint64_t* __restrict__ q, uint64_t m, uint64_t n, unsigned long long* __restrict__ cnt) {
  uint32_t c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    c += q[i] > n ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}
cudaError_t launch_count_gt(const uint64_t* q, uint64_t m, uint64_t n, unsigned long long* cnt, int device,
                            cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  k_count_gt<<<grid_stride_blocks(m, 256, sm_count(device), 8), 256, 0, st>>>(q, m, n, cnt);
  return cudaGetLastError();
}

}  // namespace qr

using namespace qr;
#define QR_EXPORT extern "C" __attribute__((visibility("default")))

QR_EXPORT qr_status qr_checksum(const void* data, uint64_t count, int word_bytes, uint64_t index0, uint64_t* sum,
                                void* stream) {
  if (!sum || (count && !data)) return fail(QR_EINVAL, "qr_checksum: null pointer");
  if (word_bytes != 4 && word_bytes != 8) return fail(QR_EINVAL, "qr_checksum: word_bytes must be 4 or 8");
  if (count == 0) return QR_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned g = grid_stride_blocks(count, 256, sm_count(dev), 8);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* s = reinterpret_cast<unsigned long long*>(sum);
  if (word_bytes == 8) k_checksum<uint64_t><<<g, 256, 0, st>>>((const uint64_t*)data, count, index0, s);
  else k_checksum<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)data, count, index0, s);
  cudaError_t e = cudaGetLastError();
  return e ? cuda_fail(e, "qr_checksum") : QR_OK;
}
