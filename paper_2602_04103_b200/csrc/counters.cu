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

}  // namespace qr
