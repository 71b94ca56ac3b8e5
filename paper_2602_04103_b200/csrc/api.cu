// api.cu — the extern "C" boundary of libqrank.so (include/qrank.h).
//
// Validation, handle lifetime, pointer-space detection and the staged host-pointer path
// live here; every step of the method runs in the kernels of birank.cu, quadrank.cu and
// fm.cu.  No exception crosses the ABI; errors are status codes plus a thread-local message.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <new>
#include <vector>

#include "qr_common.cuh"

#define QR_EXPORT extern "C" __attribute__((visibility("default")))

namespace qr {

// ---- tuning knobs (set through qr_set_tuning; defaults chosen from B200 measurements) ----
int g_rank_k = 2;               // independent queries per lane (pair) per iteration
int g_rank_blocks_per_sm = 64;  // 256-thread CTAs per SM of the grid (several waves)
int g_fm_blocks_per_sm = 64;    // 256-thread CTAs per SM of the FM grid (several waves)
int g_rank_s_lane = 1;
int g_fm_dyn = 1;               // FM count: 1 = persistent grid + warp chunks from a global counter, 0 = static grid stride
int g_fm_seed = 0;              // FM seed pre-pass (dynamic order only): 0 auto (L2-resident BWT), 1 never, 2 always
int g_fm_smem = 1;              // FM superblock words from shared memory: 0 off, 1 auto, 2 packed table whenever it fits
int g_fm_refill = 0;            // L2-resident count kernel: refill a warp's lanes once this many are idle (0 auto)
int g_fm_packed = 1;            // L2-resident count kernel: packed post-seed symbols for short fixed-length batches
extern uint64_t g_ax1_aq_per_task;   // fm.cu
extern int g_fm_ax_bfs2, g_fm_ax_bfs3, g_ax_seed_split;   // fm.cu
int g_fm_ax_bfs = 1;            // approximate search k = 1: breadth-first kernels (k_ax1_*): 0 never, 1 auto, 2 always
int g_fm_kbits = 0;             // approximate search: presence bitmap of the k-mer table, 0 auto (sparse table), 1 never, 2 always
int g_check_range = 0;          // 1: qr_rank / qr_rank_all4 count q > n and return QR_ERANGE (synchronous)
int g_fm_lean = 0;              // FM step flavour: 0 auto (by L2 residency), 1 de-duplicating, 2 lean, 3 one line per iteration
int g_index64 = 0;              // 1: force the 64-bit line-index path (tests the n >= 2^36/2^37 code on small n)
int g_rank_smem = 1;            // superblock words from cluster shared memory: 0 never, 1 large batches, 2 always
int g_rank_dyn = 1;             // cluster rank kernels: 1 = dynamic (atomic chunk) work order, 0 = static grid stride
int g_rank_smem_clusters = 0;   // cluster rank kernels: 0 = as many 2-CTA clusters as fit (occupancy API), else this many
int g_rank_smem_threads = 0;    // cluster rank kernels: CTA size (0 auto: 1024, 768 for K = 6, 512 for K = 8)
int g_rank_smem_k = 0;          // cluster rank kernels: queries per lane pair per group (0 auto, 1, 2, 4 @1024 thr, 6 @768, 8 @512)
int g_rank_lane_table = 1;      // one-lane kernels take the superblock words from a per-CTA shared-memory table when small
int g_rank_resident = 1;        // structures that fit one CTA's shared memory are queried from a per-CTA copy
int g_rank_big_pack = 0;        // 1: also build the large-n (CS-CTA cluster) BiRank16 table below n = 2^35 (tests)
int g_rank_big_cs = 0;          // cluster size of that table: 0 smallest that fits, else 4, 8 or 16
int g_rank_pair = 2;            // kernel shape: 2 by structure size (default), 1 lane pairs (one L2 request per query), 0 one lane per query
uint64_t g_stage_chunk = 1ull << 23;   // queries per chunk on the staged host path (sweep: profiles/r01_e2e_sweep)
int g_stage_slots = 3;                 // device buffers / internal streams of the staged path

cudaError_t smem_limit_raise(const void* kern, size_t bytes, int device) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> limit;
  if (bytes == 0) return cudaSuccess;
  std::lock_guard<std::mutex> g(mu);
  size_t& lim = limit[std::make_pair(kern, device)];
  if (bytes <= lim) return cudaSuccess;
  // without the opt-in, dynamic + static shared memory must stay within 48 KB
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && bytes + fa.sharedSizeBytes <= 48 * 1024) {
    lim = bytes;
    return cudaSuccess;
  }
  cudaGetLastError();
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != device) cudaSetDevice(device);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  if (e == cudaSuccess) lim = bytes;
  return e;
}

static thread_local char t_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}
qr_status fail(qr_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return st;
}
qr_status cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? QR_ENOMEM : QR_ECUDA;
}

int pointer_space(const void* p, int device) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear: unregistered host memory on older runtimes
    return 0;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return a.device == device ? 1 : -1;
  return 0;
}

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> g(mu);
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = NUM_SMS_B200;
    cache[device] = v;
  }
  return cache[device];
}

int l2_bytes(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> g(mu);
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device) != cudaSuccess || v <= 0) v = 126 << 20;
    cache[device] = v;
  }
  return cache[device];
}

qr_status alloc_index(int sigma, uint64_t n, int device, qr_index** out, int layout) {
  qr_index* h = new (std::nothrow) qr_index();
  if (!h) return fail(QR_ENOMEM, "host allocation");
  if (!layout) layout = sigma == 2 ? QR_LAYOUT_BIRANK16 : QR_LAYOUT_QUADRANK16;
  h->sigma = sigma;
  h->layout = layout;
  h->device = device;
  h->n = n;
  uint64_t B = 0;
  uint32_t sb = 0;
  switch (layout) {
    case QR_LAYOUT_BIRANK16: B = BI_B; sb = BI_SB_LOG; break;
    case QR_LAYOUT_QUADRANK16: B = QD_B; sb = QD_SB_LOG; break;
    case QR_LAYOUT_BIRANK64X2: B = 384; break;      // 2 x 192 data bits per line
    case QR_LAYOUT_BIRANK16X2: B = B16X2_B; sb = BI_SB_LOG; break;   // 2 x 240 data bits, BiRank16 superblocks
    case QR_LAYOUT_BIRANK32X2: B = B32X2_B; sb = B32X2_SB_LOG; break; // 2 x 224 data bits, u64 L1 per 2^23 lines
    case QR_LAYOUT_QUADRANK16X2: B = Q16X2_B; sb = QD_SB_LOG; break; // 2 x 96 chars, QuadRank16 superblocks
    default: B = 128; break;                        // QuadRank64: 128 chars per line
  }
  h->n_lines = n / B + 1;                               // reading R4: q = n stays in range
  h->n_super = sb ? ((h->n_lines - 1) >> sb) + 1 : 0;   // the 64-bit variants have no L1 array
  h->sm_count = sm_count(device);
  cudaError_t e;
  if ((e = cudaMalloc((void**)&h->lines, h->n_lines * 64))) { delete h; return cuda_fail(e, "alloc lines"); }
  const uint64_t sbytes = super_bytes_of(h);
  if (sbytes && (e = cudaMalloc((void**)&h->super, sbytes))) {
    cudaFree(h->lines); delete h; return cuda_fail(e, "alloc super");
  }
  *out = h;
  return QR_OK;
}

uint64_t super_bytes_of(const qr_index* h) {
  return h->n_super * (h->layout == QR_LAYOUT_BIRANK32X2 ? 8 : h->sigma == 2 ? 4 : 16);
}

void fm_copy_locked(const qr_fm* src, qr_fm* dst);
qr_status fm_build_device(const uint64_t* d_text, uint64_t n, const uint32_t* d_sa_given, int device, cudaStream_t st,
                          qr_fm** out, int kmer_k, int bwt_layout, int kmer_k_ax);
__global__ void k_mask_tail_bits(uint64_t* words, uint64_t n);
__global__ void k_mask_tail_chars(uint64_t* words, uint64_t n);
cudaError_t launch_bi_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode, cudaStream_t st);
cudaError_t launch_qd_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode, cudaStream_t st);

cudaError_t launch_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode, cudaStream_t st) {
  if (h->layout == QR_LAYOUT_BIRANK16X2) return launch_b16x2_rank(h, q, nullptr, out, m, 2, st);   // same sector loads
  if (h->layout == QR_LAYOUT_QUADRANK16X2) return launch_q16x2_rank(h, q, nullptr, out, m, 2, st);
  if (h->layout == QR_LAYOUT_BIRANK32X2) return launch_b32x2_rank(h, q, nullptr, out, m, 2, st);
  if (h->layout == QR_LAYOUT_BIRANK64X2 || h->layout == QR_LAYOUT_QUADRANK64)
    return launch_variant(h, q, nullptr, out, m, 2, st);   // the variants' loads (modes coincide)
  return h->sigma == 2 ? launch_bi_gather(h, q, out, m, mode, st) : launch_qd_gather(h, q, out, m, mode, st);
}
static bool is_variant(const qr_index* h) {
  return h->layout == QR_LAYOUT_BIRANK64X2 || h->layout == QR_LAYOUT_QUADRANK64 || h->layout == QR_LAYOUT_BIRANK16X2 ||
         h->layout == QR_LAYOUT_QUADRANK16X2 || h->layout == QR_LAYOUT_BIRANK32X2;
}

// RAII device guard
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Copy `words` u64 of a host-or-device input into a fresh zero-padded device buffer of
// `padded_words` u64 (stream-ordered).  Caller releases it with free_staged.  Plain cudaMalloc:
// the stream-ordered pool maps / unmaps GB-sized blocks ~50x slower (profiles/r01_alloc_probe.jsonl).
static qr_status stage_input(const uint64_t* src, uint64_t words, uint64_t padded_words, cudaStream_t st,
                             uint64_t** dst) {
  cudaError_t e;
  uint64_t* d = nullptr;
  if ((e = cudaMalloc((void**)&d, padded_words * 8))) return cuda_fail(e, "alloc staged input");
  if (padded_words > words) cudaMemsetAsync(d + words, 0, (padded_words - words) * 8, st);
  if (words && (e = cudaMemcpyAsync(d, src, words * 8, cudaMemcpyDefault, st))) {
    cudaStreamSynchronize(st);
    cudaFree(d);
    return cuda_fail(e, "copy input");
  }
  *dst = d;
  return QR_OK;
}

// Release a build temporary once the work queued on `st` that reads it has finished.
// Returns the synchronisation's status (an asynchronous fault of the build surfaces here).
static cudaError_t free_staged(void* d, cudaStream_t st) {
  if (!d) return cudaSuccess;
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d);
  return e;
}

// ---- staged host-pointer pipeline ----------------------------------------------------------
// S slots (default 3, knob stage_slots), one internal stream each: chunk k uses slot k%S on stream k%S, so the H2D
// copy and kernel of one chunk overlap the kernel and D2H copy of the others (separate copy
// engines).  In-order streams make slot reuse safe across chunks and across calls.
constexpr int MAX_SLOTS = 4;
struct Stager {
  std::mutex mu;
  cudaStream_t s[MAX_SLOTS] = {};
  cudaEvent_t ev_start = nullptr, ev_done[MAX_SLOTS] = {};
  void* buf[MAX_SLOTS] = {};
  size_t cap = 0;
};
static std::mutex g_stagers_mu;
static std::vector<Stager*> g_stagers;

static Stager* stager_for(int device) {
  std::lock_guard<std::mutex> g(g_stagers_mu);
  if ((int)g_stagers.size() <= device) g_stagers.resize(device + 1, nullptr);
  if (!g_stagers[device]) {
    Stager* S = new (std::nothrow) Stager();
    if (!S) return nullptr;
    bool ok = cudaEventCreateWithFlags(&S->ev_start, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < MAX_SLOTS && ok; ++i)
      ok = cudaStreamCreateWithFlags(&S->s[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&S->ev_done[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {   // the staged path never falls back to the legacy stream
      for (int i = 0; i < MAX_SLOTS; ++i) {
        if (S->s[i]) cudaStreamDestroy(S->s[i]);
        if (S->ev_done[i]) cudaEventDestroy(S->ev_done[i]);
      }
      if (S->ev_start) cudaEventDestroy(S->ev_start);
      delete S;
      cudaGetLastError();
      return nullptr;
    }
    g_stagers[device] = S;
  }
  return g_stagers[device];
}

struct StageArray {
  const void* host_in;   // input (host) or nullptr
  void* host_out;        // output (host) or nullptr
  size_t item_bytes;
};

template <typename Launch>
static qr_status run_staged(int device, cudaStream_t user, uint64_t m, const std::vector<StageArray>& arrays,
                            Launch launch) {
  Stager* S = stager_for(device);
  if (!S) return fail(QR_ECUDA, "staged path: cannot create internal streams/events on device %d", device);
  std::lock_guard<std::mutex> g(S->mu);
  size_t per_item = 0;
  for (auto& a : arrays) per_item += (a.item_bytes + 15) & ~size_t(15);
  const uint64_t chunk = g_stage_chunk;
  const int nslot = g_stage_slots;
  const size_t need = per_item * (size_t)(m < chunk ? m : chunk) + 256 * arrays.size();
  cudaError_t e;
  if (S->cap < need || !S->buf[nslot - 1]) {
    for (int i = 0; i < MAX_SLOTS; ++i) {
      if (S->buf[i]) { cudaStreamSynchronize(S->s[i]); cudaFree(S->buf[i]); S->buf[i] = nullptr; }
    }
    S->cap = 0;
    for (int i = 0; i < nslot; ++i)
      if ((e = cudaMalloc(&S->buf[i], need))) return cuda_fail(e, "alloc staging buffers");
    S->cap = need;
  }
  cudaEventRecord(S->ev_start, user);                   // respect work already queued on `user`
  for (int i = 0; i < nslot; ++i) cudaStreamWaitEvent(S->s[i], S->ev_start, 0);
  // Whatever happens below, `user` is made to wait for everything already enqueued on the
  // internal streams, so the caller can never free buffers that a copy still reads or writes.
  auto join = [&]() {
    for (int i = 0; i < nslot; ++i) {
      cudaEventRecord(S->ev_done[i], S->s[i]);
      cudaStreamWaitEvent(user, S->ev_done[i], 0);
    }
  };
  uint64_t k = 0;
  for (uint64_t lo = 0; lo < m; lo += chunk, ++k) {
    const uint64_t cnt = (m - lo < chunk) ? m - lo : chunk;
    const int slot = (int)(k % (uint64_t)nslot);
    cudaStream_t st = S->s[slot];
    char* base = static_cast<char*>(S->buf[slot]);
    std::vector<void*> dptr(arrays.size());
    size_t off = 0;
    for (size_t a = 0; a < arrays.size(); ++a) {
      dptr[a] = base + off;
      off += (((arrays[a].item_bytes + 15) & ~size_t(15)) * (size_t)cnt + 255) & ~size_t(255);
      if (arrays[a].host_in &&
          (e = cudaMemcpyAsync(dptr[a], static_cast<const char*>(arrays[a].host_in) + lo * arrays[a].item_bytes,
                               cnt * arrays[a].item_bytes, cudaMemcpyHostToDevice, st))) {
        join();
        return cuda_fail(e, "staged H2D");
      }
    }
    qr_status rs = launch(dptr, cnt, st);
    if (rs != QR_OK) { join(); return rs; }
    for (size_t a = 0; a < arrays.size(); ++a)
      if (arrays[a].host_out &&
          (e = cudaMemcpyAsync(static_cast<char*>(arrays[a].host_out) + lo * arrays[a].item_bytes, dptr[a],
                               cnt * arrays[a].item_bytes, cudaMemcpyDeviceToHost, st))) {
        join();
        return cuda_fail(e, "staged D2H");
      }
  }
  join();
  if ((e = cudaGetLastError())) return cuda_fail(e, "staged pipeline");
  return QR_OK;
}

// classify a set of query pointers: 1 = all device (on `device`), 0 = all host, -1 = mixed/foreign
static int classify(std::initializer_list<const void*> ptrs, int device) {
  int kind = -2;
  for (const void* p : ptrs) {
    if (!p) continue;
    int s = pointer_space(p, device);
    if (s < 0) return -1;
    if (kind == -2) kind = s;
    else if (kind != s) return -1;
  }
  return kind == -2 ? 1 : kind;
}

}  // namespace qr

using namespace qr;

// =============================================================================== exports

QR_EXPORT const char* qr_last_error(void) { return t_err; }
QR_EXPORT const char* qr_version(void) { return "qrank-b200 0.1 (sm_100a)"; }

QR_EXPORT qr_status qr_set_tuning(const char* key, int64_t value) {
  if (!key) return fail(QR_EINVAL, "qr_set_tuning: null key");
  if (!strcmp(key, "rank_k")) {
    if (value != 1 && value != 2 && value != 4 && value != 8) return fail(QR_EINVAL, "rank_k must be 1, 2, 4 or 8");
    g_rank_k = (int)value;
  } else if (!strcmp(key, "rank_blocks_per_sm")) {
    if (value < 1 || value > 64) return fail(QR_EINVAL, "rank_blocks_per_sm out of range");
    g_rank_blocks_per_sm = (int)value;
  } else if (!strcmp(key, "rank_pair")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "rank_pair must be 0 (lane), 1 (pair) or 2 (by size)");
    g_rank_pair = (int)value;
  } else if (!strcmp(key, "rank_s_lane")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "rank_s_lane must be 0 or 1");
    g_rank_s_lane = (int)value;
  } else if (!strcmp(key, "rank_smem")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "rank_smem must be 0 (off), 1 (auto) or 2 (always)");
    g_rank_smem = (int)value;
  } else if (!strcmp(key, "rank_smem_k")) {
    if (value != 0 && value != 1 && value != 2 && value != 3 && value != 4 && value != 6 && value != 8)
      return fail(QR_EINVAL, "rank_smem_k must be 0 (auto), 1, 2, 3, 4, 6 or 8");
    g_rank_smem_k = (int)value;
    g_rank_smem_threads = 0;
  } else if (!strcmp(key, "rank_smem_threads")) {
    // instantiated (K, threads) pairs: K 1-4 @1024, 4 and 6 @768, 8 @512 (set rank_smem_k first)
    const int k = g_rank_smem_k;
    const bool ok = value == 0 || (value == 1024 && k >= 1 && k <= 4) || (value == 768 && (k == 4 || k == 6)) ||
                    (value == 512 && k == 8);
    if (!ok) return fail(QR_EINVAL, "rank_smem_threads: no kernel for K=%d with %lld threads", k, (long long)value);
    g_rank_smem_threads = (int)value;
  } else if (!strcmp(key, "rank_smem_clusters")) {
    if (value < 0 || value > 4096) return fail(QR_EINVAL, "rank_smem_clusters must be 0..4096");
    g_rank_smem_clusters = (int)value;
  } else if (!strcmp(key, "rank_lane_table")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "rank_lane_table must be 0 or 1");
    g_rank_lane_table = (int)value;
  } else if (!strcmp(key, "rank_resident")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "rank_resident must be 0 or 1");
    g_rank_resident = (int)value;
  } else if (!strcmp(key, "rank_big_pack")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "rank_big_pack must be 0 or 1");
    g_rank_big_pack = (int)value;
  } else if (!strcmp(key, "rank_big_cs")) {
    if (value != 0 && value != 4 && value != 8 && value != 16) return fail(QR_EINVAL, "rank_big_cs must be 0, 4, 8 or 16");
    g_rank_big_cs = (int)value;
  } else if (!strcmp(key, "rank_dyn")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "rank_dyn must be 0 or 1");
    g_rank_dyn = (int)value;
  } else if (!strcmp(key, "fm_dyn")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "fm_dyn must be 0 or 1");
    g_fm_dyn = (int)value;
  } else if (!strcmp(key, "fm_seed")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "fm_seed must be 0 (auto), 1 (never) or 2 (always)");
    g_fm_seed = (int)value;
  } else if (!strcmp(key, "fm_smem")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "fm_smem must be 0 (off), 1 (auto) or 2 (packed)");
    g_fm_smem = (int)value;
  } else if (!strcmp(key, "fm_refill")) {
    if (value < 0 || value > 32) return fail(QR_EINVAL, "fm_refill must be 0 (auto) or 1..32");
    g_fm_refill = (int)value;
  } else if (!strcmp(key, "fm_packed")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "fm_packed must be 0 or 1");
    g_fm_packed = (int)value;
  } else if (!strcmp(key, "fm_ax_bfs")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "fm_ax_bfs must be 0 (never), 1 (auto) or 2 (always)");
    g_fm_ax_bfs = (int)value;
  } else if (!strcmp(key, "fm_ax_bfs2")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "fm_ax_bfs2 must be 0 or 1");
    g_fm_ax_bfs2 = (int)value;
  } else if (!strcmp(key, "fm_ax_bfs3")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "fm_ax_bfs3 must be 0 or 1");
    g_fm_ax_bfs3 = (int)value;
  } else if (!strcmp(key, "fm_ax_seed_split")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "fm_ax_seed_split must be 0 or 1");
    g_ax_seed_split = (int)value;
  } else if (!strcmp(key, "fm_ax_queue")) {
    if (value < 0 || value > 64) return fail(QR_EINVAL, "fm_ax_queue must be 0..64 (interval items per task)");
    g_ax1_aq_per_task = (uint64_t)value;
  } else if (!strcmp(key, "fm_kbits")) {
    if (value < 0 || value > 2) return fail(QR_EINVAL, "fm_kbits must be 0 (auto), 1 (never) or 2 (always)");
    g_fm_kbits = (int)value;
  } else if (!strcmp(key, "check_range")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "check_range must be 0 or 1");
    g_check_range = (int)value;
  } else if (!strcmp(key, "fm_step")) {
    if (value < 0 || value > 4) return fail(QR_EINVAL, "fm_step must be 0 (auto), 1, 2, 3 or 4");
    g_fm_lean = (int)value;
  } else if (!strcmp(key, "index64")) {
    if (value != 0 && value != 1) return fail(QR_EINVAL, "index64 must be 0 or 1");
    g_index64 = (int)value;
  } else if (!strcmp(key, "fm_blocks_per_sm")) {
    if (value < 1 || value > 64) return fail(QR_EINVAL, "fm_blocks_per_sm out of range");
    g_fm_blocks_per_sm = (int)value;
  } else if (!strcmp(key, "l2_fetch_granularity")) {
    // cudaLimitMaxL2FetchGranularity of the current device (0..128 B; a hint to the L2)
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)value);
    if (e) return cuda_fail(e, "qr_set_tuning l2_fetch_granularity");
  } else if (!strcmp(key, "stage_slots")) {
    if (value < 2 || value > MAX_SLOTS) return fail(QR_EINVAL, "stage_slots must be 2..4");
    g_stage_slots = (int)value;
  } else if (!strcmp(key, "stage_chunk")) {
    if (value < 1024) return fail(QR_EINVAL, "stage_chunk too small");
    g_stage_chunk = (uint64_t)value;
  } else {
    return fail(QR_EINVAL, "unknown tuning key '%s'", key);
  }
  return QR_OK;
}

QR_EXPORT qr_status qr_birank_build(const uint64_t* bits, uint64_t n, int device, void* stream, qr_index** out) {
  if (!out || (!bits && n)) return fail(QR_EINVAL, "qr_birank_build: null pointer");
  *out = nullptr;
  if (n >= BI_MAX_N) return fail(QR_ECAPACITY, "qr_birank_build: n >= 2^43 (PAPER.md:411-412)");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_birank_build: bad device %d", device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t L = n / BI_B + 1;
  const uint64_t words = (n + 63) >> 6;
  uint64_t padded = (L * 62 + 7) / 8 + 2;
  if (padded < words + 1) padded = words + 1;
  uint64_t* d = nullptr;
  qr_status s = stage_input(bits, words, padded, st, &d);
  if (s != QR_OK) return s;
  s = birank_build_device(d, n, device, st, out);
  const cudaError_t fe = free_staged(d, st);
  if (s == QR_OK) {
    cudaError_t e = fe ? fe : cudaStreamSynchronize(st);
    if (e) { qr_free(*out); *out = nullptr; return cuda_fail(e, "qr_birank_build"); }
  }
  return s;
}

QR_EXPORT qr_status qr_quadrank_build(const uint64_t* text2b, uint64_t n, int device, void* stream, qr_index** out) {
  if (!out || (!text2b && n)) return fail(QR_EINVAL, "qr_quadrank_build: null pointer");
  *out = nullptr;
  if (n >= QD_MAX_N) return fail(QR_ECAPACITY, "qr_quadrank_build: n >= 2^45 (PAPER.md:514-515)");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_quadrank_build: bad device %d", device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t L = n / QD_B + 1;
  const uint64_t words = (n + 31) >> 5;
  uint64_t padded = 7 * L;
  if (padded < words) padded = words;
  uint64_t* d = nullptr;
  qr_status s = stage_input(text2b, words, padded, st, &d);
  if (s != QR_OK) return s;
  s = quadrank_build_device(d, n, device, st, out);
  const cudaError_t fe = free_staged(d, st);
  if (s == QR_OK) {
    cudaError_t e = fe ? fe : cudaStreamSynchronize(st);
    if (e) { qr_free(*out); *out = nullptr; return cuda_fail(e, "qr_quadrank_build"); }
  }
  return s;
}

QR_EXPORT qr_status qr_build(const uint64_t* text, uint64_t n, int layout, int device, void* stream, qr_index** out) {
  if (layout == QR_LAYOUT_BIRANK16) return qr_birank_build(text, n, device, stream, out);
  if (layout == QR_LAYOUT_QUADRANK16) return qr_quadrank_build(text, n, device, stream, out);
  if (layout != QR_LAYOUT_BIRANK64X2 && layout != QR_LAYOUT_QUADRANK64 && layout != QR_LAYOUT_BIRANK16X2 &&
      layout != QR_LAYOUT_QUADRANK16X2 && layout != QR_LAYOUT_BIRANK32X2)
    return fail(QR_EINVAL, "qr_build: bad layout %d", layout);
  if (!out || (!text && n)) return fail(QR_EINVAL, "qr_build: null pointer");
  *out = nullptr;
  if (n >= (1ull << 48)) return fail(QR_ECAPACITY, "qr_build: n >= 2^48");
  const bool b16x2 = layout == QR_LAYOUT_BIRANK16X2, q16x2 = layout == QR_LAYOUT_QUADRANK16X2;
  const bool b32x2 = layout == QR_LAYOUT_BIRANK32X2;
  if (b32x2 && n >= BI_MAX_N) return fail(QR_ECAPACITY, "qr_build: BiRank32x2 needs n < 2^43");
  if (b16x2 && n >= (1ull << 40)) return fail(QR_ECAPACITY, "qr_build: BiRank16x2 needs n < 2^40 (u32 line index)");
  if (q16x2 && n >= (1ull << 39)) return fail(QR_ECAPACITY, "qr_build: QuadRank16x2 needs n < 2^39 (u32 line index)");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_build: bad device %d", device);
  cudaStream_t st = (cudaStream_t)stream;
  const bool bits = layout == QR_LAYOUT_BIRANK64X2 || layout == QR_LAYOUT_BIRANK16X2 || b32x2;
  const uint64_t L = b16x2 ? n / B16X2_B + 1 : b32x2 ? n / B32X2_B + 1 : q16x2 ? n / Q16X2_B + 1
                   : bits ? n / 384 + 1 : n / 128 + 1;
  const uint64_t words = bits ? (n + 63) >> 6 : (n + 31) >> 5;
  uint64_t padded = b16x2 ? (60 * L + 7) / 8 + 1 : b32x2 ? 7 * L + 1 : q16x2 ? 6 * L : bits ? 6 * L : 4 * L;
  if (padded < words) padded = words;
  uint64_t* d = nullptr;
  qr_status s = stage_input(text, words, padded, st, &d);
  if (s != QR_OK) return s;
  if (bits) k_mask_tail_bits<<<1, 1, 0, st>>>(d, n);
  else      k_mask_tail_chars<<<1, 1, 0, st>>>(d, n);
  s = b16x2 ? birank16x2_build_device(d, n, device, st, out)
      : b32x2 ? birank32x2_build_device(d, n, device, st, out)
      : q16x2 ? quadrank16x2_build_device(d, n, device, st, out)
      : bits ? birank64x2_build_device(d, n, device, st, out) : quadrank64_build_device(d, n, device, st, out);
  const cudaError_t fe = free_staged(d, st);
  if (s == QR_OK) {
    cudaError_t e = fe ? fe : cudaStreamSynchronize(st);
    if (e) { qr_free(*out); *out = nullptr; return cuda_fail(e, "qr_build"); }
  }
  return s;
}

QR_EXPORT qr_status qr_layout(const qr_index* h, int* layout) {
  if (!h || !layout) return fail(QR_EINVAL, "qr_layout: null pointer");
  *layout = h->layout;
  return QR_OK;
}

// The opt-in range check (knob check_range, QR_ERANGE): every chunk's queries are counted on
// the device (q > n) on the stream that ranks them; the call then synchronises and reports.
struct RangeCheck {
  unsigned long long* d = nullptr;
  bool on = false;
  qr_status begin(cudaStream_t st) {
    on = g_check_range != 0;
    if (!on) return QR_OK;
    cudaError_t e = cudaMallocAsync((void**)&d, 8, st);
    if (!e) e = cudaMemsetAsync(d, 0, 8, st);
    return e ? cuda_fail(e, "range check alloc") : QR_OK;
  }
  cudaError_t count(const uint64_t* dq, uint64_t cnt, uint64_t n, int device, cudaStream_t s) {
    return on ? launch_count_gt(dq, cnt, n, d, device, s) : cudaSuccess;
  }
  qr_status end(qr_status s, cudaStream_t st, const char* who) {
    if (!on) return s;
    unsigned long long h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFreeAsync(d, st);
    if (s != QR_OK) return s;
    if (e) return cuda_fail(e, "range check");
    if (h) return fail(QR_ERANGE, "%s: %llu of the queries are > n (PAPER.md:57: 0 <= q <= n)", who, h);
    return QR_OK;
  }
};

QR_EXPORT qr_status qr_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                            void* stream) {
  if (!h) return fail(QR_EINVAL, "qr_rank: null handle");
  if (m == 0) return QR_OK;
  if (!q || !out) return fail(QR_EINVAL, "qr_rank: null q/out");
  if (h->sigma == 4 && !c) return fail(QR_EINVAL, "qr_rank: sigma=4 requires c");
  DeviceGuard dg(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  auto launch = [&](const uint64_t* dq, const uint8_t* dc, uint64_t* dout, uint64_t cnt, cudaStream_t s) -> cudaError_t {
    if (is_variant(h)) return launch_variant(h, dq, dc, dout, cnt, 0, s);
    return h->sigma == 2 ? launch_birank_rank(h, dq, dc, dout, cnt, s) : launch_quadrank_rank(h, dq, dc, dout, cnt, s);
  };
  int sp = classify({q, c, out}, h->device);
  if (sp < 0) return fail(QR_EINVAL, "qr_rank: q, c, out must all be device pointers on device %d or all host", h->device);
  RangeCheck rc;
  qr_status s0 = rc.begin(st);
  if (s0 != QR_OK) return s0;
  if (sp == 1) {
    cudaError_t e = rc.count(q, m, h->n, h->device, st);
    if (!e) e = launch(q, c, out, m, st);
    return rc.end(e ? cuda_fail(e, "qr_rank launch") : QR_OK, st, "qr_rank");
  }
  std::vector<StageArray> arr = {{q, nullptr, 8}, {nullptr, out, 8}};
  if (c) arr.push_back({c, nullptr, 1});
  qr_status s1 = run_staged(h->device, st, m, arr, [&](const std::vector<void*>& d, uint64_t cnt, cudaStream_t s) -> qr_status {
    cudaError_t e = rc.count((const uint64_t*)d[0], cnt, h->n, h->device, s);
    if (!e) e = launch((const uint64_t*)d[0], c ? (const uint8_t*)d[2] : nullptr, (uint64_t*)d[1], cnt, s);
    return e ? cuda_fail(e, "qr_rank launch") : QR_OK;
  });
  return rc.end(s1, st, "qr_rank");
}

QR_EXPORT qr_status qr_rank_chain(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                  uint64_t chain_len, void* stream) {
  if (!h) return fail(QR_EINVAL, "qr_rank_chain: null handle");
  if (m == 0) return QR_OK;
  if (!q || !out || chain_len == 0) return fail(QR_EINVAL, "qr_rank_chain: null q/out or chain_len = 0");
  if (h->sigma == 4 && !c) return fail(QR_EINVAL, "qr_rank_chain: sigma=4 requires c");
  DeviceGuard dg(h->device);
  if (classify({q, c, out}, h->device) != 1) return fail(QR_EINVAL, "qr_rank_chain: device pointers only");
  cudaError_t e = launch_rank_chain(h, q, c, out, m, chain_len, (cudaStream_t)stream);
  return e ? cuda_fail(e, "qr_rank_chain launch") : QR_OK;
}

QR_EXPORT qr_status qr_rank_all4(const qr_index* h, const uint64_t* q, uint64_t* out4, uint64_t m, void* stream) {
  if (!h) return fail(QR_EINVAL, "qr_rank_all4: null handle");
  if (h->sigma != 4) return fail(QR_EINVAL, "qr_rank_all4: needs a QuadRank (sigma=4) handle");
  if (m == 0) return QR_OK;
  if (!q || !out4) return fail(QR_EINVAL, "qr_rank_all4: null q/out4");
  DeviceGuard dg(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  int sp = classify({q, out4}, h->device);
  if (sp < 0) return fail(QR_EINVAL, "qr_rank_all4: q and out4 must both be device (device %d) or both host", h->device);
  auto launch4 = [&](const uint64_t* dq, uint64_t* d4, uint64_t cnt, cudaStream_t s) -> cudaError_t {
    return is_variant(h) ? launch_variant(h, dq, nullptr, d4, cnt, 1, s) : launch_quadrank_all4(h, dq, d4, cnt, s);
  };
  RangeCheck rc;
  qr_status s0 = rc.begin(st);
  if (s0 != QR_OK) return s0;
  if (sp == 1) {
    cudaError_t e = rc.count(q, m, h->n, h->device, st);
    if (!e) e = launch4(q, out4, m, st);
    return rc.end(e ? cuda_fail(e, "qr_rank_all4 launch") : QR_OK, st, "qr_rank_all4");
  }
  std::vector<StageArray> arr = {{q, nullptr, 8}, {nullptr, out4, 32}};
  qr_status s1 = run_staged(h->device, st, m, arr, [&](const std::vector<void*>& d, uint64_t cnt, cudaStream_t s) -> qr_status {
    cudaError_t e = rc.count((const uint64_t*)d[0], cnt, h->n, h->device, s);
    if (!e) e = launch4((const uint64_t*)d[0], (uint64_t*)d[1], cnt, s);
    return e ? cuda_fail(e, "qr_rank_all4 launch") : QR_OK;
  });
  return rc.end(s1, st, "qr_rank_all4");
}

QR_EXPORT qr_status qr_gather_ceiling(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode,
                                      void* stream) {
  if (!h || (m && (!q || !out))) return fail(QR_EINVAL, "qr_gather_ceiling: null pointer");
  if (mode < 0 || mode > 4) return fail(QR_EINVAL, "qr_gather_ceiling: mode must be 0..4");
  if (mode == 4 && (h->layout != QR_LAYOUT_QUADRANK16))
    return fail(QR_EINVAL, "qr_gather_ceiling: mode 4 (rank_4 output shape) needs a QuadRank16 handle");
  if (mode == 3 && (h->sigma != 2 || !h->spack))
    return fail(QR_EINVAL, "qr_gather_ceiling: mode 3 needs a BiRank16 handle with a superblock cache");
  DeviceGuard dg(h->device);
  if (m && classify({q, out}, h->device) != 1) return fail(QR_EINVAL, "qr_gather_ceiling: device pointers only");
  cudaError_t e = mode == 3 ? launch_super_pack_rank(h, q, nullptr, out, m, 3, (cudaStream_t)stream)
                            : launch_gather(h, q, out, m, mode, (cudaStream_t)stream);
  return e ? cuda_fail(e, "qr_gather_ceiling launch") : QR_OK;
}

// Default k-mer table width: the paper's 8 for small texts; on B200 wider tables replace
// more backward steps by one lookup and HBM holds them easily: 10 (8 MiB) from n = 2^20, 12
// (128 MiB) from n = 2^24 — configs[3] 5.61 -> 6.57 G patterns/s, configs[4] 0.94 -> 0.99
// (profiles/r01_fm_k_probe*.jsonl).  Counts never depend on it.
// From n = 2^24 the width is 11 when the BWT's rank layout and the 32 MiB 11-mer table fit in
// 60% of the L2 together (the count kernel then seeds from L2, not HBM: configs[3] 9.14 -> 9.36
// G patterns/s with packed seeds, profiles/r02_fm_step_probe.jsonl), else 12.
int fm_default_kmer_k(uint64_t n, int layout, int device) {
  if (n < (1ull << 20)) return 8;
  if (n < (1ull << 24)) return 10;
  const uint64_t line_chars = layout == QR_LAYOUT_QUADRANK16X2 ? 192 : 224;
  const uint64_t bwt_bytes = ((n + 1) / line_chars + 1) * 64, t11 = (1ull << 22) * 8;
  return bwt_bytes + t11 <= (uint64_t)l2_bytes(device) * 6 / 10 ? 11 : 12;
}

QR_EXPORT qr_status qr_fm_build_ex(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k,
                                   int device, void* stream, qr_fm** out);

QR_EXPORT qr_status qr_fm_build(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int device,
                                void* stream, qr_fm** out) {
  return qr_fm_build_opts(text2b, n, sa_or_null, -1, QR_LAYOUT_QUADRANK16, device, stream, out);
}

QR_EXPORT qr_status qr_fm_build_opts(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k,
                                     int bwt_layout, int device, void* stream, qr_fm** out);

QR_EXPORT qr_status qr_fm_build_ex(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k,
                                   int device, void* stream, qr_fm** out) {
  return qr_fm_build_opts(text2b, n, sa_or_null, kmer_k, QR_LAYOUT_QUADRANK16, device, stream, out);
}

// one byte per symbol -> 2-bit LE words (char i = bits 2(i%32).. of word i/32); a byte > 3 sets *bad
__global__ void k_pack2(const uint8_t* __restrict__ t, uint64_t n, uint64_t* __restrict__ w, unsigned* __restrict__ bad) {
  const uint64_t nw = (n + 31) >> 5;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;
    unsigned b = 0;
    const uint64_t base = i << 5;
    const uint32_t cnt = n - base < 32 ? (uint32_t)(n - base) : 32u;
    for (uint32_t k = 0; k < cnt; ++k) {
      const uint32_t c = t[base + k];
      b |= c > 3u;
      v |= (uint64_t)(c & 3u) << (2 * k);
    }
    w[i] = v;
    if (b) atomicOr(bad, 1u);
  }
}

QR_EXPORT qr_status qr_fm_build_u8(const uint8_t* text, uint64_t n, const uint32_t* sa_or_null, int device,
                                   void* stream, qr_fm** out) {
  if (!out || !text) return fail(QR_EINVAL, "qr_fm_build_u8: null pointer");
  *out = nullptr;
  if (n == 0) return fail(QR_EINVAL, "qr_fm_build_u8: empty text");
  if (n + 1 >= (1ull << 32)) return fail(QR_ECAPACITY, "qr_fm_build_u8: n+1 >= 2^32 (u32 counts)");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_fm_build_u8: bad device %d", device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t words = (n + 31) >> 5;
  uint8_t* dt = nullptr;
  uint64_t* dw = nullptr;
  unsigned* dbad = nullptr;
  const bool dev_in = pointer_space(text, device) == 1;
  cudaError_t e = cudaSuccess;
  if (!dev_in) {
    if (!(e = cudaMalloc((void**)&dt, n))) e = cudaMemcpyAsync(dt, text, n, cudaMemcpyDefault, st);
  }
  if (!e) e = cudaMalloc((void**)&dw, (words + 1) * 8);
  if (!e) e = cudaMalloc((void**)&dbad, sizeof(unsigned));
  if (!e) e = cudaMemsetAsync(dbad, 0, sizeof(unsigned), st);
  if (!e) e = cudaMemsetAsync(dw + words, 0, 8, st);
  if (!e) {
    k_pack2<<<grid_stride_blocks(words, 256, sm_count(device), 8), 256, 0, st>>>(dev_in ? text : dt, n, dw, dbad);
    e = cudaGetLastError();
  }
  unsigned hbad = 0;
  if (!e) e = cudaMemcpyAsync(&hbad, dbad, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  if (!e) e = cudaStreamSynchronize(st);
  qr_status s = e ? cuda_fail(e, "qr_fm_build_u8") : hbad ? fail(QR_EINVAL, "qr_fm_build_u8: a symbol byte is > 3") : QR_OK;
  if (s == QR_OK) s = qr_fm_build_opts(dw, n, sa_or_null, -1, QR_LAYOUT_QUADRANK16, device, stream, out);
  cudaStreamSynchronize(st);
  cudaFree(dt); cudaFree(dw); cudaFree(dbad);
  return s;
}

QR_EXPORT qr_status qr_fm_build_opts(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k,
                                     int bwt_layout, int device, void* stream, qr_fm** out) {
  // The default width may pick 11 for the exact count (its table then sits in L2); the
  // approximate-search kernels enumerate every K-mer within k substitutions of the seed, where a
  // wider table saves more backtracking than HBM lookups cost: from n = 2^24 they get a 14-wide
  // table of their own (2 GiB), built on the first approximate call (fm.cu fm_params_ax).
  int kmer_k_ax = kmer_k;
  if (kmer_k == -1) {
    kmer_k = fm_default_kmer_k(n, bwt_layout, device);
    kmer_k_ax = n >= (1ull << 24) ? 14 : kmer_k;            // built on the first approximate call
  }
  if (kmer_k < 0 || kmer_k > 14) return fail(QR_EINVAL, "qr_fm_build_ex: kmer_k must be 0..14");
  if (bwt_layout != QR_LAYOUT_QUADRANK16 && bwt_layout != QR_LAYOUT_QUADRANK16X2)
    return fail(QR_EINVAL, "qr_fm_build_opts: bwt_layout must be QR_LAYOUT_QUADRANK16 or QR_LAYOUT_QUADRANK16X2");
  if (!out || !text2b) return fail(QR_EINVAL, "qr_fm_build: null pointer");
  *out = nullptr;
  if (n == 0) return fail(QR_EINVAL, "qr_fm_build: empty text");
  if (n + 1 >= (1ull << 32)) return fail(QR_ECAPACITY, "qr_fm_build: n+1 >= 2^32 (u32 counts)");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_fm_build: bad device %d", device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t words = (n + 31) >> 5;
  uint64_t* d = nullptr;
  qr_status s = stage_input(text2b, words, words + 1, st, &d);
  if (s != QR_OK) return s;
  // chars >= n are never read by the FM builder (SA keys, BWT and C stop at n)
  uint32_t* dsa = nullptr;
  if (sa_or_null) {
    cudaError_t e;
    if ((e = cudaMalloc((void**)&dsa, (n + 1) * 4))) { free_staged(d, st); return cuda_fail(e, "alloc sa"); }
    if ((e = cudaMemcpyAsync(dsa, sa_or_null, (n + 1) * 4, cudaMemcpyDefault, st))) {
      free_staged(d, st); free_staged(dsa, st); return cuda_fail(e, "copy sa");
    }
  }
  s = fm_build_device(d, n, dsa, device, st, out, kmer_k, bwt_layout, kmer_k_ax);
  cudaError_t e = free_staged(d, st);
  free_staged(dsa, st);
  if (!e) e = cudaStreamSynchronize(st);
  if (s == QR_OK && e) { qr_fm_free(*out); *out = nullptr; return cuda_fail(e, "qr_fm_build"); }
  return s;
}

static qr_status fm_count_impl(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                               uint32_t* out, uint32_t* out_rc, uint64_t m, uint64_t* work, void* stream,
                               int approx = 0) {
  if (!fm) return fail(QR_EINVAL, "qr_fm_count: null handle");
  if (m == 0) return QR_OK;
  if (!out || (!patterns && (lengths || fixed_len))) return fail(QR_EINVAL, "qr_fm_count: null pointer");
  DeviceGuard dg(fm->bwt->device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* pat = patterns;
  static const uint8_t dummy = 0;
  int sp = classify({patterns, lengths, out, out_rc, work}, fm->bwt->device);
  if (sp < 0) return fail(QR_EINVAL, "qr_fm_count: pointers must all be device (device %d) or all host", fm->bwt->device);
  if (sp == 1) return fm_count_device(fm, pat ? pat : &dummy, lengths, fixed_len, out, out_rc, m, work, st, approx);
  if (work) return fail(QR_EINVAL, "qr_fm_count_work: device pointers only");
  if (!lengths) {
    std::vector<StageArray> arr = {{patterns, nullptr, (size_t)fixed_len}, {nullptr, out, 4}};
    if (fixed_len == 0) arr[0].host_in = nullptr, arr[0].item_bytes = 1;
    if (out_rc) arr.push_back({nullptr, out_rc, 4});
    return run_staged(fm->bwt->device, st, m, arr, [&](const std::vector<void*>& d, uint64_t cnt, cudaStream_t s) {
      return fm_count_device(fm, (const uint8_t*)d[0], nullptr, fixed_len, (uint32_t*)d[1],
                             out_rc ? (uint32_t*)d[2] : nullptr, cnt, nullptr, s, approx);
    });
  }
  // variable lengths from host: chunks of <= 2^22 patterns and <= 256 MiB of symbols (one longer
  // pattern makes a chunk of its own), each copied, counted and copied back in order on `st`,
  // so device memory stays bounded whatever the batch
  constexpr uint64_t CHUNK_PATS = 1ull << 22, CHUNK_BYTES = 1ull << 28;
  uint64_t longest = 0;
  for (uint64_t i = 0; i < m; ++i) longest = lengths[i] > longest ? lengths[i] : longest;
  const uint64_t cap = longest > CHUNK_BYTES ? longest : CHUNK_BYTES;
  const uint64_t pc = m < CHUNK_PATS ? m : CHUNK_PATS;
  uint8_t* dp = nullptr;
  uint32_t *dl = nullptr, *dout = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&dp, cap + 8, st)) || (e = cudaMallocAsync((void**)&dl, pc * 4, st)) ||
      (e = cudaMallocAsync((void**)&dout, pc * 8, st))) {
    cudaFreeAsync(dp, st); cudaFreeAsync(dl, st); cudaFreeAsync(dout, st);
    return cuda_fail(e, "qr_fm_count: staging alloc");
  }
  qr_status s = QR_OK;
  uint64_t byte0 = 0;
  for (uint64_t lo = 0; lo < m && s == QR_OK;) {
    uint64_t hi = lo, bytes = 0;
    while (hi < m && hi - lo < CHUNK_PATS && (hi == lo || bytes + lengths[hi] <= cap)) bytes += lengths[hi++];
    const uint64_t cnt = hi - lo;
    if (bytes && (e = cudaMemcpyAsync(dp, patterns + byte0, bytes, cudaMemcpyHostToDevice, st))) {
      s = cuda_fail(e, "qr_fm_count: staged H2D");
      break;
    }
    if ((e = cudaMemcpyAsync(dl, lengths + lo, cnt * 4, cudaMemcpyHostToDevice, st))) {
      s = cuda_fail(e, "qr_fm_count: staged H2D");
      break;
    }
    s = fm_count_device(fm, dp, dl, 0, dout, out_rc ? dout + cnt : nullptr, cnt, nullptr, st, approx);
    if (s == QR_OK && (e = cudaMemcpyAsync(out + lo, dout, cnt * 4, cudaMemcpyDeviceToHost, st)))
      s = cuda_fail(e, "qr_fm_count: staged D2H");
    if (s == QR_OK && out_rc && (e = cudaMemcpyAsync(out_rc + lo, dout + cnt, cnt * 4, cudaMemcpyDeviceToHost, st)))
      s = cuda_fail(e, "qr_fm_count: staged D2H");
    byte0 += bytes;
    lo = hi;
  }
  cudaFreeAsync(dp, st); cudaFreeAsync(dl, st); cudaFreeAsync(dout, st);
  return s;
}

QR_EXPORT qr_status qr_fm_count(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                                uint32_t* out, uint64_t m, void* stream) {
  return fm_count_impl(fm, patterns, lengths, fixed_len, out, nullptr, m, nullptr, stream);
}

QR_EXPORT qr_status qr_fm_count_approx(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                       uint32_t fixed_len, uint32_t max_mismatches, uint32_t* out, uint64_t m,
                                       void* stream) {
  if (max_mismatches > 3) return fail(QR_EINVAL, "qr_fm_count_approx: max_mismatches must be 0..3");
  return fm_count_impl(fm, patterns, lengths, fixed_len, out, nullptr, m, nullptr, stream, (int)max_mismatches);
}

QR_EXPORT qr_status qr_fm_count_approx_both(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                            uint32_t fixed_len, uint32_t max_mismatches, uint32_t* out_fwd,
                                            uint32_t* out_rc, uint64_t m, void* stream) {
  if (max_mismatches > 3) return fail(QR_EINVAL, "qr_fm_count_approx_both: max_mismatches must be 0..3");
  if (!out_rc) return fail(QR_EINVAL, "qr_fm_count_approx_both: null out_rc");
  return fm_count_impl(fm, patterns, lengths, fixed_len, out_fwd, out_rc, m, nullptr, stream, (int)max_mismatches);
}

QR_EXPORT qr_status qr_fm_count_both(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                     uint32_t fixed_len, uint32_t* out_fwd, uint32_t* out_rc, uint64_t m, void* stream) {
  if (!out_rc) return fail(QR_EINVAL, "qr_fm_count_both: null out_rc");
  return fm_count_impl(fm, patterns, lengths, fixed_len, out_fwd, out_rc, m, nullptr, stream);
}

QR_EXPORT qr_status qr_fm_count_work(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                     uint32_t fixed_len, uint32_t* out, uint64_t m, uint64_t* work, void* stream) {
  if (!work) return fail(QR_EINVAL, "qr_fm_count_work: null work");
  return fm_count_impl(fm, patterns, lengths, fixed_len, out, nullptr, m, work, stream);
}

QR_EXPORT qr_status qr_fm_count_work_ex(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                        uint32_t fixed_len, uint32_t max_mismatches, uint32_t* out_fwd,
                                        uint32_t* out_rc, uint64_t m, uint64_t* work, void* stream) {
  if (!work) return fail(QR_EINVAL, "qr_fm_count_work_ex: null work");
  if (max_mismatches > 3) return fail(QR_EINVAL, "qr_fm_count_work_ex: max_mismatches must be 0..3");
  return fm_count_impl(fm, patterns, lengths, fixed_len, out_fwd, out_rc, m, work, stream, (int)max_mismatches);
}

QR_EXPORT qr_status qr_info(const qr_index* h, uint64_t* n, int* sigma, uint64_t* line_bytes, uint64_t* super_bytes) {
  if (!h) return fail(QR_EINVAL, "qr_info: null handle");
  if (n) *n = h->n;
  if (sigma) *sigma = h->sigma;
  if (line_bytes) *line_bytes = h->n_lines * 64;
  if (super_bytes) *super_bytes = super_bytes_of(h);
  return QR_OK;
}

QR_EXPORT qr_status qr_super_cache_bytes(const qr_index* h, uint64_t* cta_bytes) {
  if (!h || !cta_bytes) return fail(QR_EINVAL, "qr_super_cache_bytes: null pointer");
  *cta_bytes = super_pack_cta_bytes(h);
  return QR_OK;
}

QR_EXPORT qr_status qr_super_cache_clusters(const qr_index* h, int* clusters) {
  if (!h || !clusters) return fail(QR_EINVAL, "qr_super_cache_clusters: null pointer");
  DeviceGuard dg(h->device);
  *clusters = super_pack_clusters(h);
  return QR_OK;
}

QR_EXPORT qr_status qr_export_layout(const qr_index* h, void* host_lines, void* host_super) {
  if (!h) return fail(QR_EINVAL, "qr_export_layout: null handle");
  DeviceGuard dg(h->device);
  cudaError_t e;
  if (host_lines && (e = cudaMemcpy(host_lines, h->lines, h->n_lines * 64, cudaMemcpyDefault)))
    return cuda_fail(e, "qr_export_layout lines");
  if (host_super && super_bytes_of(h) &&
      (e = cudaMemcpy(host_super, h->super, super_bytes_of(h), cudaMemcpyDefault)))
    return cuda_fail(e, "qr_export_layout super");
  return QR_OK;
}

QR_EXPORT qr_status qr_import_layout(const void* lines, uint64_t line_bytes, const void* super, uint64_t super_bytes,
                                     uint64_t n, int layout, int device, void* stream, qr_index** out) {
  if (!out || !lines) return fail(QR_EINVAL, "qr_import_layout: null pointer");
  *out = nullptr;
  if (layout < QR_LAYOUT_BIRANK16 || layout > QR_LAYOUT_BIRANK32X2) return fail(QR_EINVAL, "qr_import_layout: bad layout");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_import_layout: bad device %d", device);
  const int sigma = (layout == QR_LAYOUT_BIRANK16 || layout == QR_LAYOUT_BIRANK64X2 || layout == QR_LAYOUT_BIRANK16X2 ||
                     layout == QR_LAYOUT_BIRANK32X2) ? 2 : 4;
  qr_index* h = nullptr;
  qr_status s = alloc_index(sigma, n, device, &h, layout);
  if (s != QR_OK) return s;
  if (super_bytes_of(h) && !super) { qr_free(h); return fail(QR_EINVAL, "qr_import_layout: layout needs a superblock array"); }
  if (line_bytes != h->n_lines * 64 || super_bytes != super_bytes_of(h)) {
    const uint64_t el = h->n_lines * 64, es = super_bytes_of(h);
    qr_free(h);
    return fail(QR_EINVAL, "qr_import_layout: buffer sizes (%llu, %llu) B differ from the layout's (%llu, %llu) B for n = %llu",
                (unsigned long long)line_bytes, (unsigned long long)super_bytes, (unsigned long long)el,
                (unsigned long long)es, (unsigned long long)n);
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(h->lines, lines, h->n_lines * 64, cudaMemcpyDefault, st);
  if (!e && super_bytes_of(h)) e = cudaMemcpyAsync(h->super, super, super_bytes_of(h), cudaMemcpyDefault, st);
  if (!e && (s = build_super_pack(h, st)) != QR_OK) { qr_free(h); return s; }
  if (!e) e = cudaStreamSynchronize(st);
  if (e) { qr_free(h); return cuda_fail(e, "qr_import_layout"); }
  *out = h;
  return QR_OK;
}

QR_EXPORT qr_status qr_fm_kmer_width(const qr_fm* fm, int* kmer_k) {
  if (!fm || !kmer_k) return fail(QR_EINVAL, "qr_fm_kmer_width: null pointer");
  *kmer_k = fm->kmer_k;
  return QR_OK;
}

QR_EXPORT qr_status qr_fm_info(const qr_fm* fm, uint64_t* n, uint64_t* spos, uint64_t C[5], const qr_index** bwt_rank) {
  if (!fm) return fail(QR_EINVAL, "qr_fm_info: null handle");
  if (n) *n = fm->n;
  if (spos) *spos = fm->spos;
  if (C) for (int c = 0; c < 5; ++c) C[c] = fm->C[c];
  if (bwt_rank) *bwt_rank = fm->bwt;
  return QR_OK;
}

QR_EXPORT qr_status qr_fm_export_kmer(const qr_fm* fm, uint32_t* host_pairs) {
  if (!fm || !host_pairs) return fail(QR_EINVAL, "qr_fm_export_kmer: null pointer");
  DeviceGuard dg(fm->bwt->device);
  cudaError_t e = cudaMemcpy(host_pairs, fm->kmer, kmer_entries(fm->kmer_k) * sizeof(uint2), cudaMemcpyDeviceToHost);
  return e ? cuda_fail(e, "qr_fm_export_kmer") : QR_OK;
}

QR_EXPORT qr_status qr_clone_to_device(const qr_index* h, int device, void* stream, qr_index** out) {
  if (!h || !out) return fail(QR_EINVAL, "qr_clone_to_device: null pointer");
  *out = nullptr;
  DeviceGuard dg(device);
  if (!dg.ok) return fail(QR_EINVAL, "qr_clone_to_device: bad device %d", device);
  qr_index* c = nullptr;
  qr_status s = alloc_index(h->sigma, h->n, device, &c, h->layout);
  if (s != QR_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  int can = 0;
  if (device != h->device) cudaDeviceCanAccessPeer(&can, device, h->device);
  if (can) cudaDeviceEnablePeerAccess(h->device, 0), cudaGetLastError();
  cudaError_t e = cudaMemcpyPeerAsync(c->lines, device, h->lines, h->device, h->n_lines * 64, st);
  if (!e && super_bytes_of(h)) e = cudaMemcpyPeerAsync(c->super, device, h->super, h->device, super_bytes_of(h), st);
  if (!e && (s = build_super_pack(c, st)) != QR_OK) { qr_free(c); return s; }
  if (!e) e = cudaStreamSynchronize(st);
  if (e) { qr_free(c); return cuda_fail(e, "qr_clone_to_device"); }
  *out = c;
  return QR_OK;
}

QR_EXPORT qr_status qr_fm_clone_to_device(const qr_fm* fm, int device, void* stream, qr_fm** out) {
  if (!fm || !out) return fail(QR_EINVAL, "qr_fm_clone_to_device: null pointer");
  *out = nullptr;
  qr_fm* c = new (std::nothrow) qr_fm();
  if (c) fm_copy_locked(fm, c);                            // consistent with a concurrent lazy build
  if (!c) return fail(QR_ENOMEM, "host allocation");
  c->bwt = nullptr;
  c->kmer = nullptr;
  c->kmer_ax = nullptr;
  c->kmer_bits = nullptr;                                  // rebuilt by the clone's first approximate call
  c->kmer_bits_k = 0;
  qr_status s = qr_clone_to_device(fm->bwt, device, stream, &c->bwt);
  if (s != QR_OK) { delete c; return s; }
  DeviceGuard dg(device);
  const size_t kb = (kmer_c_offset(fm->kmer_k) + 2) * sizeof(uint2);       // table + C[0..3] tail
  cudaError_t e = cudaMalloc((void**)&c->kmer, kb);
  if (!e) e = cudaMemcpyPeerAsync(c->kmer, device, fm->kmer, fm->bwt->device, kb, (cudaStream_t)stream);
  if (fm->kmer_ax == fm->kmer) {
    c->kmer_ax = c->kmer;                                  // the clone builds a wider table itself
    c->kmer_k_ax = c->kmer_k;
  } else {
    const size_t kx = kmer_entries(fm->kmer_k_ax) * sizeof(uint2);
    if (!e) e = cudaMalloc((void**)&c->kmer_ax, kx);
    if (!e) e = cudaMemcpyPeerAsync(c->kmer_ax, device, fm->kmer_ax, fm->bwt->device, kx, (cudaStream_t)stream);
  }
  if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e) { qr_fm_free(c); return cuda_fail(e, "qr_fm_clone_to_device"); }
  *out = c;
  return QR_OK;
}

QR_EXPORT qr_status qr_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (!e) e = cudaGetLastError();
  return e ? cuda_fail(e, "qr_sync") : QR_OK;
}

QR_EXPORT void qr_free(qr_index* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  if (h->lines) cudaFree(h->lines);
  if (h->super) cudaFree(h->super);
  if (h->spack) cudaFree(h->spack);
  if (h->spack_big) cudaFree(h->spack_big);
  delete h;
}

QR_EXPORT void qr_fm_free(qr_fm* fm) {
  if (!fm) return;
  if (fm->bwt) {
    DeviceGuard dg(fm->bwt->device);
    if (fm->kmer_ax && fm->kmer_ax != fm->kmer) cudaFree(fm->kmer_ax);
    if (fm->kmer_bits) cudaFree(fm->kmer_bits);
    if (fm->kmer) cudaFree(fm->kmer);
    qr_free(fm->bwt);
  }
  delete fm;
}
