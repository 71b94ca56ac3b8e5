// tma_probe.cu — does a TMA (cp.async.bulk) random gather sustain more 64-B line fetches per
// second than LDG gathers on B200?  (measurement tool, not product code)
//   kernel 0: LDG, lane pairs load the two 32-B sectors of a random 64-B line (one request)
//   kernel 1: cp.async.bulk global->shared of the random 64-B line, NSTAGE batches of 32 lines
//             in flight per warp, mbarrier complete_tx; the line is then read from shared memory
// Addresses are hash-generated (no dependent index load).  out[i] = xor of the line's words.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_ldg_pair(const char* __restrict__ buf, uint64_t nlines, uint64_t m, uint64_t seed, uint64_t* out) {
  const uint64_t npair = ((uint64_t)gridDim.x * blockDim.x) >> 1;
  const uint32_t half = threadIdx.x & 1u;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (uint64_t i0 = tid >> 1; i0 < m; i0 += npair * 4) {
    uint64_t a[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t idx = i0 + k * npair;
      const uint64_t line = __umul64hi(mix(seed ^ (idx * 0x9E3779B97F4A7C15ull)), nlines);
      const char* p = buf + line * 64 + 32 * half;
      asm volatile("ld.global.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(a[k][0]), "=l"(a[k][1]), "=l"(a[k][2]), "=l"(a[k][3]) : "l"(p));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t idx = i0 + k * npair;
      uint64_t v = a[k][0] ^ a[k][1] ^ a[k][2] ^ a[k][3];
      v ^= __shfl_xor_sync(0xffffffffu, v, 1);
      if (half == 0 && idx < m) out[idx] = v;
    }
  }
}

template <int NSTAGE>
__global__ void __launch_bounds__(256) k_tma(const char* __restrict__ buf, uint64_t nlines, uint64_t m, uint64_t seed,
                                              uint64_t* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  unsigned char* wbuf = smem + (size_t)warp * NSTAGE * 32 * 64;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwarps * NSTAGE * 32 * 64) + warp * NSTAGE;
  if (lane == 0)
    for (int s = 0; s < NSTAGE; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(bars + s);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t gw = (blockIdx.x * (uint64_t)nwarps + warp);
  const uint64_t nw = (uint64_t)gridDim.x * nwarps;
  const uint64_t nbatch = (m + 31) / 32;
  uint32_t phase[NSTAGE];
  for (int s = 0; s < NSTAGE; ++s) phase[s] = 0;
  // issue helper
  auto issue = [&](uint64_t b, int s) {
    const uint64_t idx = b * 32 + lane;
    const uint64_t line = __umul64hi(mix(seed ^ (idx * 0x9E3779B97F4A7C15ull)), nlines);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + s);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(32 * 64) : "memory");
    __syncwarp();
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(wbuf + (s * 32 + lane) * 64);
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];"
                 ::"r"(dst), "l"(buf + line * 64), "r"(bar) : "memory");
  };
  uint64_t b_issue = gw, b_done = gw;
  int s_issue = 0, s_done = 0;
  for (int s = 0; s < NSTAGE && b_issue < nbatch; ++s, b_issue += nw) { issue(b_issue, s_issue); s_issue = (s_issue + 1) % NSTAGE; }
  while (b_done < nbatch) {
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + s_done);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(bar), "r"(phase[s_done]) : "memory");
    }
    phase[s_done] ^= 1u;
    const uint64_t* ln = reinterpret_cast<const uint64_t*>(wbuf + (s_done * 32 + lane) * 64);
    uint64_t v = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) v ^= ln[t];
    const uint64_t idx = b_done * 32 + lane;
    if (idx < m) out[idx] = v;
    __syncwarp();
    b_done += nw;
    if (b_issue < nbatch) { issue(b_issue, s_done); b_issue += nw; }
    s_done = (s_done + 1) % NSTAGE;
  }
}

template <int NS>
float run_tma(const char* buf, uint64_t nlines, uint64_t m, uint64_t* out, int blocks_per_sm) {
  const int threads = 256;
  size_t smem = (size_t)(threads / 32) * NS * 32 * 64 + (threads / 32) * NS * 8;
  cudaFuncSetAttribute(k_tma<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int blocks = 148 * blocks_per_sm;
  k_tma<NS><<<blocks, threads, smem>>>(buf, nlines, m, 1, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_tma<NS><<<blocks, threads, smem>>>(buf, nlines, m, 2 + r, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err) printf("tma err %s\n", cudaGetErrorString(err));
  return ms / 3;
}

int main(int argc, char** argv) {
  uint64_t bytes = argc > 1 ? strtoull(argv[1], 0, 0) : (2ull << 30);
  uint64_t m = argc > 2 ? strtoull(argv[2], 0, 0) : 400000000ull;
  char* buf;
  uint64_t* out;
  if (cudaMalloc(&buf, bytes) || cudaMalloc(&out, m * 8)) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, bytes);
  const uint64_t nlines = bytes / 64;
  {
    int blocks = 148 * 32;
    k_ldg_pair<<<blocks, 256>>>(buf, nlines, m, 1, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) k_ldg_pair<<<blocks, 256>>>(buf, nlines, m, 2 + r, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"ldg_pair\", \"ms\": %.3f, \"G_lines_s\": %.2f}\n", ms / 3, m / (ms / 3) / 1e6);
  }
  for (int bps : {1, 2, 3}) {
    float t2 = run_tma<2>(buf, nlines, m, out, bps);
    float t4 = run_tma<4>(buf, nlines, m, out, bps);
    float t8 = run_tma<8>(buf, nlines, m, out, bps);
    printf("{\"kernel\": \"tma\", \"blocks_per_sm\": %d, \"G_lines_s_ns2\": %.2f, \"ns4\": %.2f, \"ns8\": %.2f}\n", bps,
           m / t2 / 1e6, m / t4 / 1e6, m / t8 / 1e6);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
