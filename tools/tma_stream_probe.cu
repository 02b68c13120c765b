// tma_stream_probe.cu -- HBM read bandwidth of the attend_v5 staging pattern
// (per-warp private rings filled by 1-D bulk copies, consumer = the same warp)
// as a function of warps/CTA, stages, copy size and per-chunk compute delay.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream_probe tools/tma_stream_probe.cu
// Run:   tools/tma_stream_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(b) : "memory");
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// each warp streams `chunks` chunks of `cb` bytes (in `ncopy` copies each) from random-ish offsets
__global__ void probe(const unsigned char* src, size_t src_bytes, int W, int NST, int cb, int ncopy, int chunks,
                      int delay, unsigned long long* sink, int scatter) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = sm + (size_t)warp * NST * cb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)W * NST * cb) + warp * NST;
  if (lane == 0) {
    for (int i = 0; i < NST; i++) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const size_t gw = (size_t)blockIdx.x * W + warp;
  const size_t nchunk_total = src_bytes / cb;
  auto off = [&](int k) { return ((gw * 7919 + (size_t)k * 104729) % nchunk_total) * cb; };
  const int per = cb / ncopy;
  auto issue = [&](int k) {
    const int st = k % NST;
    if (lane == 0) expect_tx(bars + st, cb);
    __syncwarp();
    if (lane < ncopy) {
      // scatter: every copy from its own random row-aligned offset (a gathered row)
      const size_t o = scatter ? ((((gw * 131 + (size_t)k * 7919 + lane * 104729) * 2654435761ull) % (src_bytes / per)) * per)
                               : off(k) + lane * per;
      bulk(ring + st * cb + lane * per, src + o, per, bars + st);
    }
  };
  for (int k = 0; k < NST - 1 && k < chunks; k++) issue(k);
  unsigned long long acc = 0;
  for (int k = 0; k < chunks; k++) {
    if (k + NST - 1 < chunks) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      issue(k + NST - 1);
    }
    wait_bar(bars + (k % NST), (k / NST) & 1);
    acc += ring[(k % NST) * cb + lane * 4];
    for (int i = 0; i < delay; i++) acc = acc * 3 + 1;
    __syncwarp();
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  const size_t bytes = 8ull << 30;
  unsigned char* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct C { int W, NST, cb, ncopy, delay, scatter; };
  const C cs[] = {
      {12, 2, 8192, 2, 0, 0},  {12, 2, 8192, 2, 0, 1},  {12, 2, 8192, 16, 0, 1}, {12, 2, 8192, 32, 0, 1},
      {12, 2, 8192, 4, 0, 1},  {12, 2, 8192, 8, 0, 1},  {8, 3, 8192, 16, 0, 1},  {6, 4, 8192, 16, 0, 1},
      {12, 2, 8192, 16, 200, 1}, {4, 6, 8192, 16, 0, 1},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const C& c : cs) {
    const size_t smem = (size_t)c.W * c.NST * c.cb + c.W * c.NST * 8;
    if (smem > 227 * 1024) { printf("skip W=%d NST=%d cb=%d\n", c.W, c.NST, c.cb); continue; }
    const int chunks = (int)((3ull << 30) / ((size_t)sms * c.W * c.cb));
    probe<<<sms, c.W * 32, smem>>>(src, bytes, c.W, c.NST, c.cb, c.ncopy, chunks, c.delay, sink, c.scatter);
    cudaEventRecord(e0);
    probe<<<sms, c.W * 32, smem>>>(src, bytes, c.W, c.NST, c.cb, c.ncopy, chunks, c.delay, sink, c.scatter);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gb = (double)sms * c.W * chunks * c.cb / 1e9;
    printf("W=%2d NST=%2d chunk=%5d copies=%2d (%4d B, %s) delay=%4d: %7.1f GB/s  (%.3f ms)  err=%s\n", c.W, c.NST,
           c.cb, c.ncopy, c.cb / c.ncopy, c.scatter ? "scattered" : "contiguous", c.delay, gb / (ms / 1e3), ms,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
