// Probe: cp.async.bulk (TMA 1-D) global->shared with a pinned host source.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const float* src, float* out, int n) {
  __shared__ __align__(128) float buf[2048];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(buf)), "l"(src), "r"(n * 4), "r"(sa(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i] * 2.f;
}
int main() {
  const int n = 2048;
  float *h, *d;
  cudaHostAlloc(&h, n * 4, cudaHostAllocDefault);
  for (int i = 0; i < n; i++) h[i] = (float)i;
  cudaMalloc(&d, n * 4);
  float* hd = nullptr;
  cudaHostGetDevicePointer(&hd, h, 0);
  printf("host %p devptr %p\n", (void*)h, (void*)hd);
  k<<<1, 256>>>(hd, d, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float* r = (float*)malloc(n * 4);
  cudaMemcpy(r, d, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; i++) bad += r[i] != 2.f * i;
  printf("mismatches %d (r[5]=%f)\n", bad, r[5]);
  // bandwidth of bulk reads from host: many CTAs
  return 0;
}
