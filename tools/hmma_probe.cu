// hmma_probe.cu -- latency and throughput of mma.sync.m16n8k16 bf16->fp32 (HMMA.16816)
// on sm_100a: one dependent chain per warp (latency) vs 8 independent chains
// (throughput), 1..16 warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_probe tools/hmma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(int iters, float* out, long long* cyc) {
  float c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  for (int warps : {1, 4, 8, 16}) {
    for (int ch : {1, 8}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (ch == 1) chains<1><<<148, warps * 32>>>(iters, out, cyc);
      else chains<8><<<148, warps * 32>>>(iters, out, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double mmas = (double)iters * ch;  // per warp
      const double flops = 148.0 * warps * mmas * 2 * 16 * 8 * 16;
      printf("warps/SM=%2d chains=%d: %.1f cycles per MMA per warp, %.1f TFLOP/s chip\n", warps, ch,
             (double)c / mmas, flops / (ms / 1e3) / 1e12);
    }
  }
  return 0;
}
