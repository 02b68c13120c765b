// score_v4.cu -- centroid scoring on tensor cores (ranking scores of
// index.py:61-76, approximate; select_v6 makes the selection exact).
//
// The scan of all m centroids per (unit, step) is the dominant byte stream of
// the decode step.  It reads C16 = fp16(C * 2^kc) (row scale Cscale = 2^-kc,
// a power of two so max|C16 row| is in [2^14, 2^15)): half the bytes of fp32.
// q is split per head into fp16 hi + lo (q * 2^kq = hi + lo + O(2^-22)), so a
// column pair (hi, lo) of the B operand carries one head.  One
// mma.sync.m16n8k16 (fp16 x fp16 -> fp32) per 16 centroid rows x 16 dims x
// 4 heads; G <= 8 uses two n-tiles.
//
// C16 is stored FRAGMENT-NATIVE: per 16-row tile and k-step s, lane l's four
// A-fragment registers are 16 contiguous bytes at ((tile*KS + s)*32 + l)*16,
// so every k-step is ONE fully coalesced 512-byte warp load (LDG.128) with no
// shared-memory staging.  The error bound of this mode (score_error_bound_v2
// mode 2) is what select_v6 uses for its exact band.
#include <cuda_fp16.h>

#include "common.cuh"
#include "decode_internal.h"

namespace wk {

WK_DEVINL void mma16816(float (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// power-of-two exponent k with max|x| * 2^k in [2^14, 2^15) (0 for a zero row)
WK_DEVINL int c16_exp(float amax) {
  if (!(amax > 0.f)) return 0;
  int e;
  frexpf(amax, &e);  // amax in [2^(e-1), 2^e)
  return 15 - e;
}

// ---------------------------------------------------------------------------
// pack: C64 rows [cid_base, cid_base + k) of each segment -> C16 tiles,
// Cscale, and the unit's max centroid norm (Cmax, for the error bound)
// ---------------------------------------------------------------------------
__global__ void km_pack16_kernel(const SegDesc* __restrict__ segs, IndexView ix, int d) {
  const SegDesc sg = segs[blockIdx.x];
  const int u = sg.unit, KS = d / 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __half* C16 = reinterpret_cast<__half*>(ix.C16) + (size_t)u * ix.m_cap * d;
  for (int c = warp; c < sg.k; c += nw) {
    const int r = sg.cid_base + c;
    const size_t row = (size_t)u * ix.m_cap + r;
    const double* src = ix.C64 + row * d;
    double dmax = 0.0;
    for (int i = lane; i < d; i += 32) dmax = fmax(dmax, fabs(src[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    int kc = 0;
    if (dmax > 0.0) { int e; frexp(dmax, &e); kc = 15 - e; }
    const int tile = r >> 4, rr = r & 15, g = rr & 7, upper = rr >> 3;
    for (int i = lane; i < d; i += 32) {
      const int s = i >> 4, cc = i & 15, t = (cc & 7) >> 1, kh = cc >> 3, lo = cc & 1;
      const int reg = kh * 2 + upper, ln = g * 4 + t;
      const size_t off = ((((size_t)tile * KS + s) * 32 + ln) * 4 + reg) * 2 + lo;
      C16[off] = __double2half(ldexp(src[i], kc));
    }
    if (lane == 0) {
      ix.Cscale[row] = ldexpf(1.f, -kc);
      const float nrm = ix.Cnorm[row];
      atomicMax(reinterpret_cast<int*>(ix.Cmax + u), __float_as_int(nrm));  // nrm >= 0
    }
  }
}

// ---------------------------------------------------------------------------
// score: grid (ceil(max tiles / tiles_per_cta), U), 128 threads; each warp
// streams tiles t0 + warp, t0 + warp + 4, ... with a one-tile register prefetch
// ---------------------------------------------------------------------------
template <int KS, int NT>
__global__ void __launch_bounds__(128) score_v4_kernel(IndexView ix, StepView sv, int G, int tiles_per_cta) {
  constexpr int D = KS * 16;
  const int u = blockIdx.y;
  const int m = sv.m[u];
  const int ntile = (m + 15) >> 4;
  const int t0 = blockIdx.x * tiles_per_cta;
  if (t0 >= ntile) return;
  const int t1 = min(ntile, t0 + tiles_per_cta);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  __shared__ float qs[8 * D];
  __shared__ int qk[8];
  for (int i = threadIdx.x; i < 8 * D; i += blockDim.x) {
    const int h = i / D;
    qs[i] = h < G ? sv.q[((size_t)u * G + h) * D + (i % D)] : 0.f;
  }
  __syncthreads();
  // per-head exponent (warp w handles heads w and w + 4)
  for (int h = warp; h < 8; h += 4) {
    float a = 0.f;
    for (int i = lane; i < D; i += 32) a = fmaxf(a, fabsf(qs[h * D + i]));
    a = warp_max(a);
    if (lane == 0) qk[h] = c16_exp(a);
  }
  __syncthreads();
  // B fragments: column n = gq of n-tile j -> head 4j + gq/2, split gq&1
  uint32_t bq[NT][KS][2];
#pragma unroll
  for (int j = 0; j < NT; j++) {
    const int h = 4 * j + (gq >> 1), split = gq & 1;
    const float sc = ldexpf(1.f, qk[h]);
#pragma unroll
    for (int s = 0; s < KS; s++) {
      __half hv[4];
      const int kk[4] = {16 * s + 2 * tq, 16 * s + 2 * tq + 1, 16 * s + 2 * tq + 8, 16 * s + 2 * tq + 9};
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const float x = qs[h * D + kk[e]] * sc;  // exact (power of two)
        const __half hi = __float2half_rn(x);
        hv[e] = split ? __float2half_rn(x - __half2float(hi)) : hi;
      }
      bq[j][s][0] = (uint32_t)__half_as_ushort(hv[0]) | ((uint32_t)__half_as_ushort(hv[1]) << 16);
      bq[j][s][1] = (uint32_t)__half_as_ushort(hv[2]) | ((uint32_t)__half_as_ushort(hv[3]) << 16);
    }
  }
  float qinv[NT];
#pragma unroll
  for (int j = 0; j < NT; j++) qinv[j] = ldexpf(1.f, -qk[4 * j + tq]);
  const uint4* Cb = reinterpret_cast<const uint4*>(ix.C16) + (size_t)u * (ix.m_cap / 16) * KS * 32;
  const float* csc = ix.Cscale + (size_t)u * ix.m_cap;
  float* out = sv.scores + (size_t)u * G * ix.m_cap;
  auto load = [&](uint4 (&a)[KS], int tl) {
#pragma unroll
    for (int s = 0; s < KS; s++) a[s] = __ldcs(Cb + ((size_t)tl * KS + s) * 32 + lane);
  };
  auto proc = [&](const uint4 (&a)[KS], int tl) {
    float c[NT][4];
#pragma unroll
    for (int j = 0; j < NT; j++) {
      c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
#pragma unroll
      for (int s = 0; s < KS; s++) mma16816(c[j], a[s], bq[j][s][0], bq[j][s][1]);
    }
    const int r0 = tl * 16 + gq, r1 = r0 + 8;
    const float s0 = r0 < m ? __ldg(csc + r0) : 0.f, s1 = r1 < m ? __ldg(csc + r1) : 0.f;
#pragma unroll
    for (int j = 0; j < NT; j++) {
      const int h = 4 * j + tq;
      if (h < G) {
        if (r0 < m) out[(size_t)h * ix.m_cap + r0] = (c[j][0] + c[j][1]) * s0 * qinv[j];
        if (r1 < m) out[(size_t)h * ix.m_cap + r1] = (c[j][2] + c[j][3]) * s1 * qinv[j];
      }
    }
  };
  uint4 a0[KS], a1[KS];
  int tl = t0 + warp;
  if (tl < t1) load(a0, tl);
  while (tl < t1) {
    int tn = tl + 4;
    if (tn < t1) load(a1, tn);
    proc(a0, tl);
    tl = tn;
    if (tl >= t1) break;
    tn = tl + 4;
    if (tn < t1) load(a0, tn);
    proc(a1, tl);
    tl = tn;
  }
}

template __global__ void score_v4_kernel<8, 1>(IndexView, StepView, int, int);
template __global__ void score_v4_kernel<8, 2>(IndexView, StepView, int, int);
template __global__ void score_v4_kernel<4, 1>(IndexView, StepView, int, int);
template __global__ void score_v4_kernel<4, 2>(IndexView, StepView, int, int);

}  // namespace wk

namespace wk {

// ---------------------------------------------------------------------------
// score_v5: the exact-precision scan on FP64 tensor cores.
//
// mma.sync.m8n8k4.f64: A = 8 centroid rows x 4 dims (fp32 C32 rows widened
// to fp64 -- exact), B = 4 dims x 8 heads (q in fp64), D = 8 rows x 8 heads
// accumulated in fp64, so |s' - s| is the C32 rounding of C64 plus the final
// fp32 store (score_error_bound_v2 mode 1), the same bound as the fp64 FMA
// scan, with ~5x fewer instructions and no shuffle reduction.
// The dot's k order is free (fp64 accumulation error is inside the bound),
// so k-step s uses dim pi(s, t) = 16 (s / 4) + 4 t + s % 4: lane (g, t) feeds
// four consecutive k-steps from ONE coalesced 16-byte load of row g.
// ---------------------------------------------------------------------------
WK_DEVINL void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int KG>  // KG = d / 16 load groups of 4 k-steps
__global__ void __launch_bounds__(128, 8) score_v5_kernel(IndexView ix, StepView sv, int G, int groups_per_warp) {
  constexpr int D = KG * 16;
  pdl_wait();
  const int u = blockIdx.y;
  const int m = sv.m[u];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ngroups = (m + 7) >> 3;
  // B fragments in smem: bq[s][lane] = q[head g][pi(s, t)] (zero for heads >= G)
  __shared__ double bq[KG * 4][32];
  {
    const int l = threadIdx.x & 31;
    const int gg = l >> 2, tt = l & 3;
    const float* qh = sv.q + ((size_t)u * G + (gg < G ? gg : 0)) * D;
    for (int j = threadIdx.x >> 5; j < KG; j += 4) {
      const float4 v = gg < G ? __ldg(reinterpret_cast<const float4*>(qh + 16 * j + 4 * tt))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      bq[4 * j][l] = (double)v.x; bq[4 * j + 1][l] = (double)v.y;
      bq[4 * j + 2][l] = (double)v.z; bq[4 * j + 3][l] = (double)v.w;
    }
  }
  __syncthreads();
  const int g0 = (blockIdx.x * 4 + warp) * groups_per_warp;
  if (g0 >= ngroups) return;
  const int g1 = min(ngroups, g0 + groups_per_warp);
  const float* Cb = ix.C32 + (size_t)u * ix.m_cap * D;
  float* out = sv.scores + (size_t)u * G * ix.m_cap;
  // one register buffer per warp, refilled slice by slice as it is consumed:
  // the next group's loads are in flight while this group's DMMAs run
  float4 a[KG];
  auto src_of = [&](int grp) {
    const int row = grp * 8 + g;
    return reinterpret_cast<const float4*>(Cb + (size_t)(row < m ? row : m - 1) * D + 4 * t);
  };
  {
    const float4* src = src_of(g0);
#pragma unroll
    for (int j = 0; j < KG; j++) a[j] = __ldcs(src + 4 * j);
  }
  for (int grp = g0; grp < g1; grp++) {
    const bool more = grp + 1 < g1;
    const float4* nsrc = src_of(more ? grp + 1 : grp);
    double c[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < KG; j++) {
      const float4 v = a[j];
      if (more) a[j] = __ldcs(nsrc + 4 * j);
      dmma884(c, (double)v.x, bq[4 * j][lane]);
      dmma884(c, (double)v.y, bq[4 * j + 1][lane]);
      dmma884(c, (double)v.z, bq[4 * j + 2][lane]);
      dmma884(c, (double)v.w, bq[4 * j + 3][lane]);
    }
    const int row = grp * 8 + g;
    if (row < m) {
      const int h0 = 2 * t;
      if (h0 < G) out[(size_t)h0 * ix.m_cap + row] = (float)c[0];
      if (h0 + 1 < G) out[(size_t)(h0 + 1) * ix.m_cap + row] = (float)c[1];
    }
  }
  pdl_trigger<1>();
}

template __global__ void score_v5_kernel<8>(IndexView, StepView, int, int);
template __global__ void score_v5_kernel<4>(IndexView, StepView, int, int);

}  // namespace wk
