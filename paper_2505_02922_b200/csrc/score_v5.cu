// score_v5.cu -- the centroid scan of the decode step (ranking scores of
// index.py:61-76, approximate; select_v6 makes the selection exact).
//
// The scan of all m centroids per (unit, step) is the dominant byte stream of
// the decode step; it reads the fp32 copy C32 of the fp64 centroids.
#include "common.cuh"
#include "decode_internal.h"

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
