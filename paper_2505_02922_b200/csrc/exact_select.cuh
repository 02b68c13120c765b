// exact_select.cuh -- tie-safe exact selection (the fallback of every
// approximate-score selector: select_v6, select_kernel, recall_kernel).
//
// The reference orders with np.lexsort((ids, -scores)) on fp64 scores
// (index.py:75, metrics.py:15): score descending, ties to the lower id, and
// -0.0 == +0.0.  The fast selectors classify rows with approximate scores and
// an error band; when the band or a scratch list overflows -- dense ties, a
// zero query, identical centroids -- they fall back to this exact path:
// every row's exact fp64 score (the reference's dgemv recipe) is computed and
// a block-wide 96-bit radix select over (score key, id) finds the K-th element
// of the lexsort order.  Membership of the top K is then one comparison:
//   key < Tk  ||  (key == Tk && id <= Ti).
#pragma once
#include "common.cuh"

namespace wk {

// descending fp64 score -> ascending u64 key; -0.0 and +0.0 map to one key
WK_DEVINL unsigned long long xs_key(double s) {
  unsigned long long u = (unsigned long long)__double_as_longlong(s);
  if (s == 0.0) u = 0ull;
  u = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
  return ~u;
}

// exact dgemv-recipe score (index.py:74, OpenBLAS dgemv_t: DESIGN.md "Numerics
// recipes") of one row per lane quad: lane j of the quad runs accumulator
// chain j; returns the score on all 4 lanes.  All 32 lanes must call.
template <typename QT>
WK_DEVINL double xs_exact_quad(const double* __restrict__ row, const QT* __restrict__ q, int d, int cls,
                               bool act) {
  const int j = threadIdx.x & 3;
  double acc = 0.0;
  if (act) {
    if (cls == 0) {
      for (int t = j; t < d; t += 4) acc = __fma_rn(__ldcg(row + t), (double)q[t], acc);
    } else if (cls == 1) {
      if (j < 2)
        for (int t = j; t < d; t += 2) acc = __dadd_rn(acc, __dmul_rn(__ldcg(row + t), (double)q[t]));
    } else {
      for (int t = j; t < d; t += 4) acc = __dadd_rn(acc, __dmul_rn(__ldcg(row + t), (double)q[t]));
    }
  }
  const int base = (threadIdx.x & 31) & ~3;
  const double a0 = __shfl_sync(0xffffffffu, acc, base), a1 = __shfl_sync(0xffffffffu, acc, base + 1),
               a2 = __shfl_sync(0xffffffffu, acc, base + 2), a3 = __shfl_sync(0xffffffffu, acc, base + 3);
  if (cls == 1) return __dadd_rn(0.0, __dadd_rn(a0, a1));
  return __dadd_rn(0.0, __dadd_rn(__dadd_rn(a0, a2), __dadd_rn(a1, a3)));
}

// xs[c] = exact score of centroid row c, c in [0, m) (8 rows per warp)
template <typename QT>
WK_DEVINL void xs_score_rows(const double* __restrict__ C64, const QT* __restrict__ q, int m, int d,
                             int blas_threads, double* __restrict__ xs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b0 = warp * 8; b0 < m; b0 += nw * 8) {
    const int c = b0 + (lane >> 2);
    const bool act = c < m;
    const int cls = act ? gemv_row_class(c, m, d, blas_threads) : 0;
    const double v = xs_exact_quad(C64 + (size_t)(act ? c : 0) * d, q, d, cls, act);
    if (act && (lane & 3) == 0) xs[c] = v;
  }
}

// K-th element (1-based, 1 <= K <= n) of the ascending (key, id) order of n
// items.  key(i) -> u64, id(i) -> u32 (distinct ids).  hist: shared int[258].
// Every thread of the block calls; returns the element's (key, id) on all.
template <typename KeyF, typename IdF>
__device__ void xs_select(int n, int K, KeyF key, IdF id, int* hist, unsigned long long& Tk, unsigned& Ti) {
  unsigned long long kp = 0ull, km = 0ull;
  unsigned ip = 0u, im = 0u;
  int k = K;
  for (int pass = 0; pass < 12; pass++) {
    const bool on_key = pass < 8;
    const int shift = on_key ? 56 - 8 * pass : 24 - 8 * (pass - 8);
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long kk = key(i);
      if ((kk & km) != kp) continue;
      if (on_key) {
        atomicAdd(&hist[(int)((kk >> shift) & 255ull)], 1);
      } else {
        const unsigned ii = id(i);
        if ((ii & im) == ip) atomicAdd(&hist[(ii >> shift) & 255u], 1);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int h[8], s = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) { h[i] = hist[8 * lane + i]; s += h[i]; }
      int x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int below = x - s;
      if (below < k && x >= k) {
        int acc = below;
        for (int i = 0; i < 8; i++) {
          if (acc + h[i] >= k) { hist[256] = 8 * lane + i; hist[257] = k - acc; break; }
          acc += h[i];
        }
      }
    }
    __syncthreads();
    const int b = hist[256];
    k = hist[257];
    if (on_key) { kp |= (unsigned long long)b << shift; km |= 255ull << shift; }
    else { ip |= (unsigned)b << shift; im |= 255u << shift; }
  }
  Tk = kp;
  Ti = ip;
  __syncthreads();  // hist reusable
}

WK_DEVINL bool xs_in(unsigned long long kk, unsigned ii, unsigned long long Tk, unsigned Ti) {
  return kk < Tk || (kk == Tk && ii <= Ti);
}

}  // namespace wk
