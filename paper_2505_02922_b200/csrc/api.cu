// api.cu -- the function-level half of the drop-in boundary, in fp64 on the
// device: tierkv's attention partials / merge / oracle (attention.py:55-148),
// rank_clusters (index.py:61-76), top_k_token_ids (metrics.py:8-16),
// finalize_cluster's centroid and value sums (index.py:43-58) and the
// BlockCache phases lookup / assemble / commit_update (block_cache.py:79-213)
// as separately callable steps.  The batched decode path does not use these
// entry points (it runs the fused kernels of abi.cu); they back the per-call
// Python API that tierkv's own tests exercise.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "exact_select.cuh"
#include "cache_internal.h"

namespace wk {

constexpr int kApiThreads = 256;

WK_DEVINL double block_max_f64(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x >> 5); i++) r = fmax(r, red[i]);
  return r;
}

WK_DEVINL double block_sum_f64(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); i++) r += red[i];
  return r;
}

// One streaming-softmax partial (attention.py:67-112), one CTA.
//   mode 0 exact_partial:          s_j = (K_j . q) / sqrt(d), den = sum w, num = w @ V
//   mode 1 estimate_partial:       s_i = (C_i . q | scores_i) / sqrt(d), den = sum size_i w_i,
//                                  num = w @ VS
//   mode 2 tail_denominator_partial: as 1 with a zero numerator
// out[0] = running_max, out[1] = denominator, out[2] = count, out[3..3+d) = numerator.
// scratch: n doubles (the scaled scores, then the weights).
__global__ void api_partial_kernel(const double* __restrict__ q, const double* __restrict__ rows,
                                   const double* __restrict__ vals, const double* __restrict__ sizes,
                                   const double* __restrict__ scores, int n, int d, int mode, int blas_threads,
                                   double* __restrict__ s, double* __restrict__ out) {
  __shared__ double red[32];
  const double sq = sqrt((double)d);
  if (scores) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) s[j] = scores[j];
  } else {
    xs_score_rows(rows, q, n, d, blas_threads, s);  // dgemv recipe (index.py:74)
  }
  __syncthreads();
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double v = s[j] / sq;
    s[j] = v;
    mx = fmax(mx, v);
  }
  mx = block_max_f64(mx, red);
  double den = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double w = exp(s[j] - mx);
    s[j] = w;
    den += (mode == 0) ? w : sizes[j] * w;
  }
  den = block_sum_f64(den, red);
  __syncthreads();
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double acc = 0.0;
    if (mode != 2)
      for (int j = 0; j < n; j++) acc = __fma_rn(s[j], vals[(size_t)j * d + t], acc);
    out[3 + t] = acc;
  }
  if (threadIdx.x == 0) {
    out[0] = mx;
    out[1] = den;
    out[2] = (double)n;
  }
}

// merge / merged_sums (attention.py:115-148): parts [P, 3 + d] as written by
// api_partial_kernel.  out[0..d) = output, out[d] = coverage, out[d+1] =
// log_denominator, out[d+2] = merged denominator, out[d+3..2d+3) = merged
// numerator (merged_sums).  exact_mask (optional) marks the exact partials.
__global__ void api_merge_kernel(const double* __restrict__ parts, int P, int d, const uint8_t* __restrict__ exact_mask,
                                 double* __restrict__ out, int* status) {
  const int W = 3 + d;
  // exact_mask[p]: 0 zone partial, 1 exact zone partial, 2 exact partial that
  // only counts toward the coverage numerator (not merged into the output)
  auto merged = [&](int p) { return parts[(size_t)p * W + 2] > 0 && !(exact_mask && exact_mask[p] == 2); };
  double g = -INFINITY;
  int live = 0;
  for (int p = 0; p < P; p++)
    if (merged(p)) { g = fmax(g, parts[(size_t)p * W]); live++; }
  if (!live) {
    if (threadIdx.x == 0) set_status(status, kErrEmptyMerge);
    return;
  }
  double den = 0.0, ex = 0.0;
  for (int p = 0; p < P; p++) {
    const double* pp = parts + (size_t)p * W;
    if (pp[2] <= 0) continue;
    const double sc = exp(pp[0] - g);
    if (merged(p)) den += pp[1] * sc;
    if (exact_mask && exact_mask[p]) ex += pp[1] * sc;
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double num = 0.0;
    for (int p = 0; p < P; p++) {
      const double* pp = parts + (size_t)p * W;
      if (!merged(p)) continue;
      num += pp[3 + t] * exp(pp[0] - g);
    }
    out[t] = num / den;
    out[d + 3 + t] = num;
  }
  if (threadIdx.x == 0) {
    out[d] = exact_mask ? (den > 0 ? ex / den : 0.0) : 1.0;
    out[d + 1] = g + log(den);
    out[d + 2] = den;
  }
}

// rank_clusters / top_k_token_ids: exact dgemv-recipe scores of m rows, then
// the full lexsort((arange(m), -scores)) order by counting: the rank of row i
// is the number of rows j with (key_j, j) < (key_i, i), key = xs_key(score).
__global__ void api_scores_kernel(const double* __restrict__ q, const double* __restrict__ rows, int m, int d,
                                  int blas_threads, double* __restrict__ scores) {
  // each CTA scores a contiguous block of rows (8 rows per warp per pass)
  const int per = (m + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(m, r0 + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b0 = r0 + warp * 8; b0 < r1; b0 += nw * 8) {
    const int c = b0 + (lane >> 2);
    const bool act = c < r1;
    const int cls = act ? gemv_row_class(c, m, d, blas_threads) : 0;
    const double v = xs_exact_quad(rows + (size_t)(act ? c : 0) * d, q, d, cls, act);
    if (act && (lane & 3) == 0) scores[c] = v;
  }
}

__global__ void api_rank_kernel(const double* __restrict__ scores, int m, int64_t* __restrict__ order) {
  __shared__ unsigned long long tk[2048];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long ki = i < m ? xs_key(scores[i]) : 0ull;
  int rank = 0;
  for (int j0 = 0; j0 < m; j0 += 2048) {
    const int nj = min(2048, m - j0);
    __syncthreads();
    for (int j = threadIdx.x; j < nj; j += blockDim.x) tk[j] = xs_key(scores[j0 + j]);
    __syncthreads();
    if (i < m)
      for (int j = 0; j < nj; j++) {
        const unsigned long long kj = tk[j];
        rank += (kj < ki) || (kj == ki && j0 + j < i);
      }
  }
  if (i < m) order[rank] = i;
}

// finalize_cluster (index.py:43-58): per cluster, fp64 sequential sums of the
// members' fp32 keys / values in member order; centroid = sum / size.
__global__ void api_cluster_sums_kernel(const float* __restrict__ keys, const float* __restrict__ vals,
                                        const int32_t* __restrict__ members, const int32_t* __restrict__ offsets,
                                        int d, double* __restrict__ C, double* __restrict__ VS) {
  const int c = blockIdx.x;
  const int o = offsets[c], s = offsets[c + 1] - o;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double kc = 0.0, vc = 0.0;
    for (int j = 0; j < s; j++) {
      const size_t r = (size_t)members[o + j] * d + t;
      kc += (double)keys[r];
      vc += (double)vals[r];
    }
    C[(size_t)c * d + t] = kc / (double)s;
    VS[(size_t)c * d + t] = vc;
  }
}

}  // namespace wk

using namespace wk;

#define API_CHECK()                                \
  do {                                             \
    if (cudaGetLastError() != cudaSuccess) return WK_ECUDA; \
  } while (0)

extern "C" {

int wk_attn_partial_f64(const double* q, const double* rows, const double* vals, const double* sizes,
                        const double* scores, int n, int d, int mode, int blas_threads, double* scratch,
                        double* out, void* stream) {
  if (!q || !out || !scratch || n < 1 || d < 1 || mode < 0 || mode > 2) return WK_ECONFIG;
  if (!scores && !rows) return WK_ECONFIG;
  if (mode != 2 && !vals) return WK_ECONFIG;
  if (mode != 0 && !sizes) return WK_ECONFIG;
  api_partial_kernel<<<1, kApiThreads, 0, (cudaStream_t)stream>>>(q, rows, vals, sizes, scores, n, d, mode,
                                                                   blas_threads < 1 ? 1 : blas_threads, scratch, out);
  API_CHECK();
  return 0;
}

int wk_merge_f64(const double* parts, int P, int d, const uint8_t* exact_mask, double* out, int* status,
                 void* stream) {
  if (!parts || !out || P < 1 || d < 1) return WK_ECONFIG;
  api_merge_kernel<<<1, kApiThreads, 0, (cudaStream_t)stream>>>(parts, P, d, exact_mask, out, status);
  API_CHECK();
  return 0;
}

int wk_rank_f64(const double* q, const double* rows, int m, int d, int blas_threads, double* scores,
                int64_t* order, void* stream) {
  if (!q || !rows || !scores || m < 1 || d < 1) return WK_ECONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = (m + 255) / 256;
  api_scores_kernel<<<grid, 256, 0, s>>>(q, rows, m, d, blas_threads < 1 ? 1 : blas_threads, scores);
  API_CHECK();
  if (order) {
    api_rank_kernel<<<grid, 256, 0, s>>>(scores, m, order);
    API_CHECK();
  }
  return 0;
}

int wk_cluster_sums_f64(const float* keys, const float* values, const int32_t* members, const int32_t* offsets,
                        int k, int d, double* centroids, double* value_sums, void* stream) {
  if (!keys || !values || !members || !offsets || !centroids || !value_sums || k < 1 || d < 1) return WK_ECONFIG;
  api_cluster_sums_kernel<<<k, d < 128 ? 128 : 256, 0, (cudaStream_t)stream>>>(keys, values, members, offsets, d,
                                                                               centroids, value_sums);
  API_CHECK();
  return 0;
}

}  // extern "C"
