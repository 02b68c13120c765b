// metrics.cu -- device recall@k (tierkv metrics.py:8-26, engine.py:200-203).
//
// recall = |top_k(q . K over every token) intersect retrieved| / k where the
// reference ranks tokens with an fp64 dgemv over keys[:n] (token order) and
// lexsort (-score, id).  Same exact-selection scheme as the zone planner:
// fp32 scores + rigorous bound, radix select of the k-th largest, exact fp64
// re-scoring of the boundary band with the dgemv recipe of the token's row.
// Not on the hot path (the reference computes it inside decode_step; the
// batched engine leaves it off).
#include "common.cuh"
#include "decode_internal.h"
#include "exact_select.cuh"

namespace wk {

struct RecallSmem {
  int bid[BAND_CAP];
  double bex[BAND_CAP];
  int hist[256];
  double q64[256];
  float red[32];
  int n_in, n_band, n_hit;
  unsigned int prefix;
  int krem;
  float fred;
};

template <typename T>
__device__ __forceinline__ void load_row_f64(const T* r, double* o, int d, long long row) {
  const bool swz = kv_swizzled<T>(d);
  for (int t = 0; t < d; t++) o[t] = (double)KV<T>::to_f(r[swz ? swz_col(t, row) : t]);
}

// grid = U*G, block = 512.  scratch: s [U*G, n_cap] f32, rflag [U*G, s_cap] u8.
template <typename T>
__global__ void __launch_bounds__(512) recall_kernel(IndexView ix, SteadyView st, StepView sv,
                                                     const int32_t* __restrict__ n_store, int G, int d,
                                                     int metrics_k, int blas_threads, float* __restrict__ s_all,
                                                     uint8_t* __restrict__ rflag_all, int64_t n_cap,
                                                     float* __restrict__ recall_out) {
  extern __shared__ __align__(16) unsigned char rc_raw[];
  RecallSmem& sm = *reinterpret_cast<RecallSmem*>(rc_raw);
  SelSmem& ssm = *reinterpret_cast<SelSmem*>(rc_raw + ((sizeof(RecallSmem) + 15) & ~size_t(15)));
  const int ug = blockIdx.x, u = ug / G, g = ug % G;
  const int ns = n_store[u], nt = st.n[u];
  const int n = ns + nt;
  const int K = metrics_k < n ? metrics_k : n;
  float* s = s_all + (int64_t)ug * n_cap;
  uint8_t* rf = rflag_all + (int64_t)ug * ix.s_cap;
  const float* q = sv.q + ((int64_t)u * G + g) * d;
  const T* sk = (const T*)ix.store_k + (int64_t)u * ix.s_cap * d;
  const T* stk = (const T*)st.k + (int64_t)u * st.t_cap * d;
  const int32_t* stok = ix.store_tok + (int64_t)u * ix.s_cap;
  const int32_t* sttok = st.tok + (int64_t)u * st.t_cap;
  const double* q64 = sv.q64 ? sv.q64 + ((int64_t)u * G + g) * d : nullptr;
  for (int t = threadIdx.x; t < d; t += blockDim.x) sm.q64[t] = q64 ? q64[t] : (double)q[t];
  // retrieved store rows: clusters of this head's retrieval list
  for (int i = threadIdx.x; i < ns; i += blockDim.x) rf[i] = 0;
  __syncthreads();
  const int r = sv.nr[u];
  const int32_t* rl = sv.rlist + ((int64_t)u * G + g) * sv.r_cap;
  for (int i = 0; i < r; i++) {
    const int c = rl[i];
    const int o = ix.cl_off[(int64_t)u * ix.m_cap + c], z = ix.cl_size[(int64_t)u * ix.m_cap + c];
    for (int j = threadIdx.x; j < z; j += blockDim.x) rf[o + j] = 1;
  }
  // approximate scores (row i < ns: store row i; else steady row i - ns)
  float kmx = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const T* kr = i < ns ? sk + (int64_t)i * d : stk + (int64_t)(i - ns) * d;
    const long long kro = i < ns ? i : i - ns;  // the row's index in its array (swizzle key)
    const bool swz = kv_swizzled<T>(d);
    float a = 0.f, nn = 0.f;
    for (int t = 0; t < d; t++) {
      float kv = KV<T>::to_f(kr[swz ? swz_col(t, kro) : t]);
      a = fmaf(kv, q[t], a);
      nn = fmaf(kv, kv, nn);
    }
    s[i] = a;
    kmx = fmaxf(kmx, nn);
  }
  __syncthreads();
  float qq = 0.f;
  for (int t = threadIdx.x; t < d; t += blockDim.x) qq = fmaf(q[t], q[t], qq);
  const float qn2 = block_reduce(qq, false, ssm);
  const float kn2 = block_reduce(kmx, true, ssm);
  const double uu = 5.9604644775390625e-08;
  const double gam = (double)d * uu / (1.0 - (double)d * uu);
  const double B = 2.0 * (gam + 1e-13) * (1.0 + 1e-5) * sqrt((double)qn2) * sqrt((double)kn2) * (1.0 + 1e-5);
  const double B2 = 2.0 * B * (q64 ? 1.5 : 1.0);  // fp64 queries: + the fp32 q rounding
  const float tau = u2f_ord(radix_kth_largest(s, n, K, ssm));
  if (threadIdx.x == 0) { sm.n_in = 0; sm.n_band = 0; sm.n_hit = 0; }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = (double)s[i];
    if (v > (double)tau + B2) {
      atomicAdd(&sm.n_in, 1);
      if (i >= ns || rf[i]) atomicAdd(&sm.n_hit, 1);
    } else if (v >= (double)tau - B2) {
      int p = atomicAdd(&sm.n_band, 1);
      if (p < BAND_CAP) sm.bid[p] = i;
    }
  }
  __syncthreads();
  const int nb = sm.n_band, nin = sm.n_in;
  if (nb > BAND_CAP || nin > K || nin + nb < K) {
    // dense ties (e.g. identical keys): exact selection over every token,
    // scores recomputed per radix pass (exact_select.cuh), ties to the lower
    // token id as lexsort (metrics.py:15)
    auto tok_of = [&](int i) { return i < ns ? stok[i] : sttok[i - ns]; };
    auto key = [&](int i) {
      const T* kr = i < ns ? sk + (int64_t)i * d : stk + (int64_t)(i - ns) * d;
      double kd[256];
      load_row_f64(kr, kd, d, i < ns ? i : i - ns);
      return xs_key(dgemv_row(kd, sm.q64, d, gemv_row_class(tok_of(i), n, d, blas_threads)));
    };
    auto idf = [&](int i) { return (unsigned)tok_of(i); };
    unsigned long long tk;
    unsigned ti;
    xs_select(n, K, key, idf, sm.bid, tk, ti);
    if (threadIdx.x == 0) sm.n_hit = 0;
    __syncthreads();
    int hit = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if ((i >= ns || rf[i]) && xs_in(key(i), idf(i), tk, ti)) hit++;
    atomicAdd(&sm.n_hit, hit);
    __syncthreads();
    if (threadIdx.x == 0) recall_out[ug] = K == 0 ? 1.f : (float)sm.n_hit / (float)K;
    return;
  }
  // exact fp64 scores in the reference's row recipe (row = token id in keys[:n])
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int row = sm.bid[i];
    const T* kr = row < ns ? sk + (int64_t)row * d : stk + (int64_t)(row - ns) * d;
    const int tok = row < ns ? stok[row] : sttok[row - ns];
    double kd[256];
    load_row_f64(kr, kd, d, row < ns ? row : row - ns);
    sm.bex[i] = dgemv_row(kd, sm.q64, d, gemv_row_class(tok, n, d, blas_threads));
  }
  __syncthreads();
  const int need = K - nin;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int ri = sm.bid[i];
    const int ti = ri < ns ? stok[ri] : sttok[ri - ns];
    int rank = 0;
    for (int j = 0; j < nb; j++) {
      const int rj = sm.bid[j];
      const int tj = rj < ns ? stok[rj] : sttok[rj - ns];
      rank += exact_better(sm.bex[j], tj, sm.bex[i], ti) ? 1 : 0;
    }
    if (rank < need && (ri >= ns || rf[ri])) atomicAdd(&sm.n_hit, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) recall_out[ug] = K == 0 ? 1.f : (float)sm.n_hit / (float)K;
}

size_t recall_smem_bytes() { return ((sizeof(RecallSmem) + 15) & ~size_t(15)) + sizeof(SelSmem); }

template __global__ void recall_kernel<float>(IndexView, SteadyView, StepView, const int32_t*, int, int, int, int,
                                              float*, uint8_t*, int64_t, float*);
template __global__ void recall_kernel<__nv_bfloat16>(IndexView, SteadyView, StepView, const int32_t*, int, int,
                                                      int, int, float*, uint8_t*, int64_t, float*);

}  // namespace wk
