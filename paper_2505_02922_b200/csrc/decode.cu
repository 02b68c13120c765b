// decode.cu -- per-step wave-index decode attention on B200 (sm_100a).
//
//   score   : s'[u,g,c] = q_g . C32_c for all clusters, GQA heads share each
//             C row read (index.py:61-76 ranking scores, fp32 first pass)
//   select  : exact retrieval/estimation zones per (unit, head): radix select
//             of the r-th and (r+e)-th largest approximate scores, a rigorous
//             error band, exact fp64 re-scoring of the band with the
//             reference's dgemv recipe, exact (score desc, id asc) order of
//             the retrieval list (index.py:61-93)
//   union   : per unit, union of the G heads' zones with per-cluster head masks
//   attend  : fused tripartite attention: steady zone + retrieved clusters
//             (exact, gathered through cluster -> store-row indirection) and
//             centroid estimation of the estimation zone, online softmax,
//             split over CTAs (attention.py:67-104)
//   merge   : log-sum-exp merge of the partials (attention.py:115-148,
//             engine.py:150-172), merged and eq2 denominator modes
#include "common.cuh"
#include "decode_internal.h"
#include "exact_select.cuh"

namespace wk {

// ---------------------------------------------------------------------------
// append new decode tokens to the steady buffer (engine.py:178-182)
// grid = U, block = 128
// ---------------------------------------------------------------------------
template <typename T>
__global__ void append_kernel(SteadyView st, const float* __restrict__ k_new,
                              const float* __restrict__ v_new, int d, int* status) {
  const int u = blockIdx.x;
  const int row = st.n[u];
  if (row >= st.t_cap) {  // capacity: the host checks first; never write past the buffer
    if (threadIdx.x == 0 && status) atomicCAS(status, 0, (int)kErrSteadyFull);
    return;
  }
  T* kd = (T*)st.k + ((size_t)u * st.t_cap + row) * d;
  T* vd = (T*)st.v + ((size_t)u * st.t_cap + row) * d;
  const bool swz = kv_swizzled<T>(d);
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    const int col = swz ? swz_col(t, row) : t;
    kd[col] = KV<T>::from_f(k_new[(size_t)u * d + t]);
    vd[col] = KV<T>::from_f(v_new[(size_t)u * d + t]);
  }
  __syncthreads();  // every thread read n[u] before it advances
  if (threadIdx.x == 0) {
    st.tok[(size_t)u * st.t_cap + row] = st.next_tok[u];
    st.next_tok[u] += 1;
    st.n[u] = row + 1;
  }
}
template __global__ void append_kernel<float>(SteadyView, const float*, const float*, int, int*);
template __global__ void append_kernel<__nv_bfloat16>(SteadyView, const float*, const float*, int, int*);

// ---------------------------------------------------------------------------
// score: warp per C row, lanes split d (float4), G heads per row read.
// grid = (ceil(m_cap/ROWS), U), block = 256
// ---------------------------------------------------------------------------
constexpr int SCORE_ROWS = 64;
__global__ void __launch_bounds__(256) score_kernel(IndexView ix, StepView sv, int d, int G) {
  const int u = blockIdx.y;
  const int m = sv.m[u];
  const int r0 = blockIdx.x * SCORE_ROWS;
  if (r0 >= m) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = d >> 2;  // float4 per row (d % 4 == 0)
  float4 q[8][2];
#pragma unroll
  for (int g = 0; g < 8; g++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      int v = lane + 32 * h;
      q[g][h] = (g < G && v < nv) ? reinterpret_cast<const float4*>(sv.q + ((size_t)u * G + g) * d)[v]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  const int r1 = min(m, r0 + SCORE_ROWS);
  for (int row = r0 + warp; row < r1; row += 8) {
    const float4* cr = reinterpret_cast<const float4*>(ix.C32 + ((size_t)u * ix.m_cap + row) * d);
    float4 c0 = lane < nv ? __ldg(cr + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 c1 = lane + 32 < nv ? __ldg(cr + lane + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
    float acc[8];
#pragma unroll
    for (int g = 0; g < 8; g++) {
      float a = 0.f;
      if (g < G) {
        a = fmaf(c0.x, q[g][0].x, a); a = fmaf(c0.y, q[g][0].y, a);
        a = fmaf(c0.z, q[g][0].z, a); a = fmaf(c0.w, q[g][0].w, a);
        a = fmaf(c1.x, q[g][1].x, a); a = fmaf(c1.y, q[g][1].y, a);
        a = fmaf(c1.z, q[g][1].z, a); a = fmaf(c1.w, q[g][1].w, a);
      }
      acc[g] = a;
    }
#pragma unroll
    for (int g = 0; g < 8; g++) {
      if (g < G) {
        float v = warp_sum(acc[g]);
        if (lane == 0) sv.scores[((size_t)u * G + g) * ix.m_cap + row] = v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// select helpers
// ---------------------------------------------------------------------------
constexpr int SEL_THREADS = 512;
constexpr int BAND_CAP = 1024;
constexpr int RL_CAP = 4096;

struct SelSmem {
  unsigned long long rl[RL_CAP];   // retrieval list sort keys
  double ex[RL_CAP];               // exact score per sorted position (NaN = unknown)
  int bid_r[BAND_CAP];             // band rows around tau_r
  double bex_r[BAND_CAP];
  int bid_e[BAND_CAP];             // band rows around tau_{r+e}
  double bex_e[BAND_CAP];
  unsigned char bsel_e[BAND_CAP];
  int hist[256];
  double q64[256];
  float red[32];
  int n_in_r, n_band_r, n_band_e, n_in_e, n_rl;
  unsigned int prefix;
  int krem;
  float fred;
};

__device__ unsigned int radix_kth_largest(const float* s, int m, int K, SelSmem& sm) {
  // K-th largest (1-based) of the order-preserving keys; 4 passes of 8 bits
  unsigned int prefix = 0, pmask = 0;
  if (threadIdx.x == 0) sm.krem = K;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) sm.hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      unsigned int key = f2u_ord(s[i]);
      if ((key & pmask) == prefix) atomicAdd(&sm.hist[(key >> shift) & 255u], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane l owns bins [8l, 8l+8); suffix sums from the top bin
      const int lane = threadIdx.x;
      int local = 0;
      for (int j = 0; j < 8; j++) local += sm.hist[8 * lane + j];
      int suf = local;  // inclusive suffix over lanes >= lane
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += v;
      }
      const int krem = sm.krem;
      int above = suf - local;  // count in lanes > lane
      bool here = above < krem && suf >= krem;
      unsigned int ball = __ballot_sync(0xffffffffu, here);
      int owner = __ffs(ball) - 1;
      if (lane == owner) {
        int acc = above;
        int sel = 8 * lane;
        for (int j = 7; j >= 0; j--) {
          int h = sm.hist[8 * lane + j];
          if (acc + h >= krem) { sel = 8 * lane + j; break; }
          acc += h;
        }
        sm.krem = krem - acc;
        sm.prefix = (unsigned int)sel;
      }
    }
    __syncthreads();
    prefix |= sm.prefix << shift;
    pmask |= 255u << shift;
    __syncthreads();
  }
  return prefix;
}

__device__ __forceinline__ double exact_score(const IndexView& ix, int u, int c, int m, int d,
                                              int blas_threads, const double* q64) {
  const double* row = ix.C64 + ((size_t)u * ix.m_cap + c) * d;
  return dgemv_row(row, q64, d, gemv_row_class(c, m, d, blas_threads));
}

// key for ascending sort = (approx score desc, id asc)
__device__ __forceinline__ unsigned long long sel_key(float s, int id) {
  return ((unsigned long long)(~f2u_ord(s)) << 32) | (unsigned int)id;
}
__device__ __forceinline__ float key_score(unsigned long long k) {
  return u2f_ord(~(unsigned int)(k >> 32));
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)(k & 0xffffffffu); }

__device__ __forceinline__ bool exact_better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

__device__ __forceinline__ float block_reduce(float v, bool is_max, SelSmem& sm) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm.red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = sm.red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) r = is_max ? fmaxf(r, sm.red[i]) : r + sm.red[i];
    sm.fred = r;
  }
  __syncthreads();
  return sm.fred;
}

// ---------------------------------------------------------------------------
// select: grid = U*G, block = SEL_THREADS, dyn smem = sizeof(SelSmem)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SEL_THREADS) select_kernel(IndexView ix, StepView sv, SelParams p) {
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelSmem& sm = *reinterpret_cast<SelSmem*>(sel_raw);
  const int G = p.G, d = p.d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int m = sv.m[u];
  float* tailp = sv.tail + ((size_t)u * G + g) * 4;
  if (m == 0) {
    if (threadIdx.x == 0) {
      if (g == 0) { sv.nr[u] = 0; sv.ne[u] = 0; }
      tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f;
    }
    return;
  }
  int r = (int)floor(p.retrieval_fraction * (double)m + 0.5);
  if (r < 1) r = 1;
  if (r > m) r = m;
  int e = (int)floor(p.estimation_fraction * (double)m + 0.5);
  if (e > m - r) e = m - r;
  if (threadIdx.x == 0 && g == 0) { sv.nr[u] = r; sv.ne[u] = e; }
  const float* s = sv.scores + ((size_t)u * G + g) * ix.m_cap;
  const float* q = sv.q + ((size_t)u * G + g) * d;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const double* q64 = sv.q64 ? sv.q64 + ((size_t)u * G + g) * d : nullptr;
  for (int t = threadIdx.x; t < d; t += blockDim.x) sm.q64[t] = q64 ? q64[t] : (double)q[t];
  if (r > RL_CAP) { set_status(sv.status, kErrBandOverflow); return; }
  // ---- error bound B >= |s'_c - s_c| for every row -------------------------
  float qq = 0.f;
  for (int t = threadIdx.x; t < d; t += blockDim.x) qq = fmaf(q[t], q[t], qq);
  float qn2 = block_reduce(qq, false, sm);
  float cm = 0.f;
  for (int c = threadIdx.x; c < m; c += blockDim.x) cm = fmaxf(cm, ix.Cnorm[(size_t)u * ix.m_cap + c]);
  float cmax = block_reduce(cm, true, sm);
  const double uu = 5.9604644775390625e-08;  // 2^-24
  const double gam = (double)d * uu / (1.0 - (double)d * uu);
  // with fp64 queries the scan's fp32 q adds 2^-24 |q| |C|
  const double B = score_error_bound((double)qn2, (double)cmax, d, p.score_fp64 != 0) * (q64 ? 1.6 : 1.0);
  const double B2 = 2.0 * B;
  // ---- thresholds -------------------------------------------------------------
  const float tau_r = u2f_ord(radix_kth_largest(s, m, r, sm));
  float tau_e = 0.f;
  if (e > 0) tau_e = u2f_ord(radix_kth_largest(s, m, r + e, sm));
  if (threadIdx.x == 0) { sm.n_in_r = 0; sm.n_band_r = 0; sm.n_band_e = 0; sm.n_in_e = 0; sm.n_rl = 0; }
  __syncthreads();
  // ---- classification ---------------------------------------------------------
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    const double sc = (double)s[c];
    if (sc > (double)tau_r + B2) {
      int pos = atomicAdd(&sm.n_rl, 1);
      if (pos < RL_CAP) sm.rl[pos] = sel_key(s[c], c);
      atomicAdd(&sm.n_in_r, 1);
    } else if (sc >= (double)tau_r - B2) {
      int pos = atomicAdd(&sm.n_band_r, 1);
      if (pos < BAND_CAP) sm.bid_r[pos] = c;
    }
    if (e > 0) {
      if (sc > (double)tau_e + B2) {
        atomicAdd(&sm.n_in_e, 1);
      } else if (sc >= (double)tau_e - B2) {
        int pos = atomicAdd(&sm.n_band_e, 1);
        if (pos < BAND_CAP) sm.bid_e[pos] = c;
      }
    }
  }
  __syncthreads();
  const int nbr = sm.n_band_r, nbe = sm.n_band_e, nin_r = sm.n_in_r, nin_e = sm.n_in_e;
  int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
  if (nbr > BAND_CAP || nbe > BAND_CAP || nin_r > r || nin_r + nbr < r ||
      (e > 0 && (nin_e > r + e || nin_e + nbe < r + e))) {
    // dense ties / band overflow: exact scores of every row + radix select
    // (exact_select.cuh), R ordered by counting
    if (!sv.xscr) {
      set_status(sv.status, kErrBandOverflow);
      return;
    }
    double* xs = sv.xscr + ((size_t)u * G + g) * ix.m_cap;
    xs_score_rows(ix.C64 + (size_t)u * ix.m_cap * d, sm.q64, m, d, p.blas_threads, xs);
    if (threadIdx.x == 0) { sm.n_rl = 0; sm.n_in_e = 0; }
    __syncthreads();
    auto key = [&](int c) { return xs_key(__ldcg(xs + c)); };
    auto idf = [&](int c) { return (unsigned)c; };
    unsigned long long k1, k2 = 0ull;
    unsigned i1, i2 = 0u;
    xs_select(m, r, key, idf, sm.bid_r, k1, i1);
    if (e > 0) xs_select(m, r + e, key, idf, sm.bid_r, k2, i2);
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      const unsigned long long kk = key(c);
      if (xs_in(kk, (unsigned)c, k1, i1)) {
        const int pos = atomicAdd(&sm.n_rl, 1);
        sm.rl[pos] = (unsigned long long)(unsigned)c;
        sm.ex[pos] = __ldcg(xs + c);
      } else if (e > 0 && xs_in(kk, (unsigned)c, k2, i2)) {
        atomicOr(zm + c, 1u << (8 + g));
        if (el_out) el_out[atomicAdd(&sm.n_in_e, 1)] = c;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
      const double ei = sm.ex[i];
      const int ii = key_id(sm.rl[i]);
      int rk = 0;
      for (int j = 0; j < r; j++) rk += exact_better(sm.ex[j], key_id(sm.rl[j]), ei, ii) ? 1 : 0;
      rl_out[rk] = ii;
      atomicOr(zm + ii, 1u << g);
    }
    if (threadIdx.x == 0 && sv.xcount) atomicAdd(sv.xcount, 1);
    __syncthreads();
  } else {
  // ---- exact fp64 re-scoring of the bands (reference dgemv recipe) ------------
  for (int i = threadIdx.x; i < nbr; i += blockDim.x)
    sm.bex_r[i] = exact_score(ix, u, sm.bid_r[i], m, d, p.blas_threads, sm.q64);
  for (int i = threadIdx.x; i < nbe; i += blockDim.x)
    sm.bex_e[i] = exact_score(ix, u, sm.bid_e[i], m, d, p.blas_threads, sm.q64);
  __syncthreads();
  // best (r - nin_r) of band_r by exact (score desc, id asc) join the list
  const int need_r = r - nin_r;
  for (int i = threadIdx.x; i < nbr; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < nbr; j++)
      rank += exact_better(sm.bex_r[j], sm.bid_r[j], sm.bex_r[i], sm.bid_r[i]) ? 1 : 0;
    if (rank < need_r) {
      int pos = atomicAdd(&sm.n_rl, 1);
      sm.rl[pos] = sel_key(s[sm.bid_r[i]], sm.bid_r[i]);
    }
  }
  const int need_e = r + e - nin_e;
  for (int i = threadIdx.x; i < nbe; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < nbe; j++)
      rank += exact_better(sm.bex_e[j], sm.bid_e[j], sm.bex_e[i], sm.bid_e[i]) ? 1 : 0;
    sm.bsel_e[i] = rank < need_e ? 1 : 0;
  }
  __syncthreads();
  // ---- sort the retrieval set by (approx desc, id asc): bitonic ---------------
  int npow = 1;
  while (npow < r) npow <<= 1;
  for (int i = r + threadIdx.x; i < npow; i += blockDim.x) sm.rl[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = sm.rl[i], b = sm.rl[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { sm.rl[i] = b; sm.rl[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  // ---- clumps: neighbours closer than 2B get exact scores and exact order -----
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    const double si = (double)key_score(sm.rl[i]);
    bool cl = (i > 0 && (double)key_score(sm.rl[i - 1]) - si <= B2) ||
              (i + 1 < r && si - (double)key_score(sm.rl[i + 1]) <= B2);
    sm.ex[i] = cl ? exact_score(ix, u, key_id(sm.rl[i]), m, d, p.blas_threads, sm.q64) : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    const double si = (double)key_score(sm.rl[i]);
    bool link_prev = i > 0 && (double)key_score(sm.rl[i - 1]) - si <= B2;
    bool link_next = i + 1 < r && si - (double)key_score(sm.rl[i + 1]) <= B2;
    if (!link_prev && link_next) {
      int end = i + 1;
      while (end + 1 < r && (double)key_score(sm.rl[end]) - (double)key_score(sm.rl[end + 1]) <= B2) end++;
      // insertion sort [i, end] by exact (desc, id asc)
      for (int a = i + 1; a <= end; a++) {
        unsigned long long kk = sm.rl[a];
        double ev = sm.ex[a];
        int b = a - 1;
        while (b >= i && exact_better(ev, key_id(kk), sm.ex[b], key_id(sm.rl[b]))) {
          sm.rl[b + 1] = sm.rl[b];
          sm.ex[b + 1] = sm.ex[b];
          b--;
        }
        sm.rl[b + 1] = kk;
        sm.ex[b + 1] = ev;
      }
    }
  }
  __syncthreads();
  // ---- outputs: ordered retrieval list, zone masks ---------------------------
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    int c = key_id(sm.rl[i]);
    rl_out[i] = c;
    atomicOr(zm + c, 1u << g);
  }
  __threadfence_block();
  __syncthreads();
  if (threadIdx.x == 0) sm.n_in_e = 0;  // reuse as E cursor
  __syncthreads();
  if (e > 0) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      if ((double)s[c] > (double)tau_e + B2 && !(zm[c] & (1u << g))) {
        atomicOr(zm + c, 1u << (8 + g));
        if (el_out) el_out[atomicAdd(&sm.n_in_e, 1)] = c;
      }
    }
    for (int i = threadIdx.x; i < nbe; i += blockDim.x) {
      int c = sm.bid_e[i];
      if (sm.bsel_e[i] && !(zm[c] & (1u << g))) {
        atomicOr(zm + c, 1u << (8 + g));
        if (el_out) el_out[atomicAdd(&sm.n_in_e, 1)] = c;
      }
    }
  }
  __syncthreads();
  }  // exact band path
  // ---- tail / all-cluster denominator terms (engine.py:153-172) ---------------
  if (p.need_tail || p.need_allc) {
    const float isd = p.inv_sqrt_d;
    float mx_t = -INFINITY, mx_a = -INFINITY;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      float v = s[c] * isd;
      mx_a = fmaxf(mx_a, v);
      if (!(zm[c] & ((1u << g) | (1u << (8 + g))))) mx_t = fmaxf(mx_t, v);
    }
    mx_t = block_reduce(mx_t, true, sm);
    mx_a = block_reduce(mx_a, true, sm);
    float dt = 0.f, da = 0.f;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      float v = s[c] * isd;
      float sz = (float)csize[c];
      da += sz * expf(v - mx_a);
      if (!(zm[c] & ((1u << g) | (1u << (8 + g))))) dt += sz * expf(v - mx_t);
    }
    dt = block_reduce(dt, false, sm);
    da = block_reduce(da, false, sm);
    if (threadIdx.x == 0) {
      tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da;
    }
  }
}

size_t select_smem_bytes() { return sizeof(SelSmem); }

// ---------------------------------------------------------------------------
// union: per unit, clusters in any head's R (resp. E) zone, ascending id, with
// head masks; prefix sums of retrieved token counts; clears the zone masks.
// grid = U, block = 1024
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) union_kernel(IndexView ix, StepView sv) {
  const int u = blockIdx.x;
  const int m = sv.m[u];
  __shared__ int wr[32], we[32], wt[32];
  __shared__ int base_r, base_e, base_t;
  if (threadIdx.x == 0) { base_r = 0; base_e = 0; base_t = 0; }
  __syncthreads();
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  int32_t* rpre = sv.ru_pre + (size_t)u * (sv.ru_cap + 1);
  int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = 0; c0 < m; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    uint32_t z = c < m ? zm[c] : 0u;
    if (c < m) zm[c] = 0u;
    const int fr = (z & 0xffu) ? 1 : 0, fe = (z & 0xff00u) ? 1 : 0;
    const int sz = fr ? csize[c] : 0;
    // warp inclusive scans
    int xr = fr, xe = fe, xt = sz;
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, xr, o), b = __shfl_up_sync(0xffffffffu, xe, o),
          t = __shfl_up_sync(0xffffffffu, xt, o);
      if (lane >= o) { xr += a; xe += b; xt += t; }
    }
    if (lane == 31) { wr[w] = xr; we[w] = xe; wt[w] = xt; }
    __syncthreads();
    if (w == 0) {
      int a = wr[lane], b = we[lane], t = wt[lane];
      int ia = a, ib = b, it = t;
      for (int o = 1; o < 32; o <<= 1) {
        int pa = __shfl_up_sync(0xffffffffu, ia, o), pb = __shfl_up_sync(0xffffffffu, ib, o),
            pt = __shfl_up_sync(0xffffffffu, it, o);
        if (lane >= o) { ia += pa; ib += pb; it += pt; }
      }
      wr[lane] = ia - a; we[lane] = ib - b; wt[lane] = it - t;  // exclusive warp offsets
    }
    __syncthreads();
    const int pr = base_r + wr[w] + xr - fr;
    const int pe = base_e + we[w] + xe - fe;
    const int pt = base_t + wt[w] + xt - sz;
    if (fr) {
      if (pr < sv.ru_cap) { ru[pr] = c; rmk[pr] = (uint8_t)(z & 0xffu); rpre[pr] = pt; }
      else set_status(sv.status, kErrUnion);
    }
    if (fe) {
      if (pe < sv.eu_cap) { eu[pe] = c; emk[pe] = (uint8_t)((z >> 8) & 0xffu); }
      else set_status(sv.status, kErrUnion);
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      base_r = pr + fr;
      base_e = pe + fe;
      base_t = pt + sz;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int nr = min(base_r, sv.ru_cap);
    rpre[nr] = base_t;
    sv.cnt[u * 4 + 0] = nr;
    sv.cnt[u * 4 + 1] = base_t;
    sv.cnt[u * 4 + 2] = min(base_e, sv.eu_cap);
  }
}

// ---------------------------------------------------------------------------
// attend: fused tripartite attention partials.
// grid = (S, U), block = 128, dyn smem = attend_smem_bytes(d, sizeof(T))
// Work of unit u = [steady tiles | retrieved-token tiles | estimation tiles],
// 64 rows per tile, split evenly over the S CTAs of the unit.  Each CTA keeps
// three online-softmax partials per head: steady (0), retrieved (1),
// estimated (2); retrieved tokens / estimation rows only count for the heads
// whose zone holds their cluster (head masks from union_kernel).
// ---------------------------------------------------------------------------
constexpr int AT_ROWS = 64;
constexpr int AT_THREADS = 128;
constexpr int GMAX = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// 16 bytes of a row -> floats
__device__ __forceinline__ int load16(const float* p, float* o) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  return 4;
}
__device__ __forceinline__ int load16(const __nv_bfloat16* p, float* o) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
  return 8;
}

size_t attend_smem_bytes(int d, int elem) {
  size_t b = 0;
  b += (size_t)GMAX * d * 4;             // q
  b += (size_t)GMAX * AT_ROWS * 4;       // logits / weights
  b += (size_t)4 * GMAX * 4;             // alpha + sM/sD (3 kinds)
  b += (size_t)3 * GMAX * 4;
  b += (size_t)AT_ROWS * 4;              // sizes of E rows
  b += (size_t)AT_ROWS * 4;              // head masks
  b += (size_t)AT_ROWS * 8;              // row sources
  b = (b + 15) & ~(size_t)15;
  size_t tk = (size_t)AT_ROWS * (d * elem + 16);
  size_t tf = (size_t)AT_ROWS * (d * 4 + 16);
  b += 2 * tk > tf ? 2 * tk : tf;
  return b;
}

template <typename T, bool FULL>
__global__ void __launch_bounds__(AT_THREADS) attend_kernel(IndexView ix, SteadyView st, StepView sv,
                                                             AttnParams p, const int32_t* __restrict__ n_store) {
  const int s_idx = blockIdx.x, u = blockIdx.y;
  const int S = gridDim.x, G = p.G, d = p.d;
  extern __shared__ __align__(16) unsigned char at_raw[];
  float* q_s = reinterpret_cast<float*>(at_raw);
  float* lg = q_s + GMAX * d;
  float* alpha = lg + GMAX * AT_ROWS;
  float* sM = alpha + GMAX;         // [3][GMAX]
  float* sD = sM + 3 * GMAX;        // [3][GMAX]
  float* wsz = sD + 3 * GMAX;       // [AT_ROWS]
  int* rmask = reinterpret_cast<int*>(wsz + AT_ROWS);
  long long* rsrc = reinterpret_cast<long long*>(rmask + AT_ROWS);
  size_t off = (size_t)(reinterpret_cast<unsigned char*>(rsrc + AT_ROWS) - at_raw);
  off = (off + 15) & ~(size_t)15;
  unsigned char* tA = at_raw + off;
  const int ldb = d * (int)sizeof(T) + 16;  // padded row bytes (K/V tiles)
  unsigned char* tB = tA + AT_ROWS * ldb;
  const int ldf = d * 4 + 16;               // padded row bytes (VS tiles, f32)

  for (int i = threadIdx.x; i < G * d; i += blockDim.x) q_s[i] = sv.q[(size_t)u * G * d + i];
  if (threadIdx.x < 3 * GMAX) { sM[threadIdx.x] = -INFINITY; sD[threadIdx.x] = 0.f; }

  const int n_st = st.n[u];
  const int n_ru = FULL ? 0 : sv.cnt[u * 4 + 0];
  const int n_rt = FULL ? n_store[u] : sv.cnt[u * 4 + 1];
  const int n_eu = FULL ? 0 : sv.cnt[u * 4 + 2];
  const int t_st = (n_st + AT_ROWS - 1) / AT_ROWS, t_r = (n_rt + AT_ROWS - 1) / AT_ROWS,
            t_e = (n_eu + AT_ROWS - 1) / AT_ROWS;
  const int T_all = t_st + t_r + t_e;
  const int tb = (int)((long long)s_idx * T_all / S), te = (int)((long long)(s_idx + 1) * T_all / S);

  float acc[3][GMAX][2];
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int g = 0; g < GMAX; g++) { acc[k][g][0] = 0.f; acc[k][g][1] = 0.f; }

  const int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  const uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  const int32_t* rpre = sv.ru_pre + (size_t)u * (sv.ru_cap + 1);
  const int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  const uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  const int32_t* coff = ix.cl_off + (size_t)u * ix.m_cap;
  const int32_t* csz = ix.cl_size + (size_t)u * ix.m_cap;
  const T* stk = (const T*)st.k + (size_t)u * st.t_cap * d;
  const T* stv = (const T*)st.v + (size_t)u * st.t_cap * d;
  const T* sk = (const T*)ix.store_k + (size_t)u * ix.s_cap * d;
  const T* svv = (const T*)ix.store_v + (size_t)u * ix.s_cap * d;
  const float* vs = ix.VS32 + (size_t)u * ix.m_cap * d;
  const float* scr = FULL ? nullptr : sv.scores + (size_t)u * G * ix.m_cap;
  const float isd = p.inv_sqrt_d;
  const int allmask = (1 << G) - 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();

  for (int tile = tb; tile < te; tile++) {
    int kind, r0, nrow;
    if (tile < t_st) { kind = 0; r0 = tile * AT_ROWS; nrow = min(AT_ROWS, n_st - r0); }
    else if (tile < t_st + t_r) { kind = 1; r0 = (tile - t_st) * AT_ROWS; nrow = min(AT_ROWS, n_rt - r0); }
    else { kind = 2; r0 = (tile - t_st - t_r) * AT_ROWS; nrow = min(AT_ROWS, n_eu - r0); }
    // ---- row sources and head masks ----
    if (threadIdx.x < AT_ROWS) {
      const int j = threadIdx.x;
      long long src = 0;
      int mk = 0;
      float sz = 0.f;
      if (j < nrow) {
        if (kind == 0) { src = r0 + j; mk = allmask; }
        else if (FULL && kind == 1) { src = r0 + j; mk = allmask; }
        else if (kind == 1) {
          const int pos = r0 + j;
          int lo = 0, hi = n_ru;  // last i with rpre[i] <= pos
          while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (rpre[mid] <= pos) lo = mid; else hi = mid; }
          const int c = ru[lo];
          src = (long long)coff[c] + (pos - rpre[lo]);
          mk = rmk[lo];
        } else {
          const int c = eu[r0 + j];
          src = c;
          mk = emk[r0 + j];
          sz = (float)csz[c];
        }
      }
      rsrc[j] = src;
      rmask[j] = mk;
      wsz[j] = sz;
    }
    __syncthreads();
    // ---- stage the tile (cp.async 16B, coalesced per row) ----
    if (kind < 2) {
      const T* kb = kind == 0 ? stk : sk;
      const T* vb = kind == 0 ? stv : svv;
      const int cpr = d * (int)sizeof(T) / 16;
      const bool swz = kv_swizzled<T>(d);  // swizzled rows (common.cuh swz_col): un-swizzle while staging
      for (int idx = threadIdx.x; idx < nrow * cpr; idx += blockDim.x) {
        const int j = idx / cpr, ch = idx % cpr;
        const long long src = rsrc[j];
        const int pch = swz ? (ch ^ (int)(src & 7)) : ch;
        cp_async16(tA + j * ldb + ch * 16, reinterpret_cast<const unsigned char*>(kb + src * d) + pch * 16);
        cp_async16(tB + j * ldb + ch * 16, reinterpret_cast<const unsigned char*>(vb + src * d) + pch * 16);
      }
    } else {
      const int cpr = d * 4 / 16;
      for (int idx = threadIdx.x; idx < nrow * cpr; idx += blockDim.x) {
        const int j = idx / cpr, ch = idx % cpr;
        cp_async16(tA + j * ldf + ch * 16, reinterpret_cast<const unsigned char*>(vs + rsrc[j] * d) + ch * 16);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- logits lg[g][j] (scaled by 1/sqrt(d)) ----
    if (kind < 2) {
      for (int pr = threadIdx.x; pr < G * AT_ROWS; pr += blockDim.x) {
        const int j = pr % AT_ROWS, g = pr / AT_ROWS;
        float v = -INFINITY;
        if (j < nrow && ((rmask[j] >> g) & 1)) {
          const T* kr = reinterpret_cast<const T*>(tA + j * ldb);
          const float* qg = q_s + g * d;
          float a0 = 0.f, a1 = 0.f;
          for (int t = 0; t < d;) {
            float kv[8];
            int nl = load16(kr + t, kv);
            for (int i = 0; i < nl; i += 2) {
              a0 = fmaf(kv[i], qg[t + i], a0);
              a1 = fmaf(kv[i + 1], qg[t + i + 1], a1);
            }
            t += nl;
          }
          v = (a0 + a1) * isd;
        }
        lg[g * AT_ROWS + j] = v;
      }
    } else {
      for (int pr = threadIdx.x; pr < G * AT_ROWS; pr += blockDim.x) {
        const int j = pr % AT_ROWS, g = pr / AT_ROWS;
        float v = -INFINITY;
        if (j < nrow && ((rmask[j] >> g) & 1)) v = scr[(size_t)g * ix.m_cap + rsrc[j]] * isd;
        lg[g * AT_ROWS + j] = v;
      }
    }
    __syncthreads();
    // ---- online softmax per head (warp w handles heads w, w+4) ----
    for (int g = w; g < G; g += 4) {
      const float a = lg[g * AT_ROWS + lane], b = lg[g * AT_ROWS + lane + 32];
      const float tm = warp_max(fmaxf(a, b));
      const float Mo = sM[kind * GMAX + g];
      const float Mn = fmaxf(Mo, tm);
      float pa = 0.f, pb = 0.f, al = 1.f, dt = 0.f;
      if (Mn != -INFINITY) {
        pa = (a == -INFINITY) ? 0.f : expf(a - Mn);
        pb = (b == -INFINITY) ? 0.f : expf(b - Mn);
        al = (Mo == -INFINITY) ? 0.f : expf(Mo - Mn);
        dt = warp_sum(kind == 2 ? pa * wsz[lane] + pb * wsz[lane + 32] : pa + pb);
      }
      lg[g * AT_ROWS + lane] = pa;
      lg[g * AT_ROWS + lane + 32] = pb;
      if (lane == 0) {
        alpha[g] = al;
        sD[kind * GMAX + g] = sD[kind * GMAX + g] * al + dt;
        sM[kind * GMAX + g] = Mn;
      }
    }
    __syncthreads();
    // ---- numerators: thread owns dims tid and tid+128 ----
    auto pv = [&](float (&a)[GMAX][2]) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int t = threadIdx.x + h * AT_THREADS;
        if (t < d) {
#pragma unroll
          for (int g = 0; g < GMAX; g++)
            if (g < G) a[g][h] *= alpha[g];
          for (int j = 0; j < nrow; j++) {
            float v;
            if (kind < 2) v = KV<T>::to_f(reinterpret_cast<const T*>(tB + j * ldb)[t]);
            else v = reinterpret_cast<const float*>(tA + j * ldf)[t];
#pragma unroll
            for (int g = 0; g < GMAX; g++)
              if (g < G) a[g][h] = fmaf(lg[g * AT_ROWS + j], v, a[g][h]);
          }
        }
      }
    };
    if (kind == 0) pv(acc[0]);
    else if (kind == 1) pv(acc[1]);
    else pv(acc[2]);
    __syncthreads();
  }
  // ---- write partials: part[(((u*S+s)*G+g)*3+kind)*(2+d)] = {M, D, num[d]} ----
  const int stride = 2 + d;
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int g = 0; g < GMAX; g++) {
      if (g < G) {
        float* dst = sv.part + ((((size_t)u * S + s_idx) * G + g) * 3 + k) * stride;
        if (threadIdx.x == 0) { dst[0] = sM[k * GMAX + g]; dst[1] = sD[k * GMAX + g]; }
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int t = threadIdx.x + h * AT_THREADS;
          if (t < d) dst[2 + t] = acc[k][g][h];
        }
      }
    }
}
template __global__ void attend_kernel<float, false>(IndexView, SteadyView, StepView, AttnParams, const int32_t*);
template __global__ void attend_kernel<__nv_bfloat16, false>(IndexView, SteadyView, StepView, AttnParams, const int32_t*);
template __global__ void attend_kernel<float, true>(IndexView, SteadyView, StepView, AttnParams, const int32_t*);
template __global__ void attend_kernel<__nv_bfloat16, true>(IndexView, SteadyView, StepView, AttnParams, const int32_t*);

// ---------------------------------------------------------------------------
// merge: combine the S split partials of each (unit, head) and the three
// zones into the output (attention.py:115-148; engine.py:150-172).
// grid = U*G, block = 128
// ---------------------------------------------------------------------------
__global__ void merge_kernel(StepView sv, AttnParams p, int S) {
  const int u = blockIdx.x / p.G, g = blockIdx.x % p.G, d = p.d, G = p.G;
  const int stride = 2 + d;
  __shared__ double kM[3], kD[3];
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    double Mx = -INFINITY;
    for (int s = 0; s < S; s++) {
      const float* src = sv.part + ((((size_t)u * S + s) * G + g) * 3 + k) * stride;
      if (src[1] > 0.f) Mx = fmax(Mx, (double)src[0]);
    }
    double Dn = 0.0;
    if (Mx != -INFINITY)
      for (int s = 0; s < S; s++) {
        const float* src = sv.part + ((((size_t)u * S + s) * G + g) * 3 + k) * stride;
        if (src[1] > 0.f) Dn += (double)src[1] * exp((double)src[0] - Mx);
      }
    kM[k] = Mx;
    kD[k] = Dn;
  }
  __syncthreads();
  const float zero4[4] = {-INFINITY, 0.f, -INFINITY, 0.f};
  const float* tl = sv.tail ? sv.tail + ((size_t)u * G + g) * 4 : zero4;
  // zone partials: exact = steady (+) retrieved; est; tail
  const bool live0 = kD[0] > 0, live1 = kD[1] > 0, live2 = kD[2] > 0;
  const bool live3 = p.tail_denominator_only && tl[1] > 0.f;
  double gmax = -INFINITY;
  if (live0) gmax = fmax(gmax, kM[0]);
  if (live1) gmax = fmax(gmax, kM[1]);
  if (live2) gmax = fmax(gmax, kM[2]);
  if (live3) gmax = fmax(gmax, (double)tl[0]);
  if (gmax == -INFINITY) {  // merge requires a non-empty partial (attention.py:117-119)
    set_status(sv.status, kErrEmptyMerge);
    return;
  }
  const double sc0 = live0 ? exp(kM[0] - gmax) : 0.0, sc1 = live1 ? exp(kM[1] - gmax) : 0.0,
               sc2 = live2 ? exp(kM[2] - gmax) : 0.0, sc3 = live3 ? exp((double)tl[0] - gmax) : 0.0;
  const double den = kD[0] * sc0 + kD[1] * sc1 + kD[2] * sc2 + (live3 ? (double)tl[1] * sc3 : 0.0);
  double out_scale, logden, cov;
  if (!p.denominator_eq2) {
    out_scale = 1.0 / den;
    logden = gmax + log(den);
    cov = den > 0 ? (kD[0] * sc0 + kD[1] * sc1) / den : 0.0;
  } else {
    // eq2: denominator = steady exact terms + centroid terms of all clusters
    const bool la = tl[3] > 0.f;
    double gd = -INFINITY;
    if (live0) gd = fmax(gd, kM[0]);
    if (la) gd = fmax(gd, (double)tl[2]);
    const double dd = (live0 ? kD[0] * exp(kM[0] - gd) : 0.0) + (la ? (double)tl[3] * exp((double)tl[2] - gd) : 0.0);
    out_scale = exp(gmax - gd) / dd;
    logden = gd + log(dd);
    cov = dd > 0 ? (live0 ? kD[0] * exp(kM[0] - gd) : 0.0) / dd : 0.0;
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double num = 0.0;
    for (int k = 0; k < 3; k++) {
      if (kD[k] <= 0) continue;
      const double zs = (k == 0 ? sc0 : (k == 1 ? sc1 : sc2));
      double nk = 0.0;
      for (int s = 0; s < S; s++) {
        const float* src = sv.part + ((((size_t)u * S + s) * G + g) * 3 + k) * stride;
        if (src[1] > 0.f) nk += (double)src[2 + t] * exp((double)src[0] - kM[k]);
      }
      num += nk * zs;
    }
    sv.out[((size_t)u * G + g) * d + t] = (float)(num * out_scale);
  }
  if (threadIdx.x == 0) {
    sv.logden[(size_t)u * G + g] = (float)logden;
    sv.cov[(size_t)u * G + g] = (float)cov;
  }
}

}  // namespace wk
