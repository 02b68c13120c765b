// decode_v2.cu -- throughput versions of the per-step decode kernels.
//
//   score_v2   : warp processes 32/HS centroid rows per iteration; the G
//                heads' partial dots (32 values per lane) are reduced with one
//                31-shuffle transposed reduction instead of 5 shuffles per
//                (row, head)
//   select_v2  : warp-aggregated 3-pass radix select (11/11/10-bit digits),
//                ballot-compacted classification, exact band re-scoring as in
//                v1; the last CTA of each unit builds the union lists and the
//                flat retrieved-token row list (replaces union_kernel)
//   attend_v2  : register-direct decode attention: a warp takes groups of
//                32/HS tokens, each lane owns d/32 contiguous dims of every
//                row, K/V rows are software-prefetched into registers one
//                group ahead, logits of the (token, head) pairs come out of a
//                transposed reduction, online softmax per head, P.V in
//                registers; no shared-memory staging of K/V.
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

constexpr unsigned FULLMASK = 0xffffffffu;

// v[i] (i < 32) summed over the warp; returns the total of index `lane`.
__device__ __forceinline__ float transpose_reduce32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; i++) {
      const float send = up ? v[i] : v[i + off];
      const float keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(FULLMASK, send, off);
    }
  }
  return v[0];
}

// ---------------------------------------------------------------------------
// score_v2: grid = (ceil(m_cap / rows_per_cta), U), block = 256
// ---------------------------------------------------------------------------
template <int HS>
__global__ void __launch_bounds__(256) score_v2_kernel(IndexView ix, StepView sv, int d, int G,
                                                        int rows_per_cta) {
  constexpr int RG = 32 / HS;
  const int u = blockIdx.y;
  const int m = sv.m[u];
  const int r0 = blockIdx.x * rows_per_cta;
  if (r0 >= m) return;
  const int r1 = min(m, r0 + rows_per_cta);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = d >> 2;
  float4 q0[HS], q1[HS];
#pragma unroll
  for (int h = 0; h < HS; h++) {
    const float4* qg = reinterpret_cast<const float4*>(sv.q + ((size_t)u * G + (h < G ? h : 0)) * d);
    q0[h] = (h < G && lane < nv) ? qg[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    q1[h] = (h < G && lane + 32 < nv) ? qg[lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float* Cb = ix.C32 + (size_t)u * ix.m_cap * d;
  float* out = sv.scores + (size_t)u * G * ix.m_cap;
  for (int g0 = r0 + warp * RG; g0 < r1; g0 += 8 * RG) {
    float4 c0[RG], c1[RG];
#pragma unroll
    for (int j = 0; j < RG; j++) {
      const int row = g0 + j;
      const float4* cr = reinterpret_cast<const float4*>(Cb + (size_t)row * d);
      c0[j] = (row < r1 && lane < nv) ? __ldcs(cr + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
      c1[j] = (row < r1 && lane + 32 < nv) ? __ldcs(cr + lane + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float v[32];
#pragma unroll
    for (int j = 0; j < RG; j++)
#pragma unroll
      for (int h = 0; h < HS; h++) {
        float a = c0[j].x * q0[h].x;
        a = fmaf(c0[j].y, q0[h].y, a); a = fmaf(c0[j].z, q0[h].z, a); a = fmaf(c0[j].w, q0[h].w, a);
        a = fmaf(c1[j].x, q1[h].x, a); a = fmaf(c1[j].y, q1[h].y, a);
        a = fmaf(c1[j].z, q1[h].z, a); a = fmaf(c1[j].w, q1[h].w, a);
        v[j * HS + h] = a;
      }
    const float tot = transpose_reduce32(v);
    const int row = g0 + lane / HS, h = lane % HS;
    if (row < r1 && h < G) out[(size_t)h * ix.m_cap + row] = tot;
  }
}

// ---------------------------------------------------------------------------
// select_v2
// ---------------------------------------------------------------------------
constexpr int S2_THREADS = 512;
constexpr int S2_BAND = 1024;
constexpr int S2_RL = 4096;
constexpr int S2_KEYS = 16384;  // scores cached in smem up to this m

struct Sel2Smem {
  unsigned int keys[S2_KEYS];
  unsigned long long rl[S2_RL];
  double ex[S2_RL];
  int bid_r[S2_BAND];
  double bex_r[S2_BAND];
  int bid_e[S2_BAND];
  double bex_e[S2_BAND];
  unsigned char bsel_e[S2_BAND];
  int hist[2048];
  double q64[256];
  float red[32];
  int wsum[32], wsum2[32], wsum3[32];
  int n_in_r, n_band_r, n_band_e, n_in_e, n_rl, n_el;
  int krem, sel, last;
  int base_r, base_e, base_t;
  float fred;
};

__device__ __forceinline__ float s2_block_reduce(float v, bool is_max, Sel2Smem& sm) {
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

// warp-aggregated append of `val` when `flag`; all lanes of the warp call it
__device__ __forceinline__ void warp_append(bool flag, int val, int* list, int* counter, int cap) {
  const unsigned mk = __ballot_sync(FULLMASK, flag);
  if (!mk) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(mk) - 1) base = atomicAdd(counter, __popc(mk));
  base = __shfl_sync(FULLMASK, base, __ffs(mk) - 1);
  if (flag) {
    const int pos = base + __popc(mk & ((1u << lane) - 1u));
    if (pos < cap) list[pos] = val;
  }
}

__device__ unsigned int s2_kth_largest(const unsigned int* keys, const float* sg, int m, int K, Sel2Smem& sm) {
  // keys: smem-cached order keys, or nullptr to derive them from sg (global)
  const int shifts[3] = {21, 10, 0};
  const unsigned widths[3] = {11, 11, 10};
  unsigned int prefix = 0, pmask = 0;
  if (threadIdx.x == 0) sm.krem = K;
  for (int pass = 0; pass < 3; pass++) {
    const int sh = shifts[pass];
    const unsigned dm = (1u << widths[pass]) - 1u;
    const int nb = 1 << widths[pass];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) sm.hist[b] = 0;
    __syncthreads();
    for (int base = 0; base < m; base += blockDim.x) {
      const int i = base + threadIdx.x;
      unsigned key = i < m ? (keys ? keys[i] : f2u_ord(sg[i])) : 0u;
      const bool act = i < m && (key & pmask) == prefix;
      const unsigned am = __ballot_sync(FULLMASK, act);
      if (act) {
        const unsigned dg = (key >> sh) & dm;
        const unsigned peers = __match_any_sync(am, dg);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sm.hist[dg], __popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x, per = nb / 32;
      int local = 0;
      for (int j = 0; j < per; j++) local += sm.hist[per * lane + j];
      int suf = local;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_down_sync(FULLMASK, suf, o);
        if (lane + o < 32) suf += t;
      }
      const int krem = sm.krem;
      const int above = suf - local;
      const unsigned ball = __ballot_sync(FULLMASK, above < krem && suf >= krem);
      const int owner = __ffs(ball) - 1;
      if (lane == owner) {
        int acc = above, sel = per * lane;
        for (int j = per - 1; j >= 0; j--) {
          const int h = sm.hist[per * lane + j];
          if (acc + h >= krem) { sel = per * lane + j; break; }
          acc += h;
        }
        sm.krem = krem - acc;
        sm.sel = sel;
      }
    }
    __syncthreads();
    prefix |= (unsigned)sm.sel << sh;
    pmask |= dm << sh;
    __syncthreads();
  }
  return prefix;
}

__device__ __forceinline__ double exact_score2(const IndexView& ix, int u, int c, int m, int d, int bt,
                                               const double* q64) {
  const double* row = ix.C64 + ((size_t)u * ix.m_cap + c) * d;
  return dgemv_row(row, q64, d, gemv_row_class(c, m, d, bt));
}

__device__ __forceinline__ unsigned long long s2_key(float s, int id) {
  return ((unsigned long long)(~f2u_ord(s)) << 32) | (unsigned int)id;
}
__device__ __forceinline__ float s2_score(unsigned long long k) { return u2f_ord(~(unsigned int)(k >> 32)); }
__device__ __forceinline__ int s2_id(unsigned long long k) { return (int)(k & 0xffffffffu); }
__device__ __forceinline__ bool s2_better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

// union of the unit's G zones (runs in the last CTA of the unit)
__device__ void s2_union(const IndexView& ix, const StepView& sv, int u, int m, Sel2Smem& sm) {
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const int* coff = ix.cl_off + (size_t)u * ix.m_cap;
  int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  int32_t* rpre = sv.ru_pre + (size_t)u * (sv.ru_cap + 1);
  int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  int32_t* trow = sv.rtok_row + (size_t)u * sv.rt_cap;
  uint8_t* tmk = sv.rtok_mask + (size_t)u * sv.rt_cap;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) { sm.base_r = 0; sm.base_e = 0; sm.base_t = 0; }
  __syncthreads();
  for (int c0 = 0; c0 < m; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    const uint32_t z = c < m ? __ldcg(zm + c) : 0u;
    if (c < m && z) zm[c] = 0u;
    const int fr = (z & 0xffu) ? 1 : 0, fe = (z & 0xff00u) ? 1 : 0;
    const int sz = fr ? csize[c] : 0;
    int xr = fr, xe = fe, xt = sz;
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(FULLMASK, xr, o), b = __shfl_up_sync(FULLMASK, xe, o),
                t = __shfl_up_sync(FULLMASK, xt, o);
      if (lane >= o) { xr += a; xe += b; xt += t; }
    }
    if (lane == 31) { sm.wsum[w] = xr; sm.wsum2[w] = xe; sm.wsum3[w] = xt; }
    __syncthreads();
    if (w == 0) {
      const int nw = blockDim.x >> 5;
      int a = lane < nw ? sm.wsum[lane] : 0, b = lane < nw ? sm.wsum2[lane] : 0,
          t = lane < nw ? sm.wsum3[lane] : 0;
      int ia = a, ib = b, it = t;
      for (int o = 1; o < 32; o <<= 1) {
        const int pa = __shfl_up_sync(FULLMASK, ia, o), pb = __shfl_up_sync(FULLMASK, ib, o),
                  pt = __shfl_up_sync(FULLMASK, it, o);
        if (lane >= o) { ia += pa; ib += pb; it += pt; }
      }
      if (lane < nw) { sm.wsum[lane] = ia - a; sm.wsum2[lane] = ib - b; sm.wsum3[lane] = it - t; }
    }
    __syncthreads();
    const int pr = sm.base_r + sm.wsum[w] + xr - fr;
    const int pe = sm.base_e + sm.wsum2[w] + xe - fe;
    const int pt = sm.base_t + sm.wsum3[w] + xt - sz;
    if (fr) {
      if (pr < sv.ru_cap && pt + sz <= sv.rt_cap) {
        ru[pr] = c;
        rmk[pr] = (uint8_t)(z & 0xffu);
        rpre[pr] = pt;
        const int o = coff[c];
        for (int j = 0; j < sz; j++) { trow[pt + j] = o + j; tmk[pt + j] = (uint8_t)(z & 0xffu); }
      } else {
        set_status(sv.status, kErrUnion);
      }
    }
    if (fe) {
      if (pe < sv.eu_cap) { eu[pe] = c; emk[pe] = (uint8_t)((z >> 8) & 0xffu); }
      else set_status(sv.status, kErrUnion);
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) { sm.base_r = pr + fr; sm.base_e = pe + fe; sm.base_t = pt + sz; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int nr = min(sm.base_r, sv.ru_cap);
    rpre[nr] = sm.base_t;
    sv.cnt[u * 4 + 0] = nr;
    sv.cnt[u * 4 + 1] = min(sm.base_t, sv.rt_cap);
    sv.cnt[u * 4 + 2] = min(sm.base_e, sv.eu_cap);
  }
}

__global__ void __launch_bounds__(S2_THREADS) select_v2_kernel(IndexView ix, StepView sv, SelParams p) {
  extern __shared__ __align__(16) unsigned char s2_raw[];
  Sel2Smem& sm = *reinterpret_cast<Sel2Smem*>(s2_raw);
  const int G = p.G, d = p.d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int m = sv.m[u];
  const int lane = threadIdx.x & 31;
  float* tailp = sv.tail + ((size_t)u * G + g) * 4;
  int r = 0, e = 0;
  if (m > 0) {
    r = (int)floor(p.retrieval_fraction * (double)m + 0.5);
    if (r < 1) r = 1;
    if (r > m) r = m;
    e = (int)floor(p.estimation_fraction * (double)m + 0.5);
    if (e > m - r) e = m - r;
  }
  if (threadIdx.x == 0 && g == 0) { sv.nr[u] = r; sv.ne[u] = e; }
  const float* s = sv.scores + ((size_t)u * G + g) * ix.m_cap;
  const float* q = sv.q + ((size_t)u * G + g) * d;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const bool ok = m > 0 && r <= S2_RL;
  const bool cached = m <= S2_KEYS;
  if (m > 0 && !ok) set_status(sv.status, kErrBandOverflow);
  if (ok) {
    for (int t = threadIdx.x; t < d; t += blockDim.x) sm.q64[t] = (double)q[t];
    float cm = 0.f;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      if (cached) sm.keys[c] = f2u_ord(s[c]);
      cm = fmaxf(cm, ix.Cnorm[(size_t)u * ix.m_cap + c]);
    }
    float qq = 0.f;
    for (int t = threadIdx.x; t < d; t += blockDim.x) qq = fmaf(q[t], q[t], qq);
    const float qn2 = s2_block_reduce(qq, false, sm);
    const float cmax = s2_block_reduce(cm, true, sm);
    const double uu = 5.9604644775390625e-08;
    const double gam = (double)d * uu / (1.0 - (double)d * uu);
    const double B = 2.0 * (gam + uu + 1e-13) * (1.0 + 1e-5) * sqrt((double)qn2) * (1.0 + 1e-5) *
                     (double)cmax * (1.0 + 1e-5);
    const double B2 = 2.0 * B;
    const unsigned* kp = cached ? sm.keys : nullptr;
    const float tau_r = u2f_ord(s2_kth_largest(kp, s, m, r, sm));
    const float tau_e = e > 0 ? u2f_ord(s2_kth_largest(kp, s, m, r + e, sm)) : 0.f;
    if (threadIdx.x == 0) { sm.n_in_r = 0; sm.n_band_r = 0; sm.n_band_e = 0; sm.n_in_e = 0; sm.n_rl = 0; }
    __syncthreads();
    int my_in_e = 0;
    for (int base = 0; base < m; base += blockDim.x) {
      const int c = base + threadIdx.x;
      const bool act = c < m;
      const double sc = act ? (double)s[c] : -INFINITY;
      const bool in_r = act && sc > (double)tau_r + B2;
      const bool bd_r = act && !in_r && sc >= (double)tau_r - B2;
      warp_append(in_r, c, reinterpret_cast<int*>(sm.ex), &sm.n_rl, S2_RL);  // ids staged in ex[]
      warp_append(bd_r, c, sm.bid_r, &sm.n_band_r, S2_BAND);
      if (e > 0) {
        const bool in_e = act && sc > (double)tau_e + B2;
        const bool bd_e = act && !in_e && sc >= (double)tau_e - B2;
        my_in_e += in_e ? 1 : 0;
        warp_append(bd_e, c, sm.bid_e, &sm.n_band_e, S2_BAND);
      }
    }
    my_in_e = __reduce_add_sync(FULLMASK, my_in_e);
    if (lane == 0 && my_in_e) atomicAdd(&sm.n_in_e, my_in_e);
    __syncthreads();
    const int nin_r = sm.n_rl, nbr = sm.n_band_r, nbe = sm.n_band_e, nin_e = sm.n_in_e;
    const bool bad = nbr > S2_BAND || nbe > S2_BAND || nin_r > r || nin_r + nbr < r ||
                     (e > 0 && (nin_e > r + e || nin_e + nbe < r + e));
    if (bad) {
      set_status(sv.status, kErrBandOverflow);
    } else {
      // certain-in ids were staged in ex[] as ints: turn them into sort keys
      const int* staged = reinterpret_cast<const int*>(sm.ex);
      for (int i = threadIdx.x; i < nin_r; i += blockDim.x) { const int c = staged[i]; sm.rl[i] = s2_key(s[c], c); }
      for (int i = threadIdx.x; i < nbr; i += blockDim.x)
        sm.bex_r[i] = exact_score2(ix, u, sm.bid_r[i], m, d, p.blas_threads, sm.q64);
      for (int i = threadIdx.x; i < nbe; i += blockDim.x)
        sm.bex_e[i] = exact_score2(ix, u, sm.bid_e[i], m, d, p.blas_threads, sm.q64);
      __syncthreads();
      const int need_r = r - nin_r;
      for (int i = threadIdx.x; i < nbr; i += blockDim.x) {
        int rank = 0;
        for (int j = 0; j < nbr; j++) rank += s2_better(sm.bex_r[j], sm.bid_r[j], sm.bex_r[i], sm.bid_r[i]) ? 1 : 0;
        if (rank < need_r) sm.rl[nin_r + rank] = s2_key(s[sm.bid_r[i]], sm.bid_r[i]);
      }
      const int need_e = r + e - nin_e;
      for (int i = threadIdx.x; i < nbe; i += blockDim.x) {
        int rank = 0;
        for (int j = 0; j < nbe; j++) rank += s2_better(sm.bex_e[j], sm.bid_e[j], sm.bex_e[i], sm.bid_e[i]) ? 1 : 0;
        sm.bsel_e[i] = rank < need_e ? 1 : 0;
      }
      __syncthreads();
      // bitonic sort of the r retrieval keys
      int npow = 1;
      while (npow < r) npow <<= 1;
      for (int i = r + threadIdx.x; i < npow; i += blockDim.x) sm.rl[i] = ~0ull;
      __syncthreads();
      for (int k = 2; k <= npow; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = threadIdx.x; i < npow; i += blockDim.x) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const unsigned long long a = sm.rl[i], b = sm.rl[ixj];
              if ((a > b) == ((i & k) == 0)) { sm.rl[i] = b; sm.rl[ixj] = a; }
            }
          }
          __syncthreads();
        }
      // clumps of neighbours closer than 2B: exact scores, exact order
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const double si = (double)s2_score(sm.rl[i]);
        const bool cl = (i > 0 && (double)s2_score(sm.rl[i - 1]) - si <= B2) ||
                        (i + 1 < r && si - (double)s2_score(sm.rl[i + 1]) <= B2);
        sm.ex[i] = cl ? exact_score2(ix, u, s2_id(sm.rl[i]), m, d, p.blas_threads, sm.q64) : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const double si = (double)s2_score(sm.rl[i]);
        const bool lp = i > 0 && (double)s2_score(sm.rl[i - 1]) - si <= B2;
        const bool ln = i + 1 < r && si - (double)s2_score(sm.rl[i + 1]) <= B2;
        if (!lp && ln) {
          int end = i + 1;
          while (end + 1 < r && (double)s2_score(sm.rl[end]) - (double)s2_score(sm.rl[end + 1]) <= B2) end++;
          for (int a = i + 1; a <= end; a++) {
            const unsigned long long kk = sm.rl[a];
            const double ev = sm.ex[a];
            int b = a - 1;
            while (b >= i && s2_better(ev, s2_id(kk), sm.ex[b], s2_id(sm.rl[b]))) {
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
      int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const int c = s2_id(sm.rl[i]);
        rl_out[i] = c;
        atomicOr(zm + c, 1u << g);
      }
      __threadfence_block();
      __syncthreads();
      int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
      if (threadIdx.x == 0) sm.n_el = 0;
      __syncthreads();
      if (e > 0) {
        for (int base = 0; base < m; base += blockDim.x) {
          const int c = base + threadIdx.x;
          const bool f = c < m && (double)s[c] > (double)tau_e + B2 && !(__ldcg(zm + c) & (1u << g));
          if (f) atomicOr(zm + c, 1u << (8 + g));
          if (el_out) warp_append(f, c, el_out, &sm.n_el, sv.e_cap);
        }
        for (int i = threadIdx.x; i < nbe; i += blockDim.x) {
          const int c = sm.bid_e[i];
          if (sm.bsel_e[i] && !(__ldcg(zm + c) & (1u << g))) {
            atomicOr(zm + c, 1u << (8 + g));
            if (el_out) el_out[atomicAdd(&sm.n_el, 1)] = c;
          }
        }
      }
      __syncthreads();
      if (p.need_tail || p.need_allc) {
        const float isd = p.inv_sqrt_d;
        float mx_t = -INFINITY, mx_a = -INFINITY;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          const float v = s[c] * isd;
          mx_a = fmaxf(mx_a, v);
          if (!(__ldcg(zm + c) & ((1u << g) | (1u << (8 + g))))) mx_t = fmaxf(mx_t, v);
        }
        mx_t = s2_block_reduce(mx_t, true, sm);
        mx_a = s2_block_reduce(mx_a, true, sm);
        float dt = 0.f, da = 0.f;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          const float v = s[c] * isd;
          const float sz = (float)csize[c];
          da += sz * expf(v - mx_a);
          if (!(__ldcg(zm + c) & ((1u << g) | (1u << (8 + g))))) dt += sz * expf(v - mx_t);
        }
        dt = s2_block_reduce(dt, false, sm);
        da = s2_block_reduce(da, false, sm);
        if (threadIdx.x == 0) { tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da; }
      }
    }
  }
  if (!ok && threadIdx.x == 0) { tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f; }
  // ---- the last CTA of the unit builds the unions ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm.last = (atomicAdd(sv.sel_done + u, 1) == G - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  if (threadIdx.x == 0) sv.sel_done[u] = 0;
  s2_union(ix, sv, u, m, sm);
}

size_t select_v2_smem_bytes() { return sizeof(Sel2Smem); }

// ---------------------------------------------------------------------------
// attend_v2
// grid = (S, U), block = 256 (8 warps); one CTA handles 1/S of its unit's
// work items [steady tokens | retrieved tokens | estimation rows].
// ---------------------------------------------------------------------------
template <typename T, int DL> struct RowLoad;
template <> struct RowLoad<__nv_bfloat16, 4> {
  using R = uint2;
  static __device__ __forceinline__ R ld(const __nv_bfloat16* p) { return __ldcs(reinterpret_cast<const uint2*>(p)); }
  static __device__ __forceinline__ void cvt(const R& r, float* o) {
    float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
  }
  static __device__ __forceinline__ R zero() { return make_uint2(0u, 0u); }
};
template <> struct RowLoad<__nv_bfloat16, 2> {
  using R = unsigned int;
  static __device__ __forceinline__ R ld(const __nv_bfloat16* p) { return __ldcs(reinterpret_cast<const unsigned int*>(p)); }
  static __device__ __forceinline__ void cvt(const R& r, float* o) {
    float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r));
    o[0] = a.x; o[1] = a.y;
  }
  static __device__ __forceinline__ R zero() { return 0u; }
};
template <> struct RowLoad<float, 4> {
  using R = float4;
  static __device__ __forceinline__ R ld(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ void cvt(const R& r, float* o) { o[0] = r.x; o[1] = r.y; o[2] = r.z; o[3] = r.w; }
  static __device__ __forceinline__ R zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <> struct RowLoad<float, 2> {
  using R = float2;
  static __device__ __forceinline__ R ld(const float* p) { return __ldcs(reinterpret_cast<const float2*>(p)); }
  static __device__ __forceinline__ void cvt(const R& r, float* o) { o[0] = r.x; o[1] = r.y; }
  static __device__ __forceinline__ R zero() { return make_float2(0.f, 0.f); }
};

template <int HS>
struct SoftState {
  float M[HS], D[HS];
};

// online-softmax update for one group.  x = this lane's masked logit for
// (token lane/HS, head lane%HS); wz = weight of the lane's row in the
// denominator (1 for tokens, cluster size for estimation rows).
// Returns p (the lane's softmax weight for the numerator) and fills alpha[].
template <int HS>
__device__ __forceinline__ float softmax_group(float x, float wz, SoftState<HS>& st, float (&alpha)[HS]) {
  float mx = x;
#pragma unroll
  for (int off = HS; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(FULLMASK, mx, off));
  const int lane = threadIdx.x & 31;
  const int h_own = lane % HS;
  float mnew_own = fmaxf(st.M[0], mx);
#pragma unroll
  for (int h = 0; h < HS; h++)
    if (h == h_own) mnew_own = fmaxf(st.M[h], mx);
  const float pw = (x == -INFINITY) ? 0.f : __expf(x - mnew_own);
  float ps = pw * wz;
#pragma unroll
  for (int off = HS; off < 32; off <<= 1) ps += __shfl_xor_sync(FULLMASK, ps, off);
#pragma unroll
  for (int h = 0; h < HS; h++) {
    const float mn = __shfl_sync(FULLMASK, mnew_own, h);
    const float sd = __shfl_sync(FULLMASK, ps, h);
    const float mo = st.M[h];
    alpha[h] = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
    if (mn == -INFINITY) alpha[h] = 1.f;
    st.D[h] = st.D[h] * alpha[h] + sd;
    st.M[h] = mn;
  }
  return pw;
}

template <typename T, int DL, int HS, bool FULL>
__global__ void __launch_bounds__(256, 1) attend_v2_kernel(IndexView ix, SteadyView st, StepView sv, AttnParams p,
                                                            const int32_t* __restrict__ n_store) {
  constexpr int RG = 32 / HS;
  using LD = RowLoad<T, DL>;
  using LV = RowLoad<float, DL>;
  const int s_idx = blockIdx.x, u = blockIdx.y, S = gridDim.x;
  const int G = p.G, d = p.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(16) float wp[];  // [8 warps][HS][2 + d]
  const int n_st = st.n[u];
  const int n_rt = FULL ? n_store[u] : sv.cnt[u * 4 + 1];
  const int n_eu = FULL ? 0 : sv.cnt[u * 4 + 2];
  const long long N = (long long)n_st + n_rt + n_eu;
  const int ib = (int)(N * s_idx / S), ie = (int)(N * (s_idx + 1) / S);
  const float isd = p.inv_sqrt_d;
  // q slices (pre-scaled by 1/sqrt(d))
  float qv[HS][DL];
#pragma unroll
  for (int h = 0; h < HS; h++)
#pragma unroll
    for (int k = 0; k < DL; k++)
      qv[h][k] = h < G ? sv.q[((size_t)u * G + h) * d + lane * DL + k] * isd : 0.f;
  const T* stk = (const T*)st.k + (size_t)u * st.t_cap * d;
  const T* stv = (const T*)st.v + (size_t)u * st.t_cap * d;
  const T* sk = (const T*)ix.store_k + (size_t)u * ix.s_cap * d;
  const T* svv = (const T*)ix.store_v + (size_t)u * ix.s_cap * d;
  const int32_t* trow = FULL ? nullptr : sv.rtok_row + (size_t)u * sv.rt_cap;
  const uint8_t* tmk = FULL ? nullptr : sv.rtok_mask + (size_t)u * sv.rt_cap;
  const int32_t* eu = FULL ? nullptr : sv.eu_ids + (size_t)u * sv.eu_cap;
  const uint8_t* emk = FULL ? nullptr : sv.eu_mask + (size_t)u * sv.eu_cap;
  const float* scr = FULL ? nullptr : sv.scores + (size_t)u * G * ix.m_cap;
  const int32_t* csz = ix.cl_size + (size_t)u * ix.m_cap;
  const float* vsb = ix.VS32 + (size_t)u * ix.m_cap * d;
  const int allmask = (1 << G) - 1;
  const int j_own = lane / HS, h_own = lane % HS;

  for (int kind = 0; kind < 3; kind++) {
    const int kb = kind == 0 ? 0 : (kind == 1 ? n_st : n_st + n_rt);
    const int ke = kind == 0 ? n_st : (kind == 1 ? n_st + n_rt : (int)N);
    const int lo = max(ib, kb), hi = min(ie, ke);
    if (lo >= hi) continue;  // uniform over the CTA
    SoftState<HS> ss;
#pragma unroll
    for (int h = 0; h < HS; h++) { ss.M[h] = -INFINITY; ss.D[h] = 0.f; }
    float acc[HS][DL];
#pragma unroll
    for (int h = 0; h < HS; h++)
#pragma unroll
      for (int k = 0; k < DL; k++) acc[h][k] = 0.f;

    if (kind < 2) {
      // ---------------- token groups: exact attention ----------------
      typename LD::R kr[2][RG], vr[2][RG];
      int rowv[2];  // row of token j_own (for masks)
      int mk[2];
      auto issue = [&](int buf, int g0) {
#pragma unroll
        for (int j = 0; j < RG; j++) {
          const int it = g0 + j;
          if (it < hi) {
            const T* kp;
            const T* vp;
            if (kind == 0) {
              kp = stk + (size_t)(it - kb) * d; vp = stv + (size_t)(it - kb) * d;
            } else {
              const long long row = FULL ? (long long)(it - kb) : (long long)trow[it - kb];
              kp = sk + (size_t)row * d; vp = svv + (size_t)row * d;
            }
            kr[buf][j] = LD::ld(kp + lane * DL);
            vr[buf][j] = LD::ld(vp + lane * DL);
          } else {
            kr[buf][j] = LD::zero();
            vr[buf][j] = LD::zero();
          }
        }
        const int itj = g0 + j_own;
        mk[buf] = itj < hi ? ((kind == 0 || FULL) ? allmask : (int)tmk[itj - kb]) : 0;
        rowv[buf] = itj;
      };
      auto compute = [&](int buf) {
        float v[32];
#pragma unroll
        for (int j = 0; j < RG; j++) {
          float kf[DL];
          LD::cvt(kr[buf][j], kf);
#pragma unroll
          for (int h = 0; h < HS; h++) {
            float a = 0.f;
#pragma unroll
            for (int k = 0; k < DL; k++) a = fmaf(kf[k], qv[h][k], a);
            v[j * HS + h] = a;
          }
        }
        float x = transpose_reduce32(v);
        if (!((mk[buf] >> h_own) & 1)) x = -INFINITY;
        float alpha[HS];
        const float pw = softmax_group<HS>(x, 1.f, ss, alpha);
#pragma unroll
        for (int h = 0; h < HS; h++)
#pragma unroll
          for (int k = 0; k < DL; k++) acc[h][k] *= alpha[h];
#pragma unroll
        for (int j = 0; j < RG; j++) {
          float vf[DL];
          LD::cvt(vr[buf][j], vf);
#pragma unroll
          for (int h = 0; h < HS; h++) {
            const float pj = __shfl_sync(FULLMASK, pw, j * HS + h);
#pragma unroll
            for (int k = 0; k < DL; k++) acc[h][k] = fmaf(pj, vf[k], acc[h][k]);
          }
        }
      };
      const int stride = 8 * RG;
      int g0 = lo + warp * RG;
      if (g0 < hi) issue(0, g0);
      while (g0 < hi) {
        const int g1 = g0 + stride;
        if (g1 < hi) issue(1, g1);
        compute(0);
        if (g1 >= hi) break;
        const int g2 = g1 + stride;
        if (g2 < hi) issue(0, g2);
        compute(1);
        g0 = g2;
      }
    } else {
      // ---------------- estimation rows: centroid-weighted value sums ----
      typename LV::R vr[2][RG];
      float xs[2], wz[2];
      int okr[2];
      auto issue = [&](int buf, int g0) {
#pragma unroll
        for (int j = 0; j < RG; j++) {
          const int it = g0 + j;
          if (it < hi) {
            const int c = eu[it - kb];
            vr[buf][j] = LV::ld(vsb + (size_t)c * d + lane * DL);
          } else {
            vr[buf][j] = LV::zero();
          }
        }
        const int itj = g0 + j_own;
        float x = -INFINITY, w = 0.f;
        if (itj < hi) {
          const int c = eu[itj - kb];
          if ((emk[itj - kb] >> h_own) & 1) x = scr[(size_t)h_own * ix.m_cap + c] * isd;
          w = (float)csz[c];
        }
        xs[buf] = x; wz[buf] = w; okr[buf] = 1;
      };
      auto compute = [&](int buf) {
        float alpha[HS];
        const float pw = softmax_group<HS>(xs[buf], wz[buf], ss, alpha);
#pragma unroll
        for (int h = 0; h < HS; h++)
#pragma unroll
          for (int k = 0; k < DL; k++) acc[h][k] *= alpha[h];
#pragma unroll
        for (int j = 0; j < RG; j++) {
          float vf[DL];
          LV::cvt(vr[buf][j], vf);
#pragma unroll
          for (int h = 0; h < HS; h++) {
            const float pj = __shfl_sync(FULLMASK, pw, j * HS + h);
#pragma unroll
            for (int k = 0; k < DL; k++) acc[h][k] = fmaf(pj, vf[k], acc[h][k]);
          }
        }
      };
      const int stride = 8 * RG;
      int g0 = lo + warp * RG;
      if (g0 < hi) issue(0, g0);
      while (g0 < hi) {
        const int g1 = g0 + stride;
        if (g1 < hi) issue(1, g1);
        compute(0);
        if (g1 >= hi) break;
        const int g2 = g1 + stride;
        if (g2 < hi) issue(0, g2);
        compute(1);
        g0 = g2;
      }
    }
    // ---- per-warp partials to smem, then combine over the 8 warps ----
    const int stride_w = 2 + d;
#pragma unroll
    for (int h = 0; h < HS; h++) {
      float* dst = wp + ((size_t)warp * HS + h) * stride_w;
      if (lane == 0) { dst[0] = ss.M[h]; dst[1] = ss.D[h]; }
#pragma unroll
      for (int k = 0; k < DL; k++) dst[2 + lane * DL + k] = acc[h][k];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * (d + 2); idx += blockDim.x) {
      const int h = idx / (d + 2), t = idx % (d + 2);
      float Mx = -INFINITY;
      for (int w = 0; w < 8; w++) Mx = fmaxf(Mx, wp[((size_t)w * HS + h) * stride_w]);
      float acc_t = 0.f;
      for (int w = 0; w < 8; w++) {
        const float* src = wp + ((size_t)w * HS + h) * stride_w;
        if (src[1] > 0.f) {
          const float sc = __expf(src[0] - Mx);
          acc_t += (t == 0 ? 0.f : (t == 1 ? src[1] : src[t])) * sc;
        }
      }
      float* out = sv.part + ((((size_t)u * S + s_idx) * G + h) * 3 + kind) * (size_t)stride_w;
      out[t] = t == 0 ? Mx : acc_t;
    }
    __syncthreads();
  }
  // kinds with no items in this CTA: mark their partials empty
  for (int kind = 0; kind < 3; kind++) {
    const int kb = kind == 0 ? 0 : (kind == 1 ? n_st : n_st + n_rt);
    const int ke = kind == 0 ? n_st : (kind == 1 ? n_st + n_rt : (int)N);
    if (max(ib, kb) < min(ie, ke)) continue;
    for (int h = threadIdx.x; h < G; h += blockDim.x) {
      float* out = sv.part + ((((size_t)u * S + s_idx) * G + h) * 3 + kind) * (size_t)(2 + d);
      out[0] = -INFINITY;
      out[1] = 0.f;
    }
  }
}

size_t attend_v2_smem_bytes(int d, int HS) { return (size_t)8 * HS * (2 + d) * sizeof(float); }

#define WK_INST_ATT2(T, DL, HS)                                                                          \
  template __global__ void attend_v2_kernel<T, DL, HS, false>(IndexView, SteadyView, StepView, AttnParams, \
                                                             const int32_t*);                             \
  template __global__ void attend_v2_kernel<T, DL, HS, true>(IndexView, SteadyView, StepView, AttnParams,  \
                                                            const int32_t*);
WK_INST_ATT2(__nv_bfloat16, 4, 4)
WK_INST_ATT2(__nv_bfloat16, 4, 8)
WK_INST_ATT2(__nv_bfloat16, 2, 4)
WK_INST_ATT2(__nv_bfloat16, 2, 8)
WK_INST_ATT2(float, 4, 4)
WK_INST_ATT2(float, 4, 8)
WK_INST_ATT2(float, 2, 4)
WK_INST_ATT2(float, 2, 8)
template __global__ void score_v2_kernel<4>(IndexView, StepView, int, int, int);
template __global__ void score_v2_kernel<8>(IndexView, StepView, int, int, int);

}  // namespace wk
