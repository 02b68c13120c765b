// select_v5.cu -- exact zone planning, latency-lean version.
//
// Produces the same bits as the reference's rank_clusters + plan_zones
// (index.py:61-93): the ordered retrieval list (top r by fp64 q.C, ties to the
// lower id) and the estimation set (the next e).  Design for many resident
// CTAs (256 threads, <= 64 registers, ~24 KB smem): scores are re-read from L2
// (just written by the scoring kernel) with vectorised loads; the r-th and
// (r+e)-th largest approximate scores come from one 512-bucket histogram plus
// rank-by-counting inside the two boundary buckets; the candidates
// (certain-in + band) are ordered by counting; band rows and the members of
// "clumps" (neighbours closer than the error bound) are re-scored exactly in
// ONE warp-parallel round with the reference dgemv recipe.  The last CTA of a
// unit builds the union lists.
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

#define S5_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 4096) { long long _t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(_t)); g_sel_dbg[blockIdx.x][i] = _t; } } while (0)

constexpr int S5_T = 256;
constexpr int S5_NB = 512;       // histogram buckets
constexpr int S5_LIST = 512;     // boundary-bucket capacity
constexpr int S5_CAND = 512;     // certain-in + band candidates (>= r + band)
constexpr int S5_BAND = 256;

struct Sel5Smem {
  int hist[S5_NB];
  unsigned long long l1[S5_LIST];
  unsigned long long l2[S5_LIST];
  unsigned long long cand[S5_CAND];   // candidate keys (approx desc, id asc)
  unsigned long long cs[S5_CAND];     // candidates in order
  unsigned long long fin[S5_CAND];    // final retrieval order
  double cex[S5_CAND];                // exact scores of ordered candidates (band / clump rows)
  double fex[S5_CAND];                // exact scores in final order
  int be_id[S5_BAND];                 // band rows around tau_{r+e}
  double be_ex[S5_BAND];
  unsigned char be_sel[S5_BAND];
  double q64[256];
  float red[8];
  int wsum[8], wsum2[8], wsum3[8];
  int n1, n2, above1, above2, b1, b2, ncand, nband_r, nband_e, n_in_e, n_el, ovf, last, ne_sel;
  int base_r, base_e, base_t;
  float fred;
};

__device__ __forceinline__ float s5_reduce(float v, bool is_max, Sel5Smem& sm) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm.red[w] = v;
  __syncthreads();
  if (w == 0) {
    float r = lane < (int)(blockDim.x >> 5) ? sm.red[lane] : (is_max ? -INFINITY : 0.f);
    r = is_max ? warp_max(r) : warp_sum(r);
    if (lane == 0) sm.fred = r;
  }
  __syncthreads();
  return sm.fred;
}

__device__ __forceinline__ unsigned long long s5_key(float s, int id) {
  return ((unsigned long long)(~f2u_ord(s)) << 32) | (unsigned int)id;
}
__device__ __forceinline__ float s5_score(unsigned long long k) { return u2f_ord(~(unsigned int)(k >> 32)); }
__device__ __forceinline__ int s5_id(unsigned long long k) { return (int)(k & 0xffffffffu); }
__device__ __forceinline__ bool s5_better(double a, int ia, double b, int ib) { return a > b || (a == b && ia < ib); }

// exact dgemv-recipe score of one fp64 centroid row by one warp (d % 32 == 0)
__device__ __forceinline__ double s5_exact_warp(const double* row, const double* q64, int d, int cls) {
  const int lane = threadIdx.x & 31;
  const int per = d >> 5;
  double a[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    a[i] = i < per ? __ldcg(row + lane * per + i) : 0.0;
    x[i] = i < per ? q64[lane * per + i] : 0.0;
  }
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  for (int l = 0; l < 32; l++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (i < per) {
        const double av = __shfl_sync(0xffffffffu, a[i], l), xv = __shfl_sync(0xffffffffu, x[i], l);
        const int t = l * per + i;
        const int j = cls == 1 ? (t & 1) : (t & 3);
        double& acc = j == 0 ? acc0 : (j == 1 ? acc1 : (j == 2 ? acc2 : acc3));
        acc = cls == 0 ? __fma_rn(av, xv, acc) : __dadd_rn(acc, __dmul_rn(av, xv));
      }
    }
  }
  if (cls == 1) return __dadd_rn(0.0, __dadd_rn(acc0, acc1));
  return __dadd_rn(0.0, __dadd_rn(__dadd_rn(acc0, acc2), __dadd_rn(acc1, acc3)));
}

__device__ __forceinline__ void s5_append(bool flag, unsigned long long val, unsigned long long* list, int* counter,
                                          int cap, int* ovf) {
  const unsigned mk = __ballot_sync(0xffffffffu, flag);
  if (!mk) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mk) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mk));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (flag) {
    const int pos = base + __popc(mk & ((1u << lane) - 1u));
    if (pos < cap) list[pos] = val; else *ovf = 1;
  }
}

// ascending rank-by-counting of n unique keys a[] into out[]
__device__ __forceinline__ void s5_rank_sort(const unsigned long long* a, int n, unsigned long long* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long k = a[i];
    int rk = 0;
    for (int j = 0; j < n; j++) rk += a[j] < k ? 1 : 0;
    out[rk] = k;
  }
}

__device__ __forceinline__ void s5_scan3(int& a, int& b, int& c, int& ta, int& tb, int& tc, Sel5Smem& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int xa = a, xb = b, xc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int pa = __shfl_up_sync(0xffffffffu, xa, o), pb = __shfl_up_sync(0xffffffffu, xb, o),
              pc = __shfl_up_sync(0xffffffffu, xc, o);
    if (lane >= o) { xa += pa; xb += pb; xc += pc; }
  }
  if (lane == 31) { sm.wsum[w] = xa; sm.wsum2[w] = xb; sm.wsum3[w] = xc; }
  __syncthreads();
  if (w == 0) {
    int va = lane < nw ? sm.wsum[lane] : 0, vb = lane < nw ? sm.wsum2[lane] : 0, vc = lane < nw ? sm.wsum3[lane] : 0;
    int ia = va, ib = vb, ic = vc;
    for (int o = 1; o < 32; o <<= 1) {
      const int pa = __shfl_up_sync(0xffffffffu, ia, o), pb = __shfl_up_sync(0xffffffffu, ib, o),
                pc = __shfl_up_sync(0xffffffffu, ic, o);
      if (lane >= o) { ia += pa; ib += pb; ic += pc; }
    }
    if (lane < nw) { sm.wsum[lane] = ia - va; sm.wsum2[lane] = ib - vb; sm.wsum3[lane] = ic - vc; }
    if (lane == nw - 1) { sm.base_r = ia; sm.base_e = ib; sm.base_t = ic; }
  }
  __syncthreads();
  const int ea = sm.wsum[w] + xa - a, eb = sm.wsum2[w] + xb - b, ec = sm.wsum3[w] + xc - c;
  ta = sm.base_r; tb = sm.base_e; tc = sm.base_t;
  a = ea; b = eb; c = ec;
  __syncthreads();
}

// union of the unit's zones; thread t owns cluster ids [lo, hi) of length <= 64
__device__ void s5_union(const IndexView& ix, const StepView& sv, int u, int m, Sel5Smem& sm) {
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const int* coff = ix.cl_off + (size_t)u * ix.m_cap;
  const int T = blockDim.x, t = threadIdx.x;
  const int lo = (int)((long long)m * t / T), hi = (int)((long long)m * (t + 1) / T);
  int nr = 0, ne = 0, nt = 0;
  for (int c0 = lo; c0 < hi; c0 += 8) {
    uint32_t z[8];
#pragma unroll
    for (int i = 0; i < 8; i++) z[i] = c0 + i < hi ? __ldcg(zm + c0 + i) : 0u;
    int szv[8];
#pragma unroll
    for (int i = 0; i < 8; i++) szv[i] = (z[i] & 0xffu) ? __ldcg(csize + c0 + i) : 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      nr += (z[i] & 0xffu) ? 1 : 0;
      ne += (z[i] & 0xff00u) ? 1 : 0;
      nt += szv[i];
    }
  }
  int tr, te, tt;
  s5_scan3(nr, ne, nt, tr, te, tt, sm);
  int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  int32_t* rpre = sv.ru_pre + (size_t)u * (sv.ru_cap + 1);
  int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  int32_t* trow = sv.rtok_row + (size_t)u * sv.rt_cap;
  uint8_t* tmk = sv.rtok_mask + (size_t)u * sv.rt_cap;
  for (int c0 = lo; c0 < hi; c0 += 8) {
    uint32_t z[8];
#pragma unroll
    for (int i = 0; i < 8; i++) z[i] = c0 + i < hi ? __ldcg(zm + c0 + i) : 0u;
    int szv[8], off[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      szv[i] = (z[i] & 0xffu) ? __ldcg(csize + c0 + i) : 0;
      off[i] = (z[i] & 0xffu) ? __ldcg(coff + c0 + i) : 0;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int c = c0 + i;
      if (z[i]) zm[c] = 0u;
      if (z[i] & 0xffu) {
        if (nr < sv.ru_cap && nt + szv[i] <= sv.rt_cap) {
          ru[nr] = c;
          rmk[nr] = (uint8_t)(z[i] & 0xffu);
          rpre[nr] = nt;
          for (int j = 0; j < szv[i]; j++) { trow[nt + j] = off[i] + j; tmk[nt + j] = (uint8_t)(z[i] & 0xffu); }
        } else {
          set_status(sv.status, kErrUnion);
        }
        nr++;
        nt += szv[i];
      }
      if (z[i] & 0xff00u) {
        if (ne < sv.eu_cap) { eu[ne] = c; emk[ne] = (uint8_t)((z[i] >> 8) & 0xffu); }
        else set_status(sv.status, kErrUnion);
        ne++;
      }
    }
  }
  if (t == 0) {
    const int n_r = min(tr, sv.ru_cap);
    rpre[n_r] = tt;
    sv.cnt[u * 4 + 0] = n_r;
    sv.cnt[u * 4 + 1] = min(tt, sv.rt_cap);
    sv.cnt[u * 4 + 2] = min(te, sv.eu_cap);
  }
}

__global__ void __launch_bounds__(S5_T, 4) select_v5_kernel(IndexView ix, StepView sv, SelParams p) {
  __shared__ Sel5Smem sm;
  extern __shared__ unsigned short bid16[];  // [m] bucket id of every cluster score
  __shared__ unsigned int rbits[512];         // retrieval set of this head (m <= 16384)
  S5_MARK(0);
  const int G = p.G, d = p.d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int m = sv.m[u];
  const int t = threadIdx.x, T = blockDim.x, lane = t & 31, warp = t >> 5, nwarps = T >> 5;
  float* tailp = sv.tail + ((size_t)u * G + g) * 4;
  int r = 0, e = 0;
  if (m > 0) {
    r = (int)floor(p.retrieval_fraction * (double)m + 0.5);
    if (r < 1) r = 1;
    if (r > m) r = m;
    e = (int)floor(p.estimation_fraction * (double)m + 0.5);
    if (e > m - r) e = m - r;
  }
  if (t == 0 && g == 0) { sv.nr[u] = r; sv.ne[u] = e; }
  const float* s = sv.scores + ((size_t)u * G + g) * ix.m_cap;
  const float* q = sv.q + ((size_t)u * G + g) * d;
  const float* cn = ix.Cnorm + (size_t)u * ix.m_cap;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const double* C64 = ix.C64 + (size_t)u * ix.m_cap * d;
  bool ok = m > 0 && r <= sv.r_cap;
  float bk_mn = 0.f, bk_scale = 0.f;  // bucket map: floor((v - mn) * scale), clamped
  auto bucket = [&](float v) {
    int b = (int)((v - bk_mn) * bk_scale);
    return b < 0 ? 0 : (b >= S5_NB ? S5_NB - 1 : b);
  };
  if (m > 0 && !ok) set_status(sv.status, kErrBandOverflow);
  if (ok) {
    // ---- pass A: min / max of scores, max centroid norm (float4 loads) ----
    float mn = INFINITY, mx = -INFINITY, cm = 0.f;
    const int m4 = m >> 2;
    for (int i = t; i < m4; i += T) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(s) + i);
      const float4 c = __ldcg(reinterpret_cast<const float4*>(cn) + i);
      mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      cm = fmaxf(cm, fmaxf(fmaxf(c.x, c.y), fmaxf(c.z, c.w)));
    }
    for (int i = 4 * m4 + t; i < m; i += T) { const float v = s[i]; mn = fminf(mn, v); mx = fmaxf(mx, v); cm = fmaxf(cm, cn[i]); }
    for (int i = t; i < d; i += T) sm.q64[i] = (double)q[i];
    for (int b = t; b < S5_NB; b += T) sm.hist[b] = 0;
    if (t == 0) { sm.n1 = 0; sm.n2 = 0; sm.ncand = 0; sm.nband_r = 0; sm.nband_e = 0; sm.n_in_e = 0; sm.n_el = 0; sm.ovf = 0; sm.ne_sel = 0; }
    float qq = 0.f;
    for (int i = t; i < d; i += T) qq = fmaf(q[i], q[i], qq);
    const float qn2 = s5_reduce(qq, false, sm);
    const float cmax = s5_reduce(cm, true, sm);
    mn = -s5_reduce(-mn, true, sm);
    mx = s5_reduce(mx, true, sm);
    const double uu = 5.9604644775390625e-08;
    const double gam = (double)d * uu / (1.0 - (double)d * uu);
    const double B = score_error_bound((double)qn2, (double)cmax, d, p.score_fp64 != 0);
    const double B2 = 2.0 * B;
    const float span = mx - mn;
    bk_mn = mn;
    bk_scale = span > 0.f ? (float)S5_NB / span : 0.f;
    S5_MARK(1);
    // ---- pass B: bucket id of every score (one batched read), histogram ----
    for (int i = t; i < m4; i += T) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(s) + i);
      const int k0 = bucket(v.x), k1 = bucket(v.y), k2 = bucket(v.z), k3 = bucket(v.w);
      bid16[4 * i] = (unsigned short)k0; bid16[4 * i + 1] = (unsigned short)k1;
      bid16[4 * i + 2] = (unsigned short)k2; bid16[4 * i + 3] = (unsigned short)k3;
      atomicAdd(&sm.hist[k0], 1); atomicAdd(&sm.hist[k1], 1); atomicAdd(&sm.hist[k2], 1); atomicAdd(&sm.hist[k3], 1);
    }
    for (int i = 4 * m4 + t; i < m; i += T) {
      const int k = bucket(s[i]);
      bid16[i] = (unsigned short)k;
      atomicAdd(&sm.hist[k], 1);
    }
    for (int w = t; w < (m + 31) / 32; w += T) rbits[w] = 0u;
    __syncthreads();
    // buckets holding rank K1 = r and K2 = r + e (descending): thread t owns
    // buckets 511-2t and 510-2t
    {
      const int K1 = r, K2 = e > 0 ? r + e : 0;
      const int b0 = S5_NB - 1 - 2 * t;
      const int h0 = sm.hist[b0], h1 = sm.hist[b0 - 1];
      int x = h0 + h1;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) sm.wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int v = lane < nwarps ? sm.wsum[lane] : 0, iv = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, iv, o);
          if (lane >= o) iv += y;
        }
        if (lane < nwarps) sm.wsum[lane] = iv - v;
      }
      __syncthreads();
      const int ab0 = sm.wsum[warp] + x - (h0 + h1), ab1 = ab0 + h0;
      if (ab0 < K1 && ab0 + h0 >= K1) { sm.b1 = b0; sm.above1 = ab0; }
      if (ab1 < K1 && ab1 + h1 >= K1) { sm.b1 = b0 - 1; sm.above1 = ab1; }
      if (K2 > 0) {
        if (ab0 < K2 && ab0 + h0 >= K2) { sm.b2 = b0; sm.above2 = ab0; }
        if (ab1 < K2 && ab1 + h1 >= K2) { sm.b2 = b0 - 1; sm.above2 = ab1; }
      }
    }
    __syncthreads();
    S5_MARK(2);
    // ---- pass C: collect the two boundary buckets ----
    {
      const int b1 = sm.b1, b2 = e > 0 ? sm.b2 : -1;
      for (int base = 0; base < m; base += T) {
        const int c = base + t;
        const int bk = c < m ? (int)bid16[c] : -1;
        const bool f1 = bk == b1, f2 = bk == b2;
        const float v = (f1 || f2) ? __ldcg(s + c) : 0.f;
        s5_append(f1, s5_key(v, c), sm.l1, &sm.n1, S5_LIST, &sm.ovf);
        s5_append(f2, s5_key(v, c), sm.l2, &sm.n2, S5_LIST, &sm.ovf);
      }
    }
    __syncthreads();
    if (sm.ovf) { set_status(sv.status, kErrBandOverflow); ok = false; }
  }
  if (ok) {
    // ---- exact k-th largest approximate values (rank by counting) ----
    float tau_r, tau_e = 0.f;
    {
      const int k1 = r - sm.above1 - 1, k2 = e > 0 ? r + e - sm.above2 - 1 : -1;
      const int n1 = sm.n1, n2 = sm.n2;
      __shared__ float s_tau[2];
      for (int i = t; i < n1; i += T) {
        int rk = 0;
        for (int j = 0; j < n1; j++) rk += sm.l1[j] < sm.l1[i] ? 1 : 0;
        if (rk == k1) s_tau[0] = s5_score(sm.l1[i]);
      }
      for (int i = t; i < n2; i += T) {
        int rk = 0;
        for (int j = 0; j < n2; j++) rk += sm.l2[j] < sm.l2[i] ? 1 : 0;
        if (rk == k2) s_tau[1] = s5_score(sm.l2[i]);
      }
      __syncthreads();
      tau_r = s_tau[0];
      if (e > 0) tau_e = s_tau[1];
    }
    float qq = 0.f;
    for (int i = t; i < d; i += T) qq = fmaf(q[i], q[i], qq);
    // (recompute the bound: identical inputs -> identical value)
    float cm = 0.f;
    for (int i = t; i < m; i += T) cm = fmaxf(cm, cn[i]);
    const float qn2 = s5_reduce(qq, false, sm);
    const float cmax = s5_reduce(cm, true, sm);
    const double uu = 5.9604644775390625e-08;
    const double gam = (double)d * uu / (1.0 - (double)d * uu);
    const double B = score_error_bound((double)qn2, (double)cmax, d, p.score_fp64 != 0);
    const double B2 = 2.0 * B;
    const double hr = (double)tau_r + B2, lr = (double)tau_r - B2, he = (double)tau_e + B2, le = (double)tau_e - B2;
    S5_MARK(3);
    // ---- pass D: candidates (certain-in + band around tau_r), band around
    //      tau_e.  bucket() is monotone, so bucket(s) > bucket(hi) => s > hi and
    //      bucket(s) < bucket(lo) => s < lo; only ids in [bucket(lo),
    //      bucket(hi)] need their score.
    const int khr = bucket(__double2float_ru(hr)), klr = bucket(__double2float_rd(lr));
    const int khe = bucket(__double2float_ru(he)), kle = bucket(__double2float_rd(le));
    int my_in_e = 0;
    for (int base = 0; base < m; base += T) {
      const int c = base + t;
      const bool act = c < m;
      const int k = act ? (int)bid16[c] : -1;
      const bool need_v = act && ((k >= klr && k <= khr) || (e > 0 && k >= kle && k <= khe));
      const bool cand_r = act && k >= klr;  // certain-in or band (subject to exact compare)
      float v = 0.f;
      if (need_v || cand_r) v = __ldcg(s + c);
      const double dv = (double)v;
      const bool in_r = act && (k > khr || (k >= klr && dv > hr));
      const bool bd_r = act && !in_r && k >= klr && dv >= lr;
      s5_append(in_r || bd_r, s5_key(v, c), sm.cand, &sm.ncand, S5_CAND, &sm.ovf);
      if (bd_r) atomicAdd(&sm.nband_r, 1);
      if (e > 0) {
        const bool in_e = act && (k > khe || (k >= kle && dv > he));
        const bool bd_e = act && !in_e && k >= kle && k <= khe && dv >= le;
        my_in_e += in_e ? 1 : 0;
        const unsigned mk = __ballot_sync(0xffffffffu, bd_e);
        if (mk) {
          int b = 0;
          if (lane == __ffs(mk) - 1) b = atomicAdd(&sm.nband_e, __popc(mk));
          b = __shfl_sync(0xffffffffu, b, __ffs(mk) - 1);
          const int pos = b + __popc(mk & ((1u << lane) - 1u));
          if (bd_e) { if (pos < S5_BAND) sm.be_id[pos] = c; else sm.ovf = 1; }
        }
      }
    }
    my_in_e = __reduce_add_sync(0xffffffffu, my_in_e);
    if (lane == 0 && my_in_e) atomicAdd(&sm.n_in_e, my_in_e);
    __syncthreads();
    const int nc = sm.ncand, nbr = sm.nband_r, nin_r = nc - nbr, nbe = sm.nband_e, nin_e = sm.n_in_e;
    if (sm.ovf || nin_r > r || nc < r || (e > 0 && (nin_e > r + e || nin_e + nbe < r + e))) {
      set_status(sv.status, kErrBandOverflow);
    } else {
      S5_MARK(4);
      if (t == 0) { g_sel_dbg[blockIdx.x][12] = nbr; g_sel_dbg[blockIdx.x][13] = nbe; g_sel_dbg[blockIdx.x][14] = sm.n1; g_sel_dbg[blockIdx.x][15] = sm.n2; }
      // ---- order candidates by (approx desc, id asc) ----
      s5_rank_sort(sm.cand, nc, sm.cs);
      for (int i = t; i < nc; i += T) sm.cex[i] = 0.0;
      __syncthreads();
      // ---- one exact round: band rows (positions >= nin_r), clump members,
      //      and the band around tau_e ----
      auto needs_exact = [&](int i) {
        if (i >= nin_r) return true;
        const double si = (double)s5_score(sm.cs[i]);
        return (i > 0 && (double)s5_score(sm.cs[i - 1]) - si <= B2) ||
               (i + 1 < nc && si - (double)s5_score(sm.cs[i + 1]) <= B2);
      };
      for (int i = warp; i < nc + nbe; i += nwarps) {
        if (i < nc) {
          if (!needs_exact(i)) continue;
          const int c = s5_id(sm.cs[i]);
          const double ex = s5_exact_warp(C64 + (size_t)c * d, sm.q64, d, gemv_row_class(c, m, d, p.blas_threads));
          if (lane == 0) sm.cex[i] = ex;
        } else {
          const int c = sm.be_id[i - nc];
          const double ex = s5_exact_warp(C64 + (size_t)c * d, sm.q64, d, gemv_row_class(c, m, d, p.blas_threads));
          if (lane == 0) sm.be_ex[i - nc] = ex;
        }
      }
      __syncthreads();
      S5_MARK(5);
      // ---- band winners: best (r - nin_r) band rows by exact score ----
      const int need_r = r - nin_r;
      for (int i = nin_r + t; i < nc; i += T) {
        int rank = 0;
        for (int j = nin_r; j < nc; j++)
          rank += s5_better(sm.cex[j], s5_id(sm.cs[j]), sm.cex[i], s5_id(sm.cs[i])) ? 1 : 0;
        if (rank >= need_r) sm.cs[i] = ~0ull;  // dropped
      }
      const int need_e = r + e - nin_e;
      for (int i = t; i < nbe; i += T) {
        int rank = 0;
        for (int j = 0; j < nbe; j++) rank += s5_better(sm.be_ex[j], sm.be_id[j], sm.be_ex[i], sm.be_id[i]) ? 1 : 0;
        sm.be_sel[i] = rank < need_e ? 1 : 0;
      }
      __syncthreads();
      // ---- final order: clumps (runs of exact-scored neighbours in the
      //      approximate order, minus dropped band rows) sorted exactly ----
      // compact: certain-in keep their positions, band winners follow in
      // approximate order (positions from counting kept band rows before them)
      for (int i = t; i < nc; i += T) {
        if (i < nin_r) { sm.fin[i] = sm.cs[i]; sm.fex[i] = sm.cex[i]; continue; }
        if (sm.cs[i] == ~0ull) continue;
        int before = 0;
        for (int j = nin_r; j < i; j++) before += sm.cs[j] != ~0ull ? 1 : 0;
        sm.fin[nin_r + before] = sm.cs[i];
        sm.fex[nin_r + before] = sm.cex[i];
      }
      __syncthreads();
      for (int i = t; i < r; i += T) { sm.cs[i] = sm.fin[i]; sm.cex[i] = sm.fex[i]; }
      __syncthreads();
      // within the surviving r entries, every maximal run of positions whose
      // neighbours are closer than 2B was exact-scored; sort each run
      for (int i = t; i < r; i += T) {
        const double si = (double)s5_score(sm.cs[i]);
        const bool lp = i > 0 && (double)s5_score(sm.cs[i - 1]) - si <= B2;
        const bool ln = i + 1 < r && si - (double)s5_score(sm.cs[i + 1]) <= B2;
        if (!lp && ln) {
          int end = i + 1;
          while (end + 1 < r && (double)s5_score(sm.cs[end]) - (double)s5_score(sm.cs[end + 1]) <= B2) end++;
          for (int a = i + 1; a <= end; a++) {
            const unsigned long long kk = sm.cs[a];
            const double ev = sm.cex[a];
            int b = a - 1;
            while (b >= i && s5_better(ev, s5_id(kk), sm.cex[b], s5_id(sm.cs[b]))) {
              sm.cs[b + 1] = sm.cs[b];
              sm.cex[b + 1] = sm.cex[b];
              b--;
            }
            sm.cs[b + 1] = kk;
            sm.cex[b + 1] = ev;
          }
        }
      }
      __syncthreads();
      S5_MARK(6);
      // ---- outputs ----
      int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
      for (int i = t; i < r; i += T) {
        const int c = s5_id(sm.cs[i]);
        rl_out[i] = c;
        atomicOr(zm + c, 1u << g);
        atomicOr(rbits + (c >> 5), 1u << (c & 31));
      }
      __syncthreads();
      int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
      if (e > 0) {
        // E = top(r+e) minus R (certain part from bucket ids; the band part below)
        for (int base = 0; base < m; base += T) {
          const int c = base + t;
          const int k = c < m ? (int)bid16[c] : -1;
          bool in_e = c < m && k > khe;
          if (c < m && !in_e && k >= kle && k <= khe) in_e = (double)__ldcg(s + c) > he;
          const bool f = in_e && !((rbits[c >> 5] >> (c & 31)) & 1u);
          if (f) atomicOr(zm + c, 1u << (8 + g));
          if (el_out) {
            const unsigned mk = __ballot_sync(0xffffffffu, f);
            if (mk) {
              int b = 0;
              if (lane == __ffs(mk) - 1) b = atomicAdd(&sm.n_el, __popc(mk));
              b = __shfl_sync(0xffffffffu, b, __ffs(mk) - 1);
              if (f) el_out[b + __popc(mk & ((1u << lane) - 1u))] = c;
            }
          }
        }
        for (int i = t; i < nbe; i += T) {
          const int c = sm.be_id[i];
          if (sm.be_sel[i] && !((rbits[c >> 5] >> (c & 31)) & 1u)) {
            atomicOr(zm + c, 1u << (8 + g));
            if (el_out) el_out[atomicAdd(&sm.n_el, 1)] = c;
          }
        }
      }
      if (p.need_tail || p.need_allc) {
        __threadfence_block();
        __syncthreads();
        const float isd = p.inv_sqrt_d;
        const uint32_t both = (1u << g) | (1u << (8 + g));
        float mx_t = -INFINITY, mx_a = -INFINITY;
        for (int c = t; c < m; c += T) {
          const float x = __ldcg(s + c) * isd;
          mx_a = fmaxf(mx_a, x);
          if (!(__ldcg(zm + c) & both)) mx_t = fmaxf(mx_t, x);
        }
        mx_t = s5_reduce(mx_t, true, sm);
        mx_a = s5_reduce(mx_a, true, sm);
        float dt = 0.f, da = 0.f;
        for (int c = t; c < m; c += T) {
          const float x = __ldcg(s + c) * isd;
          const float sz = (float)csize[c];
          da += sz * expf(x - mx_a);
          if (!(__ldcg(zm + c) & both)) dt += sz * expf(x - mx_t);
        }
        dt = s5_reduce(dt, false, sm);
        da = s5_reduce(da, false, sm);
        if (t == 0) { tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da; }
      }
    }
  }
  S5_MARK(7);
  if (!ok && t == 0) { tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f; }
  // ---- the last CTA of the unit builds the unions ----
  __threadfence();
  __syncthreads();
  if (t == 0) sm.last = (atomicAdd(sv.sel_done + u, 1) == G - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  if (t == 0) sv.sel_done[u] = 0;
  S5_MARK(9);
  s5_union(ix, sv, u, m, sm);
  S5_MARK(10);
}

}  // namespace wk
