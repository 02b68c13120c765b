// select_v4.cu -- exact zone planning with the scores held in registers.
//
// Same result as select_v3 (bit-identical retrieval lists and estimation
// sets, index.py:61-93) with far fewer dependent steps:
//   * each thread keeps PT scores in registers (m <= 512*PT),
//   * the k-th largest approximate score is found with one 1024-bucket
//     histogram over [min, max] plus an exact sort of the (small) bucket that
//     holds rank k, instead of 8 radix passes,
//   * band / clump rows are re-scored exactly by a whole warp (the dgemv
//     recipe's accumulation chains are walked lane by lane with shuffles),
//   * the retrieval list (r <= 256) is sorted by one warp in registers,
//   * the last CTA of a unit builds the union lists (as v3).
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

// g_sel_dbg: defined in decode_v3.cu (same translation unit)
#define S4_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 4096) { long long _t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(_t)); g_sel_dbg[blockIdx.x][i] = _t; } } while (0)

constexpr int S4_THREADS = 512;
constexpr int S4_NB = 1024;      // histogram buckets
constexpr int S4_LIST = 1024;    // bucket-collection capacity
constexpr int S4_BAND = 512;
constexpr int S4_RL = 1024;      // retrieval-list capacity (warp sort up to 256)

struct Sel4Smem {
  int hist[S4_NB];
  int wtot[32];
  unsigned long long list1[S4_LIST];  // (~ordkey << 32 | id) of the bucket holding rank r
  unsigned long long list2[S4_LIST];  // ... rank r+e
  unsigned long long rl[S4_RL];
  double rex[S4_RL];
  int bid_r[S4_BAND];
  double bex_r[S4_BAND];
  int bid_e[S4_BAND];
  double bex_e[S4_BAND];
  unsigned char bsel_e[S4_BAND];
  unsigned int rbits[1024];          // m <= 32768: retrieval set of this head
  unsigned int ebits[1024];          // estimation set of this head
  double q64[256];
  float red[32];
  int n1, n2, above1, above2, b1, b2;
  int n_rl, n_band_r, n_band_e, n_in_e, n_el;
  int last, ovf;
  int wsum[32], wsum2[32], wsum3[32];
  int base_r, base_e, base_t;
  float fred, fmin, fmax;
};

__device__ __forceinline__ float s4_reduce(float v, bool is_max, Sel4Smem& sm) {
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
__device__ __forceinline__ float s4_min(float v, Sel4Smem& sm) { return -s4_reduce(-v, true, sm); }

// exact fp64 score of centroid row c in the reference dgemv recipe, computed
// by one warp: lane l holds t = 4l..4l+3; the chains are walked in t order.
__device__ __forceinline__ double exact_score_warp(const double* row, const double* q64, int d, int cls) {
  const int lane = threadIdx.x & 31;
  double a[8], x[8];
  const int per = d / 32;  // 4 for d = 128, 2 for d = 64 (d % 32 == 0)
#pragma unroll
  for (int i = 0; i < 8; i++) {
    a[i] = i < per ? row[lane * per + i] : 0.0;
    x[i] = i < per ? q64[lane * per + i] : 0.0;
  }
  // term t = lane*per + i.  cls 0: acc[t%4] fma chain; cls 1: acc[t%2]
  // unfused; cls 2: acc[t%4] unfused.  Walk lanes in order.
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int l = 0; l < 32; l++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (i >= per) break;
      const double av = __shfl_sync(0xffffffffu, a[i], l), xv = __shfl_sync(0xffffffffu, x[i], l);
      const int t = l * per + i;
      if (cls == 0) acc[t & 3] = __fma_rn(av, xv, acc[t & 3]);
      else if (cls == 1) acc[t & 1] = __dadd_rn(acc[t & 1], __dmul_rn(av, xv));
      else acc[t & 3] = __dadd_rn(acc[t & 3], __dmul_rn(av, xv));
    }
  }
  if (cls == 1) return __dadd_rn(0.0, __dadd_rn(acc[0], acc[1]));
  return __dadd_rn(0.0, __dadd_rn(__dadd_rn(acc[0], acc[2]), __dadd_rn(acc[1], acc[3])));
}

__device__ __forceinline__ unsigned long long s4_key(float s, int id) {
  return ((unsigned long long)(~f2u_ord(s)) << 32) | (unsigned int)id;
}
__device__ __forceinline__ float s4_score(unsigned long long k) { return u2f_ord(~(unsigned int)(k >> 32)); }
__device__ __forceinline__ int s4_id(unsigned long long k) { return (int)(k & 0xffffffffu); }
__device__ __forceinline__ bool s4_better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

// block bitonic sort (ascending) of n <= S4_LIST u64 keys in smem
__device__ void s4_block_sort(unsigned long long* a, int n) {
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = n + threadIdx.x; i < np; i += blockDim.x) a[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) { a[i] = y; a[ixj] = x; }
        }
      }
      __syncthreads();
    }
}

// one-warp bitonic sort (ascending) of n <= 256 keys in smem
__device__ void s4_warp_sort(unsigned long long* a, int n) {
  const int lane = threadIdx.x & 31;
  int np = 32;
  while (np < n) np <<= 1;
  for (int i = n + lane; i < np; i += 32) a[i] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= np; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < np; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) { a[i] = y; a[ixj] = x; }
        }
      }
      __syncwarp();
    }
}

__device__ __forceinline__ void s4_append(bool flag, int val, int* list, int* counter, int cap) {
  const unsigned mk = __ballot_sync(0xffffffffu, flag);
  if (!mk) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mk) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mk));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (flag) {
    const int pos = base + __popc(mk & ((1u << lane) - 1u));
    if (pos < cap) list[pos] = val;
  }
}

// block-wide exclusive scan of three ints
__device__ __forceinline__ void s4_scan3(int& a, int& b, int& c, int& ta, int& tb, int& tc, Sel4Smem& sm) {
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

// union of the unit's zones (last CTA of the unit); thread t owns a slice of
// cluster ids; all loads of a slice are issued before they are used.
template <int PT>
__device__ void s4_union(const IndexView& ix, const StepView& sv, int u, int m, Sel4Smem& sm) {
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const int* coff = ix.cl_off + (size_t)u * ix.m_cap;
  const int T = blockDim.x, t = threadIdx.x;
  const int lo = (int)((long long)m * t / T), hi = (int)((long long)m * (t + 1) / T);
  uint32_t z[PT];
#pragma unroll
  for (int i = 0; i < PT; i++) z[i] = (lo + i < hi) ? __ldcg(zm + lo + i) : 0u;
  int sz[PT];
#pragma unroll
  for (int i = 0; i < PT; i++) sz[i] = (z[i] & 0xffu) ? __ldcg(csize + lo + i) : 0;
  int nr = 0, ne = 0, nt = 0;
#pragma unroll
  for (int i = 0; i < PT; i++) {
    if (z[i]) zm[lo + i] = 0u;
    nr += (z[i] & 0xffu) ? 1 : 0;
    ne += (z[i] & 0xff00u) ? 1 : 0;
    nt += sz[i];
  }
  int tr, te, tt;
  s4_scan3(nr, ne, nt, tr, te, tt, sm);
  int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  int32_t* rpre = sv.ru_pre + (size_t)u * (sv.ru_cap + 1);
  int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  int32_t* trow = sv.rtok_row + (size_t)u * sv.rt_cap;
  uint8_t* tmk = sv.rtok_mask + (size_t)u * sv.rt_cap;
  int off[PT];
#pragma unroll
  for (int i = 0; i < PT; i++) off[i] = (z[i] & 0xffu) ? __ldcg(coff + lo + i) : 0;
#pragma unroll
  for (int i = 0; i < PT; i++) {
    const int c = lo + i;
    if (z[i] & 0xffu) {
      if (nr < sv.ru_cap && nt + sz[i] <= sv.rt_cap) {
        ru[nr] = c;
        rmk[nr] = (uint8_t)(z[i] & 0xffu);
        rpre[nr] = nt;
        for (int j = 0; j < sz[i]; j++) { trow[nt + j] = off[i] + j; tmk[nt + j] = (uint8_t)(z[i] & 0xffu); }
      } else {
        set_status(sv.status, kErrUnion);
      }
      nr++;
      nt += sz[i];
    }
    if (z[i] & 0xff00u) {
      if (ne < sv.eu_cap) { eu[ne] = c; emk[ne] = (uint8_t)((z[i] >> 8) & 0xffu); }
      else set_status(sv.status, kErrUnion);
      ne++;
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

// k-th largest (1-based) of the register-resident scores: bucket histogram
// over [mn, mx], then an exact sort of the bucket containing rank k.
// Returns false on bucket-list overflow (degenerate concentration).
template <int PT>
__device__ bool s4_two_thresholds(const float (&sc)[PT], int m, int K1, int K2, float mn, float mx, Sel4Smem& sm,
                                  float& tau1, float& tau2) {
  const int t = threadIdx.x, T = blockDim.x;
  for (int b = t; b < S4_NB; b += T) sm.hist[b] = 0;
  if (t == 0) { sm.n1 = 0; sm.n2 = 0; sm.ovf = 0; }
  __syncthreads();
  const float span = mx - mn;
  const float scale = span > 0.f ? (float)S4_NB / span : 0.f;
  auto bucket = [&](float v) {
    int b = (int)((v - mn) * scale);
    return b < 0 ? 0 : (b >= S4_NB ? S4_NB - 1 : b);
  };
#pragma unroll
  for (int i = 0; i < PT; i++) {
    const int c = t + i * T;
    if (c < m) atomicAdd(&sm.hist[bucket(sc[i])], 1);
  }
  __syncthreads();
  // suffix sums over buckets (descending score): thread t owns buckets 2t, 2t+1
  {
    const int lane = t & 31, w = t >> 5;
    const int b0 = S4_NB - 1 - 2 * t;  // highest bucket of this thread's pair
    const int h0 = b0 >= 0 ? sm.hist[b0] : 0, h1 = b0 - 1 >= 0 ? sm.hist[b0 - 1] : 0;
    int x = h0 + h1;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sm.wtot[w] = x;
    __syncthreads();
    if (w == 0) {
      const int nw = T >> 5;
      int v = lane < nw ? sm.wtot[lane] : 0, iv = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= o) iv += y;
      }
      if (lane < nw) sm.wtot[lane] = iv - v;
    }
    __syncthreads();
    const int above_pair = sm.wtot[w] + x - (h0 + h1);  // elements in buckets > b0
    // bucket b0: elements above = above_pair; bucket b0-1: above_pair + h0
    if (b0 >= 0) {
      if (above_pair < K1 && above_pair + h0 >= K1) { sm.b1 = b0; sm.above1 = above_pair; }
      if (above_pair < K2 && above_pair + h0 >= K2) { sm.b2 = b0; sm.above2 = above_pair; }
    }
    if (b0 - 1 >= 0) {
      const int ab = above_pair + h0;
      if (ab < K1 && ab + h1 >= K1) { sm.b1 = b0 - 1; sm.above1 = ab; }
      if (ab < K2 && ab + h1 >= K2) { sm.b2 = b0 - 1; sm.above2 = ab; }
    }
  }
  __syncthreads();
  const int b1 = sm.b1, b2 = sm.b2;
#pragma unroll
  for (int i = 0; i < PT; i++) {
    const int c = t + i * T;
    const int bki = c < m ? bucket(sc[i]) : -1;
    if (bki == b1) {
      const int p = atomicAdd(&sm.n1, 1);
      if (p < S4_LIST) sm.list1[p] = s4_key(sc[i], c); else sm.ovf = 1;
    }
    if (K2 > 0 && bki == b2) {
      const int p = atomicAdd(&sm.n2, 1);
      if (p < S4_LIST) sm.list2[p] = s4_key(sc[i], c); else sm.ovf = 1;
    }
  }
  __syncthreads();
  if (sm.ovf) return false;
  const int n1 = sm.n1, n2 = sm.n2;
  if (n1 <= 256) { if (t < 32) s4_warp_sort(sm.list1, n1); }
  else s4_block_sort(sm.list1, n1);
  if (K2 > 0) {
    if (n2 <= 256) { if (t >= 32 && t < 64) s4_warp_sort(sm.list2, n2); }
    else s4_block_sort(sm.list2, n2);
  }
  __syncthreads();
  tau1 = s4_score(sm.list1[K1 - sm.above1 - 1]);
  tau2 = K2 > 0 ? s4_score(sm.list2[K2 - sm.above2 - 1]) : 0.f;
  return true;
}

template <int PT>
__global__ void __launch_bounds__(S4_THREADS) select_v4_kernel(IndexView ix, StepView sv, SelParams p) {
  extern __shared__ __align__(128) unsigned char s4_raw[];
  Sel4Smem& sm = *reinterpret_cast<Sel4Smem*>(s4_raw);
  S4_MARK(0);
  const int G = p.G, d = p.d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int m = sv.m[u];
  const int t = threadIdx.x, T = blockDim.x, lane = t & 31, warp = t >> 5;
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
  uint32_t* zm = sv.zmask + (size_t)u * ix.m_cap;
  const double* C64 = ix.C64 + (size_t)u * ix.m_cap * d;
  const bool ok = m > 0 && r <= sv.r_cap && m <= PT * T;
  if (m > 0 && !ok) set_status(sv.status, kErrBandOverflow);
  if (ok) {
    // ---- scores and norms into registers (independent coalesced loads) ----
    float sc[PT];
    float cm = 0.f, mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < PT; i++) {
      const int c = t + i * T;
      sc[i] = c < m ? __ldcg(s + c) : -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < PT; i++) {
      const int c = t + i * T;
      if (c < m) {
        cm = fmaxf(cm, __ldcg(cn + c));
        mn = fminf(mn, sc[i]);
        mx = fmaxf(mx, sc[i]);
      }
    }
    for (int i = t; i < d; i += T) sm.q64[i] = (double)q[i];
    for (int w = t; w < (m + 31) / 32; w += T) { sm.rbits[w] = 0u; sm.ebits[w] = 0u; }
    float qq = 0.f;
    for (int i = t; i < d; i += T) qq = fmaf(q[i], q[i], qq);
    const float qn2 = s4_reduce(qq, false, sm);
    const float cmax = s4_reduce(cm, true, sm);
    const float smin = s4_min(mn, sm);
    const float smax = s4_reduce(mx, true, sm);
    const double uu = 5.9604644775390625e-08;
    const double gam = (double)d * uu / (1.0 - (double)d * uu);
    const double B = score_error_bound((double)qn2, (double)cmax, d, p.score_fp64 != 0);
    const double B2 = 2.0 * B;
    S4_MARK(1);
    float tau_r = 0.f, tau_e = 0.f;
    if (!s4_two_thresholds<PT>(sc, m, r, e > 0 ? r + e : 0, smin, smax, sm, tau_r, tau_e)) {
      set_status(sv.status, kErrBandOverflow);
    } else {
      S4_MARK(2);
      // ---- classification (registers) ----
      if (t == 0) { sm.n_rl = 0; sm.n_band_r = 0; sm.n_band_e = 0; sm.n_in_e = 0; sm.n_el = 0; }
      __syncthreads();
      int my_in_e = 0;
      const double hr = (double)tau_r + B2, lr = (double)tau_r - B2;
      const double he = (double)tau_e + B2, le = (double)tau_e - B2;
#pragma unroll
      for (int i = 0; i < PT; i++) {
        const int c = t + i * T;
        const bool act = c < m;
        const double v = (double)sc[i];
        const bool in_r = act && v > hr;
        const bool bd_r = act && !in_r && v >= lr;
        s4_append(in_r, c, reinterpret_cast<int*>(sm.rex), &sm.n_rl, S4_RL);
        s4_append(bd_r, c, sm.bid_r, &sm.n_band_r, S4_BAND);
        if (e > 0) {
          const bool in_e = act && v > he;
          const bool bd_e = act && !in_e && v >= le;
          my_in_e += in_e ? 1 : 0;
          s4_append(bd_e, c, sm.bid_e, &sm.n_band_e, S4_BAND);
        }
      }
      my_in_e = __reduce_add_sync(0xffffffffu, my_in_e);
      if (lane == 0 && my_in_e) atomicAdd(&sm.n_in_e, my_in_e);
      __syncthreads();
      S4_MARK(3);
      const int nin_r = sm.n_rl, nbr = sm.n_band_r, nbe = sm.n_band_e, nin_e = sm.n_in_e;
      if (t == 0) { g_sel_dbg[blockIdx.x][12] = nbr; g_sel_dbg[blockIdx.x][13] = nbe; g_sel_dbg[blockIdx.x][14] = sm.n1; g_sel_dbg[blockIdx.x][15] = sm.n2; }
      const bool bad = r > S4_RL || nbr > S4_BAND || nbe > S4_BAND || nin_r > r || nin_r + nbr < r ||
                       (e > 0 && (nin_e > r + e || nin_e + nbe < r + e));
      if (bad) {
        set_status(sv.status, kErrBandOverflow);
      } else {
        const int* staged = reinterpret_cast<const int*>(sm.rex);
        for (int i = t; i < nin_r; i += T) { const int c = staged[i]; sm.rl[i] = s4_key(__ldcg(s + c), c); }
        // exact scores of the band rows: one warp per row
        const int nwarps = T >> 5;
        for (int i = warp; i < nbr + nbe; i += nwarps) {
          const int c = i < nbr ? sm.bid_r[i] : sm.bid_e[i - nbr];
          const double ex = exact_score_warp(C64 + (size_t)c * d, sm.q64, d, gemv_row_class(c, m, d, p.blas_threads));
          if (lane == 0) { if (i < nbr) sm.bex_r[i] = ex; else sm.bex_e[i - nbr] = ex; }
        }
        __syncthreads();
        const int need_r = r - nin_r, need_e = r + e - nin_e;
        for (int i = t; i < nbr; i += T) {
          int rank = 0;
          for (int j = 0; j < nbr; j++) rank += s4_better(sm.bex_r[j], sm.bid_r[j], sm.bex_r[i], sm.bid_r[i]) ? 1 : 0;
          if (rank < need_r) sm.rl[nin_r + rank] = s4_key(__ldcg(s + sm.bid_r[i]), sm.bid_r[i]);
        }
        for (int i = t; i < nbe; i += T) {
          int rank = 0;
          for (int j = 0; j < nbe; j++) rank += s4_better(sm.bex_e[j], sm.bid_e[j], sm.bex_e[i], sm.bid_e[i]) ? 1 : 0;
          sm.bsel_e[i] = rank < need_e ? 1 : 0;
        }
        __syncthreads();
        S4_MARK(4);
        // ---- order the retrieval list: warp 0 sorts, every warp re-scores clumps
        if (r <= 256) { if (warp == 0) s4_warp_sort(sm.rl, r); }
        else s4_block_sort(sm.rl, r);
        __syncthreads();
        for (int i = t; i < r; i += T) sm.rex[i] = 0.0;
        __syncthreads();
        S4_MARK(5);
        // clump members: exact scores (one warp per member)
        for (int i = warp; i < r; i += nwarps) {
          const double si = (double)s4_score(sm.rl[i]);
          const bool cl = (i > 0 && (double)s4_score(sm.rl[i - 1]) - si <= B2) ||
                          (i + 1 < r && si - (double)s4_score(sm.rl[i + 1]) <= B2);
          if (cl) {
            const int c = s4_id(sm.rl[i]);
            const double ex = exact_score_warp(C64 + (size_t)c * d, sm.q64, d, gemv_row_class(c, m, d, p.blas_threads));
            if (lane == 0) sm.rex[i] = ex;
          }
        }
        __syncthreads();
        for (int i = t; i < r; i += T) {
          const double si = (double)s4_score(sm.rl[i]);
          const bool lp = i > 0 && (double)s4_score(sm.rl[i - 1]) - si <= B2;
          const bool ln = i + 1 < r && si - (double)s4_score(sm.rl[i + 1]) <= B2;
          if (!lp && ln) {
            int end = i + 1;
            while (end + 1 < r && (double)s4_score(sm.rl[end]) - (double)s4_score(sm.rl[end + 1]) <= B2) end++;
            for (int a = i + 1; a <= end; a++) {
              const unsigned long long kk = sm.rl[a];
              const double ev = sm.rex[a];
              int b = a - 1;
              while (b >= i && s4_better(ev, s4_id(kk), sm.rex[b], s4_id(sm.rl[b]))) {
                sm.rl[b + 1] = sm.rl[b];
                sm.rex[b + 1] = sm.rex[b];
                b--;
              }
              sm.rl[b + 1] = kk;
              sm.rex[b + 1] = ev;
            }
          }
        }
        __syncthreads();
        S4_MARK(6);
        // ---- outputs ----
        int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
        for (int i = t; i < r; i += T) {
          const int c = s4_id(sm.rl[i]);
          rl_out[i] = c;
          atomicOr(zm + c, 1u << g);
          atomicOr(sm.rbits + (c >> 5), 1u << (c & 31));
        }
        __syncthreads();
        int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
        if (e > 0) {
#pragma unroll
          for (int i = 0; i < PT; i++) {
            const int c = t + i * T;
            const bool f = c < m && (double)sc[i] > he && !((sm.rbits[c >> 5] >> (c & 31)) & 1u);
            if (f) { atomicOr(zm + c, 1u << (8 + g)); atomicOr(sm.ebits + (c >> 5), 1u << (c & 31)); }
            if (el_out) s4_append(f, c, el_out, &sm.n_el, sv.e_cap);
          }
          for (int i = t; i < nbe; i += T) {
            const int c = sm.bid_e[i];
            if (sm.bsel_e[i] && !((sm.rbits[c >> 5] >> (c & 31)) & 1u)) {
              atomicOr(zm + c, 1u << (8 + g));
              atomicOr(sm.ebits + (c >> 5), 1u << (c & 31));
              if (el_out) el_out[atomicAdd(&sm.n_el, 1)] = c;
            }
          }
        }
        if (p.need_tail || p.need_allc) {
          // tail / all-cluster denominator terms (engine.py:153-172)
          __syncthreads();
          const float isd = p.inv_sqrt_d;
          const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
          float mx_t = -INFINITY, mx_a = -INFINITY;
          bool inz[PT];
#pragma unroll
          for (int i = 0; i < PT; i++) {
            const int c = t + i * T;
            inz[i] = c < m && (((sm.rbits[c >> 5] | sm.ebits[c >> 5]) >> (c & 31)) & 1u);
            if (c < m) {
              const float x = sc[i] * isd;
              mx_a = fmaxf(mx_a, x);
              if (!inz[i]) mx_t = fmaxf(mx_t, x);
            }
          }
          mx_t = s4_reduce(mx_t, true, sm);
          mx_a = s4_reduce(mx_a, true, sm);
          float dt = 0.f, da = 0.f;
#pragma unroll
          for (int i = 0; i < PT; i++) {
            const int c = t + i * T;
            if (c < m) {
              const float sz = (float)__ldcg(csize + c);
              const float x = sc[i] * isd;
              da += sz * expf(x - mx_a);
              if (!inz[i]) dt += sz * expf(x - mx_t);
            }
          }
          dt = s4_reduce(dt, false, sm);
          da = s4_reduce(da, false, sm);
          if (t == 0) { tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da; }
        }
      }
    }
  }
  S4_MARK(7);
  if (!ok && t == 0) { tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f; }
  // ---- the last CTA of the unit builds the unions ----
  __threadfence();
  __syncthreads();
  if (t == 0) sm.last = (atomicAdd(sv.sel_done + u, 1) == G - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  if (t == 0) sv.sel_done[u] = 0;
  S4_MARK(9);
  s4_union<PT>(ix, sv, u, m, sm);
  S4_MARK(10);
}

size_t select_v4_smem() { return sizeof(Sel4Smem); }
template __global__ void select_v4_kernel<16>(IndexView, StepView, SelParams);
template __global__ void select_v4_kernel<32>(IndexView, StepView, SelParams);

}  // namespace wk
