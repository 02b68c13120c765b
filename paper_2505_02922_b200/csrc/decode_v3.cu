// decode_v3.cu -- TMA-fed decode kernels.
//
// Every warp owns a private ring of NST shared-memory stages.  A stage is
// filled by 1-D bulk copies (cp.async.bulk, the TMA unit: one instruction per
// contiguous run) that complete on the stage's mbarrier; the warp consumes
// stage k while stages k+1.. are in flight.  No register staging of loads and
// no CTA-wide barrier inside the pipelines, so 16 warps/SM keep ~100 KB/SM of
// reads in flight.
//
//   score_v3  : centroid scan; a group = 32/HS consecutive C32 rows = ONE bulk
//               copy; 32 (row, head) dots reduced with a transposed shuffle
//               reduction (index.py:61-76 ranking scores)
//   select_v3 : exact zones (as select_v2) with a dynamically sized smem
//               layout and 8-bit radix digits (4 passes) so several CTAs
//               share an SM; the last CTA of a unit builds the unions
//   attend_v3 : fused tripartite attention (attention.py:67-148): warps are
//               split over the unit's three zones (steady tokens, retrieved
//               tokens, estimation rows) in proportion to their work; a group
//               of 32/HS rows arrives by per-row bulk copies (K and V rows of
//               256 B, or fp32 value-sum rows of 512 B)
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

// ---------------------------------------------------------------------------
// select_v3: exact zones (index.py:61-93) + unit unions
// ---------------------------------------------------------------------------
__device__ long long g_sel_dbg[4096][16];  // per-CTA phase timestamps (globaltimer, ns)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SEL_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_sel_dbg[blockIdx.x][i] = gtimer(); } while (0)

constexpr int S2_THREADS = 256;
constexpr int S2_BAND = 512;
constexpr int S2_RL = 4096;     // max r (retrieval clusters per head)
constexpr int S2_KEYS = 16384;  // scores cached in smem up to this m

// fixed header; the variable arrays follow it in dynamic smem (see sel_layout)
struct Sel2Smem {
  unsigned int* keys;          // [m] order keys (nullptr: derive from global)
  unsigned long long* rl;      // [rlcap] retrieval sort keys
  double* ex;                  // [rlcap] exact scores / staged ids
  int* bid_r;                  // [S2_BAND]
  double* bex_r;
  int* bid_e;
  double* bex_e;
  unsigned char* bsel_e;
  unsigned int* rbits;         // [ceil(m/32)] this head's retrieval set
  unsigned int* ebits;         // [ceil(m/32)] this head's estimation set
  int hist[256];
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
  // keys: smem-cached order keys, or nullptr to derive them from sg (global).
  // 4 passes of 8-bit digits; per-warp aggregated histogram increments.
  unsigned int prefix = 0, pmask = 0;
  if (threadIdx.x == 0) sm.krem = K;
  for (int pass = 0; pass < 4; pass++) {
    const int sh = 24 - 8 * pass;
    const unsigned dm = 255u;
    const int nb = 256;
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

// block-wide exclusive scan of three ints (blockDim.x <= 1024)
__device__ __forceinline__ void scan3(int& a, int& b, int& c, int& ta, int& tb, int& tc, Sel2Smem& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int xa = a, xb = b, xc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int pa = __shfl_up_sync(FULLMASK, xa, o), pb = __shfl_up_sync(FULLMASK, xb, o),
              pc = __shfl_up_sync(FULLMASK, xc, o);
    if (lane >= o) { xa += pa; xb += pb; xc += pc; }
  }
  if (lane == 31) { sm.wsum[w] = xa; sm.wsum2[w] = xb; sm.wsum3[w] = xc; }
  __syncthreads();
  if (w == 0) {
    int va = lane < nw ? sm.wsum[lane] : 0, vb = lane < nw ? sm.wsum2[lane] : 0, vc = lane < nw ? sm.wsum3[lane] : 0;
    int ia = va, ib = vb, ic = vc;
    for (int o = 1; o < 32; o <<= 1) {
      const int pa = __shfl_up_sync(FULLMASK, ia, o), pb = __shfl_up_sync(FULLMASK, ib, o),
                pc = __shfl_up_sync(FULLMASK, ic, o);
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

// union of the unit's G zones (runs in the last CTA of the unit): each thread
// owns a contiguous slice of cluster ids, so one block scan orders everything.
__device__ void s2_union(const IndexView& ix, const StepView& sv, int u, int m, int sv_G, Sel2Smem& sm) {
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
  const int T = blockDim.x, t = threadIdx.x;
  const int lo = (int)((long long)m * t / T), hi = (int)((long long)m * (t + 1) / T);
  // stage the zone bits in smem (coalesced batch of independent loads), then
  // clear them for the next step
  unsigned int* zb = sm.keys;
  const bool staged = zb != nullptr;
  if (staged) {
    for (int c = t; c < m; c += T) zb[c] = __ldcg(zm + c);
    __syncthreads();
    for (int c = t; c < m; c += T)
      if (zb[c]) zm[c] = 0u;
  }
  int nr = 0, ne = 0, nt = 0;
  for (int c = lo; c < hi; c++) {
    const uint32_t z = staged ? zb[c] : __ldcg(zm + c);
    if (z & 0xffu) { nr++; nt += csize[c]; }
    if (z & 0xff00u) ne++;
  }
  int tr, te, tt;
  scan3(nr, ne, nt, tr, te, tt, sm);
  for (int c = lo; c < hi; c++) {
    const uint32_t z = staged ? zb[c] : __ldcg(zm + c);
    if (!z) continue;
    if (!staged) zm[c] = 0u;
    if (z & 0xffu) {
      const int sz = csize[c];
      if (nr < sv.ru_cap && nt + sz <= sv.rt_cap) {
        ru[nr] = c;
        rmk[nr] = (uint8_t)(z & 0xffu);
        rpre[nr] = nt;
        const int o = coff[c];
        for (int j = 0; j < sz; j++) { trow[nt + j] = o + j; tmk[nt + j] = (uint8_t)(z & 0xffu); }
      } else {
        set_status(sv.status, kErrUnion);
      }
      nr++;
      nt += sz;
    }
    if (z & 0xff00u) {
      if (ne < sv.eu_cap) {
        eu[ne] = c;
        emk[ne] = (uint8_t)((z >> 8) & 0xffu);
      } else {
        set_status(sv.status, kErrUnion);
      }
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

__host__ __device__ inline size_t sel_rlcap(int r_max) {
  size_t c = 1;
  while ((int)c < r_max) c <<= 1;
  return c < 32 ? 32 : c;
}
__host__ __device__ inline size_t sel_smem_bytes(int m_max, int r_max) {
  const size_t hdr = (sizeof(Sel2Smem) + 127) & ~(size_t)127;
  const size_t keys = m_max <= S2_KEYS ? (size_t)m_max * 4 : 0;
  const size_t rl = sel_rlcap(r_max);
  const size_t bits = ((size_t)(m_max + 31) / 32) * 4 * 2;
  return hdr + ((keys + 15) & ~(size_t)15) + rl * 16 + (size_t)S2_BAND * (4 + 8 + 4 + 8 + 1) + 64 + bits + 32;
}

__global__ void __launch_bounds__(S2_THREADS) select_v3_kernel(IndexView ix, StepView sv, SelParams p, int m_max,
                                                               int r_max) {
  extern __shared__ __align__(128) unsigned char s2_raw[];
  Sel2Smem& sm = *reinterpret_cast<Sel2Smem*>(s2_raw);
  if (threadIdx.x == 0) {
    unsigned char* q = s2_raw + ((sizeof(Sel2Smem) + 127) & ~(size_t)127);
    const size_t keys = m_max <= S2_KEYS ? (size_t)m_max * 4 : 0;
    sm.keys = keys ? reinterpret_cast<unsigned int*>(q) : nullptr;
    q += (keys + 15) & ~(size_t)15;
    const size_t rlc = sel_rlcap(r_max);
    sm.rl = reinterpret_cast<unsigned long long*>(q); q += rlc * 8;
    sm.ex = reinterpret_cast<double*>(q); q += rlc * 8;
    sm.bex_r = reinterpret_cast<double*>(q); q += S2_BAND * 8;
    sm.bex_e = reinterpret_cast<double*>(q); q += S2_BAND * 8;
    sm.bid_r = reinterpret_cast<int*>(q); q += S2_BAND * 4;
    sm.bid_e = reinterpret_cast<int*>(q); q += S2_BAND * 4;
    sm.bsel_e = q; q += S2_BAND;
    q = reinterpret_cast<unsigned char*>(((size_t)q + 15) & ~(size_t)15);
    sm.rbits = reinterpret_cast<unsigned int*>(q); q += ((size_t)(m_max + 31) / 32) * 4;
    sm.ebits = reinterpret_cast<unsigned int*>(q);
  }
  __syncthreads();
  SEL_MARK(0);
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
  const bool ok = m > 0 && r <= r_max && r <= S2_RL;
  const bool cached = sm.keys != nullptr && m <= m_max;
  if (m > 0 && !ok) set_status(sv.status, kErrBandOverflow);
  if (ok) {
    for (int t = threadIdx.x; t < d; t += blockDim.x) sm.q64[t] = (double)q[t];
    float cm = 0.f;
#pragma unroll 4
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      if (cached) sm.keys[c] = f2u_ord(s[c]);
      cm = fmaxf(cm, ix.Cnorm[(size_t)u * ix.m_cap + c]);
    }
    for (int w = threadIdx.x; w < (m + 31) / 32; w += blockDim.x) { sm.rbits[w] = 0u; sm.ebits[w] = 0u; }
    float qq = 0.f;
    for (int t = threadIdx.x; t < d; t += blockDim.x) qq = fmaf(q[t], q[t], qq);
    const float qn2 = s2_block_reduce(qq, false, sm);
    const float cmax = s2_block_reduce(cm, true, sm);
    const double uu = 5.9604644775390625e-08;
    const double gam = (double)d * uu / (1.0 - (double)d * uu);
    const double B = score_error_bound((double)qn2, (double)cmax, d, p.score_fp64 != 0);
    const double B2 = 2.0 * B;
    SEL_MARK(1);
    const unsigned* kp = cached ? sm.keys : nullptr;
    const float tau_r = u2f_ord(s2_kth_largest(kp, s, m, r, sm));
    const float tau_e = e > 0 ? u2f_ord(s2_kth_largest(kp, s, m, r + e, sm)) : 0.f;
    SEL_MARK(2);
    if (threadIdx.x == 0) { sm.n_in_r = 0; sm.n_band_r = 0; sm.n_band_e = 0; sm.n_in_e = 0; sm.n_rl = 0; }
    __syncthreads();
    int my_in_e = 0;
    const int rl_cap = (int)sel_rlcap(r_max);
    for (int base = 0; base < m; base += blockDim.x) {
      const int c = base + threadIdx.x;
      const bool act = c < m;
      const double sc = act ? (double)(cached ? u2f_ord(sm.keys[c]) : s[c]) : -INFINITY;
      const bool in_r = act && sc > (double)tau_r + B2;
      const bool bd_r = act && !in_r && sc >= (double)tau_r - B2;
      warp_append(in_r, c, reinterpret_cast<int*>(sm.ex), &sm.n_rl, rl_cap);  // ids staged in ex[]
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
    SEL_MARK(3);
    const int nin_r = sm.n_rl, nbr = sm.n_band_r, nbe = sm.n_band_e, nin_e = sm.n_in_e;
    if (threadIdx.x == 0 && blockIdx.x < 4096) { g_sel_dbg[blockIdx.x][12] = nbr; g_sel_dbg[blockIdx.x][13] = nbe; }
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
      SEL_MARK(4);
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
      SEL_MARK(5);
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
      SEL_MARK(6);
      int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const int c = s2_id(sm.rl[i]);
        rl_out[i] = c;
        atomicOr(zm + c, 1u << g);
        atomicOr(sm.rbits + (c >> 5), 1u << (c & 31));
      }
      __threadfence_block();
      __syncthreads();
      int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
      if (threadIdx.x == 0) sm.n_el = 0;
      __syncthreads();
      if (e > 0) {
        for (int base = 0; base < m; base += blockDim.x) {
          const int c = base + threadIdx.x;
          const bool f = c < m && (double)(cached ? u2f_ord(sm.keys[c]) : s[c]) > (double)tau_e + B2 &&
                         !((sm.rbits[c >> 5] >> (c & 31)) & 1u);
          if (f) { atomicOr(zm + c, 1u << (8 + g)); atomicOr(sm.ebits + (c >> 5), 1u << (c & 31)); }
          if (el_out) warp_append(f, c, el_out, &sm.n_el, sv.e_cap);
        }
        for (int i = threadIdx.x; i < nbe; i += blockDim.x) {
          const int c = sm.bid_e[i];
          if (sm.bsel_e[i] && !((sm.rbits[c >> 5] >> (c & 31)) & 1u)) {
            atomicOr(zm + c, 1u << (8 + g));
            atomicOr(sm.ebits + (c >> 5), 1u << (c & 31));
            if (el_out) el_out[atomicAdd(&sm.n_el, 1)] = c;
          }
        }
      }
      __syncthreads();
      SEL_MARK(7);
      if (p.need_tail || p.need_allc) {
        const float isd = p.inv_sqrt_d;
        float mx_t = -INFINITY, mx_a = -INFINITY;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          const float v = s[c] * isd;
          mx_a = fmaxf(mx_a, v);
          if (!(((sm.rbits[c >> 5] | sm.ebits[c >> 5]) >> (c & 31)) & 1u)) mx_t = fmaxf(mx_t, v);
        }
        mx_t = s2_block_reduce(mx_t, true, sm);
        mx_a = s2_block_reduce(mx_a, true, sm);
        float dt = 0.f, da = 0.f;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          const float v = s[c] * isd;
          const float sz = (float)csize[c];
          da += sz * expf(v - mx_a);
          if (!(((sm.rbits[c >> 5] | sm.ebits[c >> 5]) >> (c & 31)) & 1u)) dt += sz * expf(v - mx_t);
        }
        dt = s2_block_reduce(dt, false, sm);
        da = s2_block_reduce(da, false, sm);
        if (threadIdx.x == 0) { tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da; }
      }
    }
  }
  if (!ok && threadIdx.x == 0) { tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f; }
  SEL_MARK(8);
  // ---- the last CTA of the unit builds the unions ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm.last = (atomicAdd(sv.sel_done + u, 1) == G - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  if (threadIdx.x == 0) sv.sel_done[u] = 0;
  SEL_MARK(9);
  s2_union(ix, sv, u, m, G, sm);
  SEL_MARK(10);
}




// ===========================================================================
// attend_v3 (v5 inner loop): half-warp rows.
//   A group is RG rows; lanes 0-15 take the even rows, lanes 16-31 the odd
//   rows, each lane owning DPL = d/16 contiguous dims of its rows (one 16-byte
//   smem read per row for bf16 d=128).  QK partials (RG/2 rows x HS heads = 16
//   per lane) are reduced over the 16 lanes of the half with a 15-shuffle
//   transposed reduction; lane (half, sub) ends with the logit of token
//   j = half + 2*(sub / HS), head sub % HS.  P.V accumulates per half and the
//   halves are folded once per warp.  Packed FFMA2 throughout.  Rows past the
//   end of a zone are bulk-copied from a zero row: no per-row predicates.
// ===========================================================================
__device__ __align__(16) unsigned char g_zero_row[1024];

template <typename T, int DPL, int HS, bool FULL>
struct AttV3Cfg {
  static constexpr int RG = 32 / HS;                        // rows per group (8 or 4)
  static constexpr int NST = 3;                             // stages per warp
  static constexpr int D = 16 * DPL;
  static constexpr int ROWT = D * (int)sizeof(T);           // K or V row bytes
  static constexpr int ROWV = D * 4;                        // value-sum row bytes
  static constexpr int SBT = 2 * RG * ROWT;
  static constexpr int SB = ((SBT > RG * ROWV ? SBT : RG * ROWV) + 127) / 128 * 128;
  static constexpr int WARPS = 8;
  static constexpr size_t SMEM = (size_t)WARPS * NST * SB + (size_t)WARPS * NST * 8 + 64 +
                                 (size_t)WARPS * NST * 32 * 12 + (size_t)WARPS * 32 * 4;
};

// DPL elements of a row at `p` -> DPL/2 float2
template <typename T, int DPL> struct RowF2;
template <> struct RowF2<__nv_bfloat16, 8> {
  static __device__ __forceinline__ void ld(const void* p, float2 (&o)[4]) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; i++) o[i] = __bfloat1622float2(h[i]);
  }
};
template <> struct RowF2<__nv_bfloat16, 4> {
  static __device__ __forceinline__ void ld(const void* p, float2 (&o)[2]) {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
    o[0] = __bfloat1622float2(h[0]);
    o[1] = __bfloat1622float2(h[1]);
  }
};
template <> struct RowF2<float, 8> {
  static __device__ __forceinline__ void ld(const void* p, float2 (&o)[4]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    o[0] = make_float2(a.x, a.y); o[1] = make_float2(a.z, a.w); o[2] = make_float2(b.x, b.y); o[3] = make_float2(b.z, b.w);
  }
};
template <> struct RowF2<float, 4> {
  static __device__ __forceinline__ void ld(const void* p, float2 (&o)[2]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    o[0] = make_float2(a.x, a.y); o[1] = make_float2(a.z, a.w);
  }
};

// 16 values summed over the 16 lanes of each half-warp; returns the total of
// index (lane & 15)
__device__ __forceinline__ float transpose_reduce16(float (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; i++) {
      const float send = up ? v[i] : v[i + off];
      const float keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

template <typename T, int DPL, int HS, bool FULL>
__global__ void __launch_bounds__(256, 2) attend_v3_kernel(IndexView ix, SteadyView st, StepView sv, AttnParams p,
                                                            const int32_t* __restrict__ n_store) {
  using CF = AttV3Cfg<T, DPL, HS, FULL>;
  constexpr int RG = CF::RG, NST = CF::NST, ROWT = CF::ROWT, ROWV = CF::ROWV, SB = CF::SB;
  constexpr int D = CF::D, RH = RG / 2, DP2 = DPL / 2;
  const int s_idx = blockIdx.x, u = blockIdx.y, S = gridDim.x;
  const int G = p.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, sub = lane & 15;
  extern __shared__ __align__(128) unsigned char at3[];
  unsigned char* ring = at3 + (size_t)warp * NST * SB;
  unsigned char* tb = at3 + (size_t)CF::WARPS * NST * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tb) + warp * NST;
  int* wkind = reinterpret_cast<int*>(tb + (size_t)CF::WARPS * NST * 8);
  unsigned char* meta = tb + (size_t)CF::WARPS * NST * 8 + 64 + (size_t)warp * NST * 32 * 12;
  int* smask = reinterpret_cast<int*>(meta);
  float* sx = reinterpret_cast<float*>(meta + NST * 32 * 4);
  float* sw = reinterpret_cast<float*>(meta + NST * 32 * 8);
  float* pbuf = reinterpret_cast<float*>(tb + (size_t)CF::WARPS * NST * 8 + 64 + (size_t)CF::WARPS * NST * 32 * 12) +
                warp * 32;

  const int n_st = st.n[u];
  const int n_rt = FULL ? n_store[u] : sv.cnt[u * 4 + 1];
  const int n_eu = FULL ? 0 : sv.cnt[u * 4 + 2];
  const int g_st = (n_st + RG - 1) / RG, g_rt = (n_rt + RG - 1) / RG, g_eu = (n_eu + RG - 1) / RG;
  const long long NG = (long long)g_st + g_rt + g_eu;
  const int W = S * CF::WARPS, wg = s_idx * CF::WARPS + warp;
  int W0 = g_st ? max(1, (int)((long long)W * g_st / max(NG, 1LL))) : 0;
  int W2 = g_eu ? max(1, (int)((long long)W * g_eu / max(NG, 1LL))) : 0;
  int W1 = W - W0 - W2;
  if (g_rt && W1 < 1) { if (W0 > W2) W0--; else W2--; W1 = 1; }
  if (!g_rt) { W1 = 0; if (g_eu) W2 = W - W0; else W0 = W; }
  int kind, li, nw, gk, n_kind;
  if (wg < W0) { kind = 0; li = wg; nw = W0; gk = g_st; n_kind = n_st; }
  else if (wg < W0 + W1) { kind = 1; li = wg - W0; nw = W1; gk = g_rt; n_kind = n_rt; }
  else { kind = 2; li = wg - W0 - W1; nw = W2; gk = g_eu; n_kind = n_eu; }
  const int gb = nw > 0 ? (int)((long long)li * gk / nw) : 0;
  const int ge = nw > 0 ? (int)((long long)(li + 1) * gk / nw) : 0;

  if (lane == 0) {
    for (int i = 0; i < NST; i++) mbar_init(bars + i, 1);
    fence_mbar_init();
    wkind[warp] = (ge > gb) ? kind : -1;
  }
  __syncwarp();

  const float isd = p.inv_sqrt_d;
  // q slice of this lane's dims, pre-scaled: qv[h][k] covers dims sub*DPL + 2k, +1
  float2 qv[HS][DP2];
#pragma unroll
  for (int h = 0; h < HS; h++)
#pragma unroll
    for (int k = 0; k < DP2; k++) {
      const float* qp = sv.q + ((size_t)u * G + (h < G ? h : 0)) * D + sub * DPL + 2 * k;
      qv[h][k] = h < G ? make_float2(qp[0] * isd, qp[1] * isd) : make_float2(0.f, 0.f);
    }

  const T* stk = (const T*)st.k + (size_t)u * st.t_cap * D;
  const T* stv = (const T*)st.v + (size_t)u * st.t_cap * D;
  const T* sk = (const T*)ix.store_k + (size_t)u * ix.s_cap * D;
  const T* svv = (const T*)ix.store_v + (size_t)u * ix.s_cap * D;
  const int32_t* trow = FULL ? nullptr : sv.rtok_row + (size_t)u * sv.rt_cap;
  const uint8_t* tmk = FULL ? nullptr : sv.rtok_mask + (size_t)u * sv.rt_cap;
  const int32_t* eu = FULL ? nullptr : sv.eu_ids + (size_t)u * sv.eu_cap;
  const uint8_t* emk = FULL ? nullptr : sv.eu_mask + (size_t)u * sv.eu_cap;
  const float* scr = FULL ? nullptr : sv.scores + (size_t)u * G * ix.m_cap;
  const int32_t* csz = ix.cl_size + (size_t)u * ix.m_cap;
  const float* vsb = ix.VS32 + (size_t)u * ix.m_cap * D;
  const int allmask = (1 << G) - 1;
  // (token, head) whose logit this lane holds after the reduction
  const int j_own = half + 2 * (sub / HS), h_own = sub % HS;

  SoftState<HS> ss;
#pragma unroll
  for (int h = 0; h < HS; h++) { ss.M[h] = -INFINITY; ss.D[h] = 0.f; }
  float2 acc[HS][DP2];
#pragma unroll
  for (int h = 0; h < HS; h++)
#pragma unroll
    for (int k = 0; k < DP2; k++) acc[h][k] = make_float2(0.f, 0.f);

  struct Meta { const void* k; const void* v; int mk; float x, w; };
  auto load_meta = [&](int g) {
    Meta mt{g_zero_row, g_zero_row, 0, -INFINITY, 0.f};
    if (g >= ge) return mt;
    const int item0 = g * RG;
    const int it = item0 + (lane % RG);
    if (it < n_kind) {
      if (kind == 0) { mt.k = stk + (size_t)it * D; mt.v = stv + (size_t)it * D; }
      else if (kind == 1) {
        const long long row = FULL ? (long long)it : (long long)__ldcg(trow + it);
        mt.k = sk + (size_t)row * D; mt.v = svv + (size_t)row * D;
      } else {
        mt.k = vsb + (size_t)__ldcg(eu + it) * D;
      }
    }
    const int io = item0 + j_own;
    if (io < n_kind) {
      if (kind == 0 || FULL) mt.mk = allmask;
      else if (kind == 1) mt.mk = __ldcg(tmk + io);
      else {
        const int c = __ldcg(eu + io);
        mt.mk = __ldcg(emk + io);
        mt.x = ((mt.mk >> h_own) & 1) ? __ldcg(scr + (size_t)h_own * ix.m_cap + c) * isd : -INFINITY;
        mt.w = (float)__ldcg(csz + c);
      }
    }
    return mt;
  };
  auto issue = [&](int sti, const Meta& mt) {
    unsigned char* stage = ring + sti * SB;
    if (lane == 0) mbar_arrive_expect_tx(bars + sti, kind < 2 ? (uint32_t)(RG * 2 * ROWT) : (uint32_t)(RG * ROWV));
    __syncwarp();
    if (lane < RG) {
      if (kind < 2) {
        bulk_g2s(stage + lane * ROWT, mt.k, ROWT, bars + sti);
        bulk_g2s(stage + RG * ROWT + lane * ROWT, mt.v, ROWT, bars + sti);
      } else {
        bulk_g2s(stage + lane * ROWV, mt.k, ROWV, bars + sti);
      }
    }
    smask[sti * 32 + lane] = mt.mk;
    sx[sti * 32 + lane] = mt.x;
    sw[sti * 32 + lane] = mt.w;
  };

  auto compute = [&](int sti) {
    const unsigned char* stage = ring + sti * SB;
    float alpha[HS];
    float pw;
    if (kind < 2) {
      float v[16];
#pragma unroll
      for (int jj = 0; jj < RH; jj++) {
        const int j = half + 2 * jj;
        float2 kf[DP2];
        RowF2<T, DPL>::ld(stage + j * ROWT + sub * DPL * (int)sizeof(T), kf);
#pragma unroll
        for (int h = 0; h < HS; h++) {
          float2 a2 = __fmul2_rn(kf[0], qv[h][0]);
#pragma unroll
          for (int k = 1; k < DP2; k++) a2 = __ffma2_rn(kf[k], qv[h][k], a2);
          v[jj * HS + h] = a2.x + a2.y;
        }
      }
      float x = transpose_reduce16(v);
      if (!((smask[sti * 32 + lane] >> h_own) & 1)) x = -INFINITY;
      pw = softmax_group<HS>(x, 1.f, ss, alpha);
    } else {
      pw = softmax_group<HS>(sx[sti * 32 + lane], sw[sti * 32 + lane], ss, alpha);
    }
    pbuf[j_own * HS + h_own] = pw;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < HS; h++) {
      const float2 a = make_float2(alpha[h], alpha[h]);
#pragma unroll
      for (int k = 0; k < DP2; k++) acc[h][k] = __fmul2_rn(acc[h][k], a);
    }
#pragma unroll
    for (int jj = 0; jj < RH; jj++) {
      const int j = half + 2 * jj;
      float2 vf[DP2];
      if (kind < 2) RowF2<T, DPL>::ld(stage + RG * ROWT + j * ROWT + sub * DPL * (int)sizeof(T), vf);
      else RowF2<float, DPL>::ld(stage + j * ROWV + sub * DPL * 4, vf);
#pragma unroll
      for (int h = 0; h < HS; h++) {
        const float pj = pbuf[j * HS + h];
        const float2 p2 = make_float2(pj, pj);
#pragma unroll
        for (int k = 0; k < DP2; k++) acc[h][k] = __ffma2_rn(p2, vf[k], acc[h][k]);
      }
    }
  };

  if (ge > gb) {
    Meta mnext = load_meta(gb);
#pragma unroll
    for (int i = 0; i < NST - 1; i++)
      if (gb + i < ge) {
        const Meta mcur = mnext;
        mnext = load_meta(gb + i + 1);
        issue(i, mcur);
      }
    for (int g = gb; g < ge; g++) {
      const int k = g - gb;
      const int sti = k % NST;
      const int nxt = g + NST - 1;
      if (nxt < ge) {
        const Meta mcur = mnext;
        mnext = load_meta(nxt + 1);
        fence_proxy_async();
        issue((k + NST - 1) % NST, mcur);
      }
      mbar_wait(bars + sti, (uint32_t)((k / NST) & 1));
      compute(sti);
      __syncwarp();
    }
  }
  // fold the two halves (same heads, same dims, disjoint rows)
#pragma unroll
  for (int h = 0; h < HS; h++)
#pragma unroll
    for (int k = 0; k < DP2; k++) {
      acc[h][k].x += __shfl_xor_sync(0xffffffffu, acc[h][k].x, 16);
      acc[h][k].y += __shfl_xor_sync(0xffffffffu, acc[h][k].y, 16);
    }
  // ---- per-warp partial into the warp's own ring, then CTA combine per kind
  float* slot = reinterpret_cast<float*>(ring);  // [HS][2 + D]
  if (half == 0) {
#pragma unroll
    for (int h = 0; h < HS; h++) {
      if (sub == 0) { slot[h * (2 + D)] = ss.M[h]; slot[h * (2 + D) + 1] = ss.D[h]; }
#pragma unroll
      for (int k = 0; k < DP2; k++) {
        slot[h * (2 + D) + 2 + sub * DPL + 2 * k] = acc[h][k].x;
        slot[h * (2 + D) + 2 + sub * DPL + 2 * k + 1] = acc[h][k].y;
      }
    }
  }
  __syncthreads();
  for (int kk = 0; kk < 3; kk++) {
    for (int idx = threadIdx.x; idx < G * (2 + D); idx += blockDim.x) {
      const int h = idx / (2 + D), t = idx % (2 + D);
      float Mx = -INFINITY;
      for (int w = 0; w < CF::WARPS; w++)
        if (wkind[w] == kk) {
          const float* sl = reinterpret_cast<const float*>(at3 + (size_t)w * NST * SB) + h * (2 + D);
          if (sl[1] > 0.f) Mx = fmaxf(Mx, sl[0]);
        }
      float a = 0.f;
      if (t > 0 && Mx != -INFINITY)
        for (int w = 0; w < CF::WARPS; w++)
          if (wkind[w] == kk) {
            const float* sl = reinterpret_cast<const float*>(at3 + (size_t)w * NST * SB) + h * (2 + D);
            if (sl[1] > 0.f) a += sl[t] * __expf(sl[0] - Mx);
          }
      float* out = sv.part + ((((size_t)u * S + s_idx) * G + h) * 3 + kk) * (size_t)(2 + D);
      out[t] = t == 0 ? Mx : a;
    }
  }
}

template <typename T, int DL, int HS, bool FULL>
size_t attend_v3_smem() { return AttV3Cfg<T, DL, HS, FULL>::SMEM; }

#define WK_INST_ATT3(T, DL, HS)                                                                           \
  template __global__ void attend_v3_kernel<T, DL, HS, false>(IndexView, SteadyView, StepView, AttnParams,  \
                                                             const int32_t*);                              \
  template __global__ void attend_v3_kernel<T, DL, HS, true>(IndexView, SteadyView, StepView, AttnParams,   \
                                                            const int32_t*);                               \
  template size_t attend_v3_smem<T, DL, HS, false>();                                                      \
  template size_t attend_v3_smem<T, DL, HS, true>();
WK_INST_ATT3(__nv_bfloat16, 8, 4)
WK_INST_ATT3(__nv_bfloat16, 8, 8)
WK_INST_ATT3(__nv_bfloat16, 4, 4)
WK_INST_ATT3(__nv_bfloat16, 4, 8)
WK_INST_ATT3(float, 8, 4)
WK_INST_ATT3(float, 8, 8)
WK_INST_ATT3(float, 4, 4)
WK_INST_ATT3(float, 4, 8)

// ===========================================================================
// score_v3: grid = (nblk, U), block = 128 (4 warps); each warp streams a
// contiguous row range through a 4-stage bulk-copy ring.
// ===========================================================================
// fp64 twin of transpose_reduce32
__device__ __forceinline__ double transpose_reduce32d(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; i++) {
      const double send = up ? v[i] : v[i + off];
      const double keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

template <int HS, int DL>
struct ScoreV3Cfg {
  static constexpr int RG = 32 / HS;
  static constexpr int NST = 4;
  static constexpr int ROW = 32 * DL * 4;
  static constexpr int SB = RG * ROW;
  static constexpr size_t SMEM = (size_t)4 * NST * SB + 4 * NST * 8;
};

template <int HS, int DL>
__global__ void __launch_bounds__(128) score_v3_kernel(IndexView ix, StepView sv, int G, int rows_per_cta) {
  using CF = ScoreV3Cfg<HS, DL>;
  constexpr int RG = CF::RG, NST = CF::NST, ROW = CF::ROW, SB = CF::SB;
  const int d = 32 * DL;
  const int u = blockIdx.y;
  const int m = sv.m[u];
  const int r0 = blockIdx.x * rows_per_cta;
  if (r0 >= m) return;
  const int r1 = min(m, r0 + rows_per_cta);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(128) unsigned char sc3[];
  unsigned char* ring = sc3 + (size_t)warp * NST * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sc3 + (size_t)4 * NST * SB) + warp * NST;
  // warp's contiguous rows
  const int per = (r1 - r0 + 3) / 4;
  const int wr0 = r0 + warp * per, wr1 = min(r1, wr0 + per);
  if (lane == 0) {
    for (int i = 0; i < NST; i++) mbar_init(bars + i, 1);
    fence_mbar_init();
  }
  __syncwarp();
  float qv[HS][DL];
#pragma unroll
  for (int h = 0; h < HS; h++)
#pragma unroll
    for (int k = 0; k < DL; k++) qv[h][k] = h < G ? sv.q[((size_t)u * G + h) * d + lane * DL + k] : 0.f;
  const float* Cb = ix.C32 + (size_t)u * ix.m_cap * d;
  float* out = sv.scores + (size_t)u * G * ix.m_cap;
  const int ng = wr1 > wr0 ? (wr1 - wr0 + RG - 1) / RG : 0;
  auto issue = [&](int gi, int sti) {
    const int row0 = wr0 + gi * RG;
    const int nv = min(RG, wr1 - row0);
    if (lane == 0) {
      mbar_arrive_expect_tx(bars + sti, (uint32_t)(nv * ROW));
      bulk_g2s(ring + sti * SB, Cb + (size_t)row0 * d, (uint32_t)(nv * ROW), bars + sti);
    }
  };
#pragma unroll
  for (int i = 0; i < NST - 1; i++)
    if (i < ng) issue(i, i);
  for (int gi = 0; gi < ng; gi++) {
    const int sti = gi % NST;
    if (gi + NST - 1 < ng) {
      fence_proxy_async();
      issue(gi + NST - 1, (gi + NST - 1) % NST);
    }
    mbar_wait(bars + sti, (uint32_t)((gi / NST) & 1));
    const unsigned char* stage = ring + sti * SB;
    const int row0 = wr0 + gi * RG;
    const int nv = min(RG, wr1 - row0);
    // fp64 accumulation: fp32 x fp32 products are exact in fp64, so the only
    // error left vs the reference's fp64 dgemv is the rounding of C64 to C32
    // and of the final store (2^-23 |q||C|): the exact-selection band shrinks
    // ~100x compared with an fp32 dot.
    double v[32];
#pragma unroll
    for (int j = 0; j < RG; j++) {
      float c[DL];
      RowLoad<float, DL>::cvt(*reinterpret_cast<const typename RowLoad<float, DL>::R*>(stage + j * ROW + lane * DL * 4), c);
#pragma unroll
      for (int h = 0; h < HS; h++) {
        double a = (double)c[0] * (double)qv[h][0];
#pragma unroll
        for (int k = 1; k < DL; k++) a = fma((double)c[k], (double)qv[h][k], a);
        v[j * HS + h] = j < nv ? a : 0.0;
      }
    }
    const float tot = (float)transpose_reduce32d(v);
    const int jr = lane / HS, h = lane % HS;
    if (jr < nv && h < G) out[(size_t)h * ix.m_cap + row0 + jr] = tot;
    __syncwarp();
  }
}

template <int HS, int DL>
size_t score_v3_smem() { return ScoreV3Cfg<HS, DL>::SMEM; }
template __global__ void score_v3_kernel<4, 4>(IndexView, StepView, int, int);
template __global__ void score_v3_kernel<8, 4>(IndexView, StepView, int, int);
template __global__ void score_v3_kernel<4, 2>(IndexView, StepView, int, int);
template __global__ void score_v3_kernel<8, 2>(IndexView, StepView, int, int);
template size_t score_v3_smem<4, 4>();
template size_t score_v3_smem<8, 4>();
template size_t score_v3_smem<4, 2>();
template size_t score_v3_smem<8, 2>();

}  // namespace wk

extern "C" int wk_debug_select_timing(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, wk::g_sel_dbg, sizeof(long long) * 16 * (size_t)n) == cudaSuccess ? 0 : -2;
}
