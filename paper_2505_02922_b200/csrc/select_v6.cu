// select_v6.cu -- exact zone planning (index.py:61-93) + per-unit unions.
//
// One CTA per (unit, head).  Produces the reference's bits: the ordered
// retrieval list (top r of the fp64 dgemv score q.C, ties to the lower id,
// lexsort((arange, -s)) at index.py:75) and the estimation set (the next e,
// plan_zones index.py:79-93).
//
//   1. the head's approximate scores s' (score kernel, |s' - s| <= B) are
//      staged once in shared memory (SMS) -- every later pass reads smem;
//   2. 512 linear buckets over [min, max] locate the buckets holding rank r and
//      rank r+e; rank-by-counting inside them gives the exact r-th / (r+e)-th
//      largest s' (tau_r, tau_e);
//   3. rows with s' > tau + 2B are certainly in, s' < tau - 2B certainly out;
//      the band between and "clumps" (approx-order neighbours closer than 2B)
//      are re-scored EXACTLY with the reference's dgemv recipe on the fp64
//      centroid row -- 8 rows per warp, 4 lanes per row (one FMA chain each);
//   4. R / E membership goes to per-head bitmaps; the last CTA of the unit ORs
//      the G bitmaps and emits the unit's union: retrieval "pieces" (runs of
//      <= piece_rows contiguous store rows of one cluster + head mask) and
//      estimation rows (cluster id, head mask, per-head logits, size) -- the
//      work lists of attend_v4.
#include "common.cuh"
#include "decode_internal.h"
#include "exact_select.cuh"

#include <cooperative_groups.h>

namespace wk {

// phase timestamps for tools/sel_timing.py (a separate -DWK_SEL_TIMING build;
// compiled out of the product library)
#ifdef WK_SEL_TIMING
__device__ long long g_s6_ts[16384 * 16];
#define S6_MARK(i) do { if (threadIdx.x == 0) g_s6_ts[(size_t)blockIdx.x * 16 + (i)] = clock64(); } while (0)
#else
#define S6_MARK(i) do {} while (0)
#endif

constexpr int S6_T = 256;
constexpr int S6_NW = S6_T / 32;
constexpr int S6_NB = 2048;    // histogram buckets (linear over [min, max])
constexpr int S6_BAND = 256;   // band rows around tau_{r+e}
constexpr int S6_SMEM_M = 16384;  // largest m whose scores are staged in smem

template <int CAND>
struct Sel6Smem {
  union {
    int hist[S6_NB];                                               // passes A-B
    struct { unsigned long long fin[CAND]; double fex[CAND]; } f;  // final order
  } x;
  union {
    unsigned long long cand[CAND];  // candidates (unordered), until sorted
    double cex[CAND];               // exact scores (band / clump rows), by position
  } y;
  unsigned long long cs[CAND];      // candidates ordered (approx desc, id asc)
  int xpos[CAND];                   // positions needing an exact score
  int be_id[S6_BAND];
  double be_ex[S6_BAND];
  unsigned char be_sel[S6_BAND];
  float red[3][S6_NW];
  int wsum[4][S6_NW + 1];
  int ncand, n_in_r, nband_e, n_in_e, nx, ovf, last, b1, b2;
  int base[4];
  int ctot[4];                      // union: this CTA's slice totals (read by peers)
  float fred[3];
};


WK_DEVINL unsigned long long s6_key(float s, int id) {
  return ((unsigned long long)(~f2u_ord(s)) << 32) | (unsigned int)id;
}
WK_DEVINL float s6_score(unsigned long long k) { return u2f_ord(~(unsigned int)(k >> 32)); }
WK_DEVINL int s6_id(unsigned long long k) { return (int)(k & 0xffffffffu); }
WK_DEVINL bool s6_better(double a, int ia, double b, int ib) { return a > b || (a == b && ia < ib); }

// warp-aggregated append (all lanes of the warp call it)
template <typename V>
WK_DEVINL void s6_append(bool flag, V val, V* list, int* counter, int cap, int* ovf) {
  const unsigned mk = __ballot_sync(0xffffffffu, flag);
  if (!mk) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mk) - 1;
  int b = 0;
  if (lane == leader) b = atomicAdd(counter, __popc(mk));
  b = __shfl_sync(0xffffffffu, b, leader);
  if (flag) {
    const int pos = b + __popc(mk & ((1u << lane) - 1u));
    if (pos < cap) list[pos] = val; else *ovf = 1;
  }
}

// block reduction of three floats: (sum, max, max)
template <int CAND>
WK_DEVINL void s6_reduce3(float& a, float& b, float& c, Sel6Smem<CAND>& sm) {
  a = warp_sum(a); b = warp_max(b); c = warp_max(c);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sm.red[0][w] = a; sm.red[1][w] = b; sm.red[2][w] = c; }
  __syncthreads();
  if (w == 0) {
    float x = lane < S6_NW ? sm.red[0][lane] : 0.f;
    float y = lane < S6_NW ? sm.red[1][lane] : -INFINITY;
    float z = lane < S6_NW ? sm.red[2][lane] : -INFINITY;
    x = warp_sum(x); y = warp_max(y); z = warp_max(z);
    if (lane == 0) { sm.fred[0] = x; sm.fred[1] = y; sm.fred[2] = z; }
  }
  __syncthreads();
  a = sm.fred[0]; b = sm.fred[1]; c = sm.fred[2];
}

// block exclusive scan of four ints; returns totals in tot[]
template <int CAND>
WK_DEVINL void s6_scan4(int (&v)[4], int (&tot)[4], Sel6Smem<CAND>& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    x[i] = v[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x[i], o);
      if (lane >= o) x[i] += y;
    }
  }
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < 4; i++) sm.wsum[i][w] = x[i];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int val = lane < S6_NW ? sm.wsum[i][lane] : 0;
      int iv = val;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= o) iv += y;
      }
      if (lane < S6_NW) sm.wsum[i][lane] = iv - val;
      if (lane == S6_NW - 1) sm.base[i] = iv;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int ex = sm.wsum[i][w] + x[i] - v[i];
    tot[i] = sm.base[i];
    v[i] = ex;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// union of the unit's G zone bitmaps -> attend_v4 work lists
//
// The G CTAs of a unit form a thread-block cluster.  Once every head's R / E
// bitmaps are final in its shared memory, CTA g takes the g-th slice of the
// bitmap words (whole 128-cluster groups), per tile of S6_TWC clusters:
//   * one coalesced round trip stages the tile's cluster sizes / store
//     offsets, one DSMEM round trip copies all G heads' R / E words of the
//     tile into local smem;
//   * pass 1 counts (clusters, tokens, pieces, estimation rows) -- one warp
//     per word, one lane per bit; the CTA totals are exchanged over DSMEM for
//     the slice's output base;
//   * pass 2 emits retrieval pieces (runs of <= piece_rows contiguous store
//     rows of one cluster + head mask) and estimation rows (id, head mask,
//     size), in (word, bit) order -- the order of a single-CTA union;
//     with every head's logit s'_h(c) / sqrt(d) read from head h's staged
//     scores (DSMEM); a last cluster barrier keeps the smem alive until the
//     peers are done with it.
// ---------------------------------------------------------------------------
constexpr int S6_TWC = 2048;            // clusters per staging tile
constexpr int S6_TWW = S6_TWC / 32;     // bitmap words per tile (16 groups)

template <int CAND, bool SMS, int GM>
__device__ void s6_union_cl(const IndexView& ix, const StepView& sv, const SelParams& p, int u, int g, int m,
                            Sel6Smem<CAND>& sm, uint32_t* rbits, uint32_t* tre, float* scs) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int G = p.G, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int W = zb_words(m), NGR = W >> 2;
  const int cw0 = (NGR * g / G) << 2, cw1 = (NGR * (g + 1) / G) << 2;
  const int ntile = (cw1 - cw0 + S6_TWW - 1) / S6_TWW;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const int* coff = ix.cl_off + (size_t)u * ix.m_cap;
  // staging (the select phases' dead smem): sizes | offsets | words [2][G][S6_TWW]
  static_assert(offsetof(Sel6Smem<CAND>, red) - offsetof(Sel6Smem<CAND>, x) >=
                    (2 * S6_TWC + 2 * 8 * S6_TWW) * sizeof(int), "union staging must fit the dead select smem");
  int* csz = reinterpret_cast<int*>(&sm.x);
  int* cof = csz + S6_TWC;
  uint32_t* lw = reinterpret_cast<uint32_t*>(cof + S6_TWC);  // [R/E][h][word - tw0]
  const uint32_t rb_loc = (uint32_t)__cvta_generic_to_shared(rbits);
  const uint32_t tr_loc = (uint32_t)__cvta_generic_to_shared(tre);
  auto peer = [&](uint32_t loc, int h) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(loc), "r"(h));
    return r;
  };
  const int PR = p.piece_rows, PRS = PR == 16 ? 4 : 3;  // pieces of <= PR = 2^PRS rows
  auto stage = [&](int tw0, int tw1) {  // clusters [32 tw0, 32 tw1) + every head's words, one round trip
    constexpr int K = S6_TWC / S6_T;
    const int c0 = tw0 << 5, c1 = min(m, tw1 << 5), nw = tw1 - tw0;
    int a[K], b[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const int c = c0 + t + k * S6_T;
      a[k] = c < c1 ? __ldg(csize + c) : 0;
      b[k] = c < c1 ? __ldg(coff + c) : 0;
    }
    // words: thread t takes word t % 64 of (R/E, head) pairs t / 64, t / 64 + 4, ... (2G <= 16 pairs)
    uint32_t wv[4];
    const int w = t & (S6_TWW - 1), eh0 = t / S6_TWW;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int eh = eh0 + 4 * k, e = eh >= G, h = eh - (e ? G : 0);
      wv[k] = (eh < 2 * G && w < nw) ? dsmem_ld_u32(peer((e ? tr_loc : rb_loc) + 4u * (tw0 + w), h)) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) {
      csz[t + k * S6_T] = a[k];
      cof[t + k * S6_T] = b[k];
    }
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (eh0 + 4 * k < 2 * G) lw[(eh0 + 4 * k) * S6_TWW + w] = wv[k];
    __syncthreads();
  };
  // this warp's words of tile [tw0, tw1): contiguous block
  auto wrange = [&](int tw0, int tw1, int& a, int& b) {
    const int n = tw1 - tw0;
    a = tw0 + n * warp / S6_NW;
    b = tw0 + n * (warp + 1) / S6_NW;
  };
  auto load_words = [&](int wl, uint32_t (&rw)[GM], uint32_t (&ew)[GM], uint32_t& ur, uint32_t& ue) {
    ur = 0u; ue = 0u;
#pragma unroll
    for (int h = 0; h < GM; h++) {
      rw[h] = h < G ? lw[h * S6_TWW + wl] : 0u;
      ew[h] = h < G ? lw[(G + h) * S6_TWW + wl] : 0u;
      ur |= rw[h];
      ue |= ew[h];
    }
  };
  // per-warp counts over its words of a tile: (clusters, tokens, pieces, est rows)
  auto count = [&](int tw0, int tw1, int (&c4)[4]) {
    int a, b;
    wrange(tw0, tw1, a, b);
    int nr = 0, ne = 0, tok = 0, pcs = 0;
    for (int w = a; w < b; w++) {
      uint32_t rw[GM], ew[GM], ur, ue;
      load_words(w - tw0, rw, ew, ur, ue);
      nr += __popc(ur);
      ne += __popc(ue);
      if ((ur >> lane) & 1u) {
        const int sz = csz[zb_cluster(w, lane) - (tw0 << 5)];
        tok += sz;
        pcs += (sz + PR - 1) >> PRS;
      }
    }
    c4[0] = nr; c4[1] = tok; c4[2] = pcs; c4[3] = ne;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c4[1] += __shfl_xor_sync(0xffffffffu, c4[1], o);
      c4[2] += __shfl_xor_sync(0xffffffffu, c4[2], o);
    }
  };
  // ---- pass 1: slice totals ----
  int wc[4] = {0, 0, 0, 0};
  if (t < 4) sm.ctot[t] = 0;
  for (int k = 0; k < ntile; k++) {
    const int tw0 = cw0 + k * S6_TWW, tw1 = min(cw1, tw0 + S6_TWW);
    stage(tw0, tw1);
    count(tw0, tw1, wc);
    if (lane < 4) atomicAdd(&sm.ctot[lane], wc[lane]);
  }
  // ---- slice bases from the peers' totals (DSMEM) ----
  S6_MARK(8);
  cl.sync();
  S6_MARK(9);
  if (t < 4) {
    int base = 0, tot = 0;
    const uint32_t loc = (uint32_t)__cvta_generic_to_shared(&sm.ctot[t]);
    for (int h = 0; h < G; h++) {
      const int v = (int)dsmem_ld_u32(peer(loc, h));
      if (h < g) base += v;
      tot += v;
    }
    sm.base[t] = base;
    sm.wsum[t][0] = tot;
  }
  __syncthreads();
  const int n_ru = sm.wsum[0][0], n_rt = sm.wsum[1][0], n_pc = sm.wsum[2][0], n_eu = sm.wsum[3][0];
  // row mode (sv.rtok_row set, attend_v5): every retrieved token's store row +
  // head mask instead of the pieces
  const bool rows_mode = sv.rtok_row != nullptr;
  const bool fits = (rows_mode ? n_rt <= sv.rt_cap : n_pc <= sv.pc_cap) && n_eu <= sv.eu_cap && n_ru <= sv.ru_cap;
  if (g == 0 && t == 0) {
    if (!fits) set_status(sv.status, kErrUnion);
    sv.cnt[u * 4 + 0] = fits ? n_ru : 0;
    sv.cnt[u * 4 + 1] = fits ? n_rt : 0;
    sv.cnt[u * 4 + 2] = fits ? n_eu : 0;
    sv.cnt[u * 4 + 3] = fits ? n_pc : 0;
  }
  // ---- pass 2: emit ----
  int2* pcs = reinterpret_cast<int2*>(sv.pieces) + (size_t)u * sv.pc_cap;
  int32_t* rows = rows_mode ? sv.rtok_row + (size_t)u * sv.rt_cap : nullptr;
  int32_t* ru = sv.ru_ids + (size_t)u * sv.ru_cap;
  uint8_t* rmk = sv.ru_mask + (size_t)u * sv.ru_cap;
  int32_t* eu = sv.eu_ids + (size_t)u * sv.eu_cap;
  uint8_t* emk = sv.eu_mask + (size_t)u * sv.eu_cap;
  float* eusz = sv.eu_sz + (size_t)u * sv.eu_cap;
  float* eux = sv.eu_x + (size_t)u * sv.eu_cap * G;
  const float isd = p.inv_sqrt_d;
  const uint32_t sc_loc = SMS ? (uint32_t)__cvta_generic_to_shared(scs) : 0u;
  int tb[4] = {sm.base[0], sm.base[1], sm.base[2], sm.base[3]};  // running tile base
  const uint32_t lt = (1u << lane) - 1u;
  for (int k = 0; fits && k < ntile; k++) {
    const int tw0 = cw0 + k * S6_TWW, tw1 = min(cw1, tw0 + S6_TWW);
    if (ntile > 1) {
      stage(tw0, tw1);
      count(tw0, tw1, wc);
    }
    __syncthreads();
    if (lane < 4) sm.wsum[lane][warp + 1] = wc[lane];  // wsum[i][1..NW]: per-warp counts
    __syncthreads();
    int o[4], ttot[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      int ex = 0, all = 0;
      for (int w2 = 0; w2 < S6_NW; w2++) {
        const int v = sm.wsum[i][w2 + 1];
        if (w2 < warp) ex += v;
        all += v;
      }
      o[i] = tb[i] + ex;
      ttot[i] = all;
    }
    int a, b;
    wrange(tw0, tw1, a, b);
    S6_MARK(13);
    for (int w = a; w < b; w++) {
      uint32_t rw[GM], ew[GM], ur, ue;
      load_words(w - tw0, rw, ew, ur, ue);
      const int c = zb_cluster(w, lane);
      const int ci = c - (tw0 << 5);
      if (ur && rows_mode) {
        const bool in = (ur >> lane) & 1u;
        const int sz = in ? csz[ci] : 0;
        int x = sz;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, off);
          if (lane >= off) x += y;
        }
        int mk = 0;
#pragma unroll
        for (int h = 0; h < GM; h++) mk |= ((rw[h] >> lane) & 1u) << h;
        const int r0 = in ? cof[ci] : 0;
        if (in) {
          const int ir = o[0] + __popc(ur & lt);
          ru[ir] = c;
          rmk[ir] = (uint8_t)mk;
        }
        // the rows of each retrieved cluster of the word, written by the whole
        // warp (coalesced): one pass per cluster instead of a serial loop per lane
        for (uint32_t rem = ur; rem; rem &= rem - 1u) {
          const int src = __ffs(rem) - 1;
          const int szc = __shfl_sync(0xffffffffu, sz, src);
          const int r0c = __shfl_sync(0xffffffffu, r0, src);
          const int mkc = __shfl_sync(0xffffffffu, mk, src);
          int32_t* dst = rows + o[1] + __shfl_sync(0xffffffffu, x, src) - szc;
          for (int j = lane; j < szc; j += 32) dst[j] = (r0c + j) | (mkc << 24);
        }
        o[0] += __popc(ur);
        o[1] += __shfl_sync(0xffffffffu, x, 31);
      } else if (ur) {
        const bool in = (ur >> lane) & 1u;
        const int sz = in ? csz[ci] : 0;
        const int np = (sz + PR - 1) >> PRS;
        int x = np;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, off);
          if (lane >= off) x += y;
        }
        if (in) {
          int mk = 0;
#pragma unroll
          for (int h = 0; h < GM; h++) mk |= ((rw[h] >> lane) & 1u) << h;
          const int ir = o[0] + __popc(ur & lt);
          ru[ir] = c;
          rmk[ir] = (uint8_t)mk;
          const int r0 = cof[ci];
          int ip = o[2] + x - np;
          for (int j = 0; j < sz; j += PR) pcs[ip++] = make_int2(r0 + j, min(PR, sz - j) | (mk << 8));
        }
        o[0] += __popc(ur);
        o[2] += __shfl_sync(0xffffffffu, x, 31);
      }
      if (ue) {
        if ((ue >> lane) & 1u) {
          int mk = 0;
#pragma unroll
          for (int h = 0; h < GM; h++) mk |= ((ew[h] >> lane) & 1u) << h;
          const int ie = o[3] + __popc(ue & lt);
          eu[ie] = c;
          emk[ie] = (uint8_t)mk;
          eusz[ie] = (float)csz[ci];
          // every head's logit s'_h(c) / sqrt(d) of the row, from head h's
          // staged scores (peer smem over DSMEM, or the global score rows)
          float sc[GM];
#pragma unroll
          for (int h = 0; h < GM; h++)
            sc[h] = (h < G && ((mk >> h) & 1))
                        ? (SMS ? __uint_as_float(dsmem_ld_u32(peer(sc_loc + 4u * (uint32_t)c, h)))
                               : __ldcg(sv.scores + ((size_t)u * G + h) * ix.m_cap + c))
                        : 0.f;
          float* ex = eux + (size_t)ie * G;
#pragma unroll
          for (int h = 0; h < GM; h++)
            if (h < G) ex[h] = (mk >> h) & 1 ? sc[h] * isd : -INFINITY;
        }
        o[3] += __popc(ue);
      }
    }
    S6_MARK(14);
#pragma unroll
    for (int i = 0; i < 4; i++) tb[i] += ttot[i];
  }
  // peers may still be reading this CTA's staged scores: keep the smem alive
  S6_MARK(10);
  cl.sync();
  S6_MARK(11);
  S6_MARK(12);
}

// ---------------------------------------------------------------------------
template <int CAND, bool SMS, int GM>
__global__ void __launch_bounds__(S6_T, 4) select_v6_kernel(IndexView ix, StepView sv, SelParams p) {
  extern __shared__ __align__(16) unsigned char s6_raw[];  // Sel6Smem | SMS: scores [m] | bitmaps R, TRE [W]
  Sel6Smem<CAND>& sm = *reinterpret_cast<Sel6Smem<CAND>*>(s6_raw);
  float* s6_dyn = reinterpret_cast<float*>(s6_raw + ((sizeof(Sel6Smem<CAND>) + 15) & ~(size_t)15));
  pdl_wait();
  const int G = p.G, d = p.d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  S6_MARK(0);
  const int m = sv.m[u];
  const int t = threadIdx.x, T = S6_T, lane = t & 31, warp = t >> 5;
  const int W = zb_words(m);
  if (p.k_new && g == 0) {
    // append this step's token to the unit's steady buffer (engine.py:178-182)
    const int row = p.st.n[u];
    const bool fits = row < p.st.t_cap;
    const size_t o = ((size_t)u * p.st.t_cap + row) * d;
    for (int i = t; fits && i < d; i += T) {
      const float kv = p.k_new[(size_t)u * d + i], vv = p.v_new[(size_t)u * d + i];
      if (p.store_bf16) {  // swizzled rows (common.cuh swz_col; d in {64, 128} here)
        const int c = swz_col(i, row);
        reinterpret_cast<__nv_bfloat16*>(p.st.k)[o + c] = __float2bfloat16_rn(kv);
        reinterpret_cast<__nv_bfloat16*>(p.st.v)[o + c] = __float2bfloat16_rn(vv);
      } else {
        reinterpret_cast<float*>(p.st.k)[o + i] = kv;
        reinterpret_cast<float*>(p.st.v)[o + i] = vv;
      }
    }
    __syncthreads();  // every thread read n[u] before it advances
    if (t == 0) {
      if (fits) {
        p.st.tok[(size_t)u * p.st.t_cap + row] = p.st.next_tok[u];
        p.st.next_tok[u] += 1;
        p.st.n[u] = row + 1;
      } else {
        set_status(sv.status, kErrSteadyFull);
      }
    }
  }
  float* scs = s6_dyn;
  uint32_t* rbits = reinterpret_cast<uint32_t*>(s6_dyn + (SMS ? ((m + 3) & ~3) : 0));
  uint32_t* tre = rbits + W;  // certain or selected members of the top r+e
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
  const double* q64 = sv.q64 ? sv.q64 + ((size_t)u * G + g) * d : nullptr;
  const double* C64 = ix.C64 + (size_t)u * ix.m_cap * d;
  uint32_t* rb_out = sv.rbits + ((size_t)u * G + g) * sv.w_cap;
  uint32_t* eb_out = sv.ebits + ((size_t)u * G + g) * sv.w_cap;
  auto S_ = [&](int c) -> float { return SMS ? scs[c] : __ldcg(s + c); };
  // capacity (r fits the candidate and output lists): a configuration error
  // r beyond the candidate list (e.g. retrieval_fraction near 1) takes the
  // exact path with the ordered list built in global memory
  const bool cap_ok = m > 0 && r <= sv.r_cap && (r <= CAND || sv.xscr);
  if (m > 0 && !cap_ok) set_status(sv.status, kErrBandOverflow);
  bool ok = cap_ok && r <= CAND;
  for (int w = t; w < W; w += T) { rbits[w] = 0u; tre[w] = 0u; }
  double B2 = 0.0;
  float bk_mn = 0.f, bk_scale = 0.f;
  auto bucket = [&](float v) {
    int b = (int)((v - bk_mn) * bk_scale);
    return b < 0 ? 0 : (b >= S6_NB ? S6_NB - 1 : b);
  };
  // rigorous value range of bucket b under the float evaluation of bucket():
  // fl(fl(v - mn) * scale) in [b, b + 1)  =>  v - mn in
  // [b / (scale (1+u)^2), (b + 1) / (scale (1-u)^2)),  u = 2^-24
  auto edge_lo = [&](int b) -> double {
    return (double)bk_mn + (double)b / ((double)bk_scale * (1.0 + 1.1920928955078125e-07));
  };
  auto edge_hi = [&](int b) -> double {
    return b >= S6_NB - 1 ? (double)INFINITY
                          : (double)bk_mn + (double)(b + 1) / ((double)bk_scale * (1.0 - 1.1920928955078125e-07));
  };
  double hr = 0, lr = 0, he = 0, le = 0;
  if (m > 0) {
    // ---- pass A: stage scores, min / max, |q|^2 (always: the union reads them) ----
    float mn = INFINITY, mx = -INFINITY;
    const int m4 = m >> 2;
#pragma unroll 4
    for (int i = t; i < m4; i += T) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(s) + i);
      if (SMS) reinterpret_cast<float4*>(scs)[i] = v;
      mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int i = 4 * m4 + t; i < m; i += T) {
      const float v = __ldcg(s + i);
      if (SMS) scs[i] = v;
      mn = fminf(mn, v); mx = fmaxf(mx, v);
    }
    float qq = 0.f;
    for (int i = t; i < d; i += T) { const float qi = q[i]; qq = fmaf(qi, qi, qq); }
    for (int b = t; b < S6_NB; b += T) sm.x.hist[b] = 0;
    if (t == 0) { sm.ncand = sm.n_in_r = sm.nband_e = sm.n_in_e = sm.nx = sm.ovf = 0; sm.b1 = sm.b2 = -1; }
    float nmn = -mn;
    s6_reduce3(qq, mx, nmn, sm);
    S6_MARK(1);
    mn = -nmn;
    // |s' - s| <= B; with fp64 queries the scan's fp32 q adds 2^-24 |q| |C|
    const double B = score_error_bound_v2((double)qq, (double)ix.Cmax[u], d, p.score_mode) * (q64 ? 1.6 : 1.0);
    B2 = 2.0 * B;
    const float span = mx - mn;
    bk_mn = mn;
    bk_scale = span > 0.f ? (float)S6_NB / span : 0.f;
    // a zero span (every score tied: q = 0, q orthogonal to every centroid,
    // a single cluster) or a non-finite one goes to the exact path
    if (!(span > 0.f) || !(bk_scale < INFINITY)) ok = false;
  }
  if (ok) {
    // ---- pass B: histogram ----
#pragma unroll 4
    for (int c = t; c < m; c += T) atomicAdd(&sm.x.hist[bucket(S_(c))], 1);
    __syncthreads();
    // buckets holding rank K1 = r and K2 = r + e (descending): thread t owns
    // the 8 buckets 2047-8t .. 2040-8t
    {
      constexpr int PB = S6_NB / S6_T;
      const int K1 = r, K2 = e > 0 ? r + e : 0;
      const int top = S6_NB - 1 - PB * t;
      int h[PB], x = 0;
#pragma unroll
      for (int i = 0; i < PB; i++) { h[i] = sm.x.hist[top - i]; x += h[i]; }
      const int own = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) sm.wsum[0][warp] = x;
      __syncthreads();
      if (warp == 0) {
        const int val = lane < S6_NW ? sm.wsum[0][lane] : 0;
        int iv = val;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, iv, o);
          if (lane >= o) iv += y;
        }
        if (lane < S6_NW) sm.wsum[0][lane] = iv - val;
      }
      __syncthreads();
      int ab = sm.wsum[0][warp] + x - own;  // elements above this thread's buckets
#pragma unroll
      for (int i = 0; i < PB; i++) {
        if (ab < K1 && ab + h[i] >= K1) sm.b1 = top - i;
        if (K2 > 0 && ab < K2 && ab + h[i] >= K2) sm.b2 = top - i;
        ab += h[i];
      }
    }
    __syncthreads();
    // tau_r (the r-th largest s') lies in bucket b1, tau_e in b2: rows above
    // edge_hi + 2B are certainly in, rows below edge_lo - 2B certainly out
    const int b1 = sm.b1, b2 = sm.b2;
    if (b1 < 0 || (e > 0 && b2 < 0)) ok = false;
    hr = edge_hi(b1) + B2; lr = edge_lo(b1) - B2;
    if (e > 0) { he = edge_hi(b2) + B2; le = edge_lo(b2) - B2; }
    S6_MARK(2);
  }
  if (ok) {
    // ---- pass D: candidates for R (certain-in + band), band around tau_e,
    //      certain members of the top r+e (bitmap, one ballot per word).
    //      Float thresholds rounded outward (certain sets only shrink,
    //      candidate sets only grow); counts kept in registers.  Band rows'
    //      fp64 centroid rows are prefetched to L2 for the exact round. ----
    const float fhr = __double2float_ru(hr), flr = __double2float_rd(lr);
    const float fhe = e > 0 ? __double2float_ru(he) : INFINITY, fle = e > 0 ? __double2float_rd(le) : INFINITY;
    int cnt_in_r = 0, cnt_in_e = 0;
    // four clusters per lane: a warp covers 128 clusters = 4 zone-bitmap words
    const int mq = (m + 3) >> 2;
    for (int base = 0; base < mq; base += T) {
      const int qi = base + t;
      float v[4];
      if (SMS && qi < (m >> 2)) {
        const float4 f = reinterpret_cast<const float4*>(scs)[qi];
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = 4 * qi + k < m ? S_(4 * qi + k) : -INFINITY;
      }
      bool cand[4], bd_e[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const bool in_r = v[k] > fhr, in_e = v[k] > fhe;
        cand[k] = v[k] >= flr;
        bd_e[k] = !in_e && v[k] >= fle;
        cnt_in_r += in_r;
        cnt_in_e += in_e;
        const unsigned mie = __ballot_sync(0xffffffffu, in_e);
        if (lane == k && 4 * (base + 32 * warp) + k < m) tre[((base + 32 * warp) >> 5) * 4 + k] = mie;
      }
      // warp-aggregated appends: one warp prefix sum + one shared-memory
      // atomic per list per iteration (all four clusters of every lane)
      {
        const int nc4 = (int)cand[0] + (int)cand[1] + (int)cand[2] + (int)cand[3];
        const int nb4 = (int)bd_e[0] + (int)bd_e[1] + (int)bd_e[2] + (int)bd_e[3];
        int xc = nc4 | (nb4 << 16);  // both counts in one scan (each <= 128 per warp)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, xc, o);
          if (lane >= o) xc += y;
        }
        const int tot = __shfl_sync(0xffffffffu, xc, 31);
        if (tot) {
          int bc = 0, bb = 0;
          if (lane == 0) {
            if (tot & 0xffff) bc = atomicAdd(&sm.ncand, tot & 0xffff);
            if (tot >> 16) bb = atomicAdd(&sm.nband_e, tot >> 16);
          }
          bc = __shfl_sync(0xffffffffu, bc, 0) + (xc & 0xffff) - nc4;
          bb = __shfl_sync(0xffffffffu, bb, 0) + (xc >> 16) - nb4;
#pragma unroll
          for (int k = 0; k < 4; k++) {
            if (cand[k]) {
              if (bc < CAND) sm.y.cand[bc] = s6_key(v[k], 4 * qi + k); else sm.ovf = 1;
              bc++;
            }
            if (bd_e[k]) {
              if (bb < S6_BAND) sm.be_id[bb] = 4 * qi + k; else sm.ovf = 1;
              bb++;
            }
          }
        }
      }
    }
    cnt_in_r = __reduce_add_sync(0xffffffffu, cnt_in_r);
    cnt_in_e = __reduce_add_sync(0xffffffffu, cnt_in_e);
    if (lane == 0) {
      atomicAdd(&sm.n_in_r, cnt_in_r);
      atomicAdd(&sm.n_in_e, cnt_in_e);
    }
    __syncthreads();
    S6_MARK(3);
    const int nc = sm.ncand, nin_r = sm.n_in_r, nbe = sm.nband_e, nin_e = e > 0 ? sm.n_in_e : 0;
    if (sm.ovf || nin_r > r || nc < r || (e > 0 && (nin_e > r + e || nin_e + nbe < r + e))) {
      ok = false;
    } else {
      // the band rows' fp64 centroid rows (the exact round's input) go to L2
      // while the candidates are ordered
      const int lpr = d >> 4;  // 128-byte lines per fp64 row
      for (int i = t; i < (nc + nbe) * lpr; i += T) {
        const int row = i / lpr;
        int c;
        if (row < nc) {
          const unsigned long long kk = sm.y.cand[row];
          if (s6_score(kk) > fhr) continue;  // certainly in: exact only if it is in a clump
          c = s6_id(kk);
        } else {
          c = sm.be_id[row - nc];
        }
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(C64 + (size_t)c * d) + (i - row * lpr) * 128));
      }
      // ---- order candidates by (approx desc, id asc): rank by counting
      //      (a bitonic sort measured 2.4x slower: 36+ block barriers) ----
      for (int i = t; i < nc; i += T) {
        const unsigned long long k = sm.y.cand[i];
        int rk = 0;
        for (int j = 0; j < nc; j++) rk += sm.y.cand[j] < k ? 1 : 0;
        sm.cs[rk] = k;
      }
      __syncthreads();
      S6_MARK(4);
      // ---- positions needing an exact score: band rows and clump members ----
      for (int base = 0; base < nc; base += T) {
        const int i = base + t;
        bool need = false;
        if (i < nc) {
          sm.y.cex[i] = 0.0;
          if (i >= nin_r) need = true;
          else {
            const double si = (double)s6_score(sm.cs[i]);
            need = (i > 0 && (double)s6_score(sm.cs[i - 1]) - si <= B2) ||
                   (i + 1 < nc && si - (double)s6_score(sm.cs[i + 1]) <= B2);
          }
        }
        s6_append(need, i, sm.xpos, &sm.nx, CAND, &sm.ovf);
      }
      __syncthreads();
      // ---- one exact round: 8 rows per warp, 4 lanes per row ----
      const int nx = sm.nx, nall = nx + nbe;
      for (int b0 = warp * 8; b0 < nall; b0 += S6_NW * 8) {
        const int it = b0 + (lane >> 2);
        const bool act = it < nall;
        const int c = !act ? 0 : (it < nx ? s6_id(sm.cs[sm.xpos[it]]) : sm.be_id[it - nx]);
        const int cls = gemv_row_class(c, m, d, p.blas_threads);
        const double ex = q64 ? xs_exact_quad(C64 + (size_t)c * d, q64, d, cls, act)
                              : xs_exact_quad(C64 + (size_t)c * d, q, d, cls, act);
        if (act && (lane & 3) == 0) {
          if (it < nx) sm.y.cex[sm.xpos[it]] = ex;
          else sm.be_ex[it - nx] = ex;
        }
      }
      __syncthreads();
      S6_MARK(5);
      // ---- band winners for R: best (r - nin_r) band rows by exact score ----
      const int need_r = r - nin_r;
      for (int i = nin_r + t; i < nc; i += T) {
        int rank = 0;
        const double ci = sm.y.cex[i];
        const int ii = s6_id(sm.cs[i]);
        for (int j = nin_r; j < nc; j++) rank += s6_better(sm.y.cex[j], s6_id(sm.cs[j]), ci, ii) ? 1 : 0;
        if (rank >= need_r) sm.cs[i] = ~0ull;  // dropped
      }
      // ---- band winners for the top r+e ----
      const int need_e = r + e - nin_e;
      for (int i = t; i < nbe; i += T) {
        int rank = 0;
        for (int j = 0; j < nbe; j++) rank += s6_better(sm.be_ex[j], sm.be_id[j], sm.be_ex[i], sm.be_id[i]) ? 1 : 0;
        sm.be_sel[i] = rank < need_e ? 1 : 0;
      }
      __syncthreads();
      // compact: certain-in keep their positions, band winners follow in approx order
      for (int i = t; i < nc; i += T) {
        if (i < nin_r) { sm.x.f.fin[i] = sm.cs[i]; sm.x.f.fex[i] = sm.y.cex[i]; continue; }
        if (sm.cs[i] == ~0ull) continue;
        int before = 0;
        for (int j = nin_r; j < i; j++) before += sm.cs[j] != ~0ull ? 1 : 0;
        sm.x.f.fin[nin_r + before] = sm.cs[i];
        sm.x.f.fex[nin_r + before] = sm.y.cex[i];
      }
      for (int i = t; i < nbe; i += T)
        if (sm.be_sel[i]) atomicOr(tre + zb_word(sm.be_id[i]), 1u << zb_bit(sm.be_id[i]));
      __syncthreads();
      // every maximal run of approx-order neighbours closer than 2B was
      // exact-scored: sort each run exactly (insertion sort by its first thread)
      for (int i = t; i < r; i += T) {
        const double si = (double)s6_score(sm.x.f.fin[i]);
        const bool lp = i > 0 && (double)s6_score(sm.x.f.fin[i - 1]) - si <= B2;
        const bool ln = i + 1 < r && si - (double)s6_score(sm.x.f.fin[i + 1]) <= B2;
        if (!lp && ln) {
          int end = i + 1;
          while (end + 1 < r && (double)s6_score(sm.x.f.fin[end]) - (double)s6_score(sm.x.f.fin[end + 1]) <= B2) end++;
          for (int a = i + 1; a <= end; a++) {
            const unsigned long long kk = sm.x.f.fin[a];
            const double ev = sm.x.f.fex[a];
            int b = a - 1;
            while (b >= i && s6_better(ev, s6_id(kk), sm.x.f.fex[b], s6_id(sm.x.f.fin[b]))) {
              sm.x.f.fin[b + 1] = sm.x.f.fin[b];
              sm.x.f.fex[b + 1] = sm.x.f.fex[b];
              b--;
            }
            sm.x.f.fin[b + 1] = kk;
            sm.x.f.fex[b + 1] = ev;
          }
        }
      }
      __syncthreads();
    }
  }
  if (cap_ok && !ok && sv.xscr) {
    // ---- tie-safe exact path (exact_select.cuh): exact scores of every row,
    //      96-bit radix select of ranks r and r+e in lexsort order, R ordered
    //      by counting.  Taken on band / candidate overflow and zero spans. ----
    double* xs = sv.xscr + ((size_t)u * G + g) * ix.m_cap;
    if (q64) xs_score_rows(C64, q64, m, d, p.blas_threads, xs);
    else xs_score_rows(C64, q, m, d, p.blas_threads, xs);
    for (int w = t; w < W; w += T) { rbits[w] = 0u; tre[w] = 0u; }
    if (t == 0) sm.ncand = 0;
    __syncthreads();
    auto key = [&](int c) { return xs_key(__ldcg(xs + c)); };
    auto idf = [&](int c) { return (unsigned)c; };
    unsigned long long k1, k2 = 0ull;
    unsigned i1, i2 = 0u;
    int* hist = reinterpret_cast<int*>(&sm.y);  // 258 ints of the dead candidate list
    static_assert(sizeof(sm.y) >= 258 * sizeof(int), "radix histogram must fit");
    xs_select(m, r, key, idf, hist, k1, i1);
    if (e > 0) xs_select(m, r + e, key, idf, hist, k2, i2);
    if (r > CAND) {
      // large R: each member's position in the ordered list is its lexsort
      // rank over all rows (every better row is in R as well)
      int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
      for (int c = t; c < m; c += T) {
        const unsigned long long kk = key(c);
        if (xs_in(kk, (unsigned)c, k1, i1)) {
          int rk = 0;
          for (int j = 0; j < m; j++) {
            const unsigned long long kj = key(j);
            rk += (kj < kk) || (kj == kk && j < c);
          }
          rl_out[rk] = c;
          atomicOr(rbits + zb_word(c), 1u << zb_bit(c));
        } else if (e > 0 && xs_in(kk, (unsigned)c, k2, i2)) {
          atomicOr(tre + zb_word(c), 1u << zb_bit(c));
        }
      }
      __syncthreads();
      if (t == 0 && sv.xcount) atomicAdd(sv.xcount, 1);
      ok = true;
    } else {
    for (int c = t; c < m; c += T) {
      const unsigned long long kk = key(c);
      if (xs_in(kk, (unsigned)c, k1, i1)) {
        const int pos = atomicAdd(&sm.ncand, 1);
        sm.x.f.fin[pos] = (unsigned long long)(unsigned)c;
        sm.x.f.fex[pos] = __ldcg(xs + c);
      } else if (e > 0 && xs_in(kk, (unsigned)c, k2, i2)) {
        atomicOr(tre + zb_word(c), 1u << zb_bit(c));
      }
    }
    __syncthreads();
    // R in (exact desc, id asc) order: rank by counting into cs / cex
    for (int i = t; i < r; i += T) {
      const double ei = sm.x.f.fex[i];
      const int ii = s6_id(sm.x.f.fin[i]);
      int rk = 0;
      for (int j = 0; j < r; j++) rk += s6_better(sm.x.f.fex[j], s6_id(sm.x.f.fin[j]), ei, ii) ? 1 : 0;
      sm.cs[rk] = sm.x.f.fin[i];
    }
    __syncthreads();
    for (int i = t; i < r; i += T) sm.x.f.fin[i] = sm.cs[i];
    __syncthreads();
    if (t == 0 && sv.xcount) atomicAdd(sv.xcount, 1);
    ok = true;
    }
  }
  if (ok) {
    // ---- outputs: ordered retrieval list, R bitmap ----
    int32_t* rl_out = sv.rlist + ((size_t)u * G + g) * sv.r_cap;
    if (r <= CAND)
      for (int i = t; i < r; i += T) {
        const int c = s6_id(sm.x.f.fin[i]);
        rl_out[i] = c;
        atomicOr(rbits + zb_word(c), 1u << zb_bit(c));
      }
    __syncthreads();
    // E = top(r+e) minus R
    int32_t* el_out = sv.elist ? sv.elist + ((size_t)u * G + g) * sv.e_cap : nullptr;
    int ecnt = 0;
    for (int w = t; w < W; w += T) {
      const uint32_t ew = tre[w] & ~rbits[w];
      rb_out[w] = rbits[w];
      eb_out[w] = ew;
      tre[w] = ew;
      ecnt += __popc(ew);
    }
    if (el_out) {
      int v4[4] = {ecnt, 0, 0, 0}, tot[4];
      s6_scan4(v4, tot, sm);
      int pos = v4[0];
      for (int w = t; w < W; w += T) {
        uint32_t ew = tre[w];
        while (ew) {
          el_out[pos++] = zb_cluster(w, __ffs(ew) - 1);
          ew &= ew - 1;
        }
      }
    }
    if (p.need_tail || p.need_allc) {
      __syncthreads();
      const float isd = p.inv_sqrt_d;
      const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
      float mx_t = -INFINITY, mx_a = -INFINITY;
      for (int c = t; c < m; c += T) {
        const float xv = S_(c) * isd;
        mx_a = fmaxf(mx_a, xv);
        const bool z = ((rbits[zb_word(c)] | tre[zb_word(c)]) >> zb_bit(c)) & 1u;
        if (!z) mx_t = fmaxf(mx_t, xv);
      }
      float dummy = 0.f;
      s6_reduce3(dummy, mx_t, mx_a, sm);
      float dt = 0.f, da = 0.f, dz = -INFINITY;
      for (int c = t; c < m; c += T) {
        const float xv = S_(c) * isd;
        const float sz = (float)csize[c];
        da += sz * expf(xv - mx_a);
        const bool z = ((rbits[zb_word(c)] | tre[zb_word(c)]) >> zb_bit(c)) & 1u;
        if (!z) dt += sz * expf(xv - mx_t);
      }
      float dz2 = -INFINITY;
      s6_reduce3(dt, dz, dz2, sm);
      s6_reduce3(da, dz, dz2, sm);
      if (t == 0) { tailp[0] = mx_t; tailp[1] = dt; tailp[2] = mx_a; tailp[3] = da; }
    }
  }
  if (m > 0 && !ok) {
    set_status(sv.status, kErrBandOverflow);
    for (int w = t; w < W; w += T) { rb_out[w] = 0u; eb_out[w] = 0u; rbits[w] = 0u; tre[w] = 0u; }
  }
  if (!ok && t == 0) { tailp[0] = -INFINITY; tailp[1] = 0.f; tailp[2] = -INFINITY; tailp[3] = 0.f; }
  S6_MARK(6);
  pdl_trigger<2>();
  // ---- the unit's G CTAs (one cluster) build the union together ----
  cooperative_groups::this_cluster().sync();  // every head's R / E bitmaps final in its smem
  S6_MARK(7);
  s6_union_cl<CAND, SMS, GM>(ix, sv, p, u, g, m, sm, rbits, tre, scs);
}

#ifdef WK_SEL_TIMING
extern "C" int wk_sel_timing(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_s6_ts, sizeof(long long) * (size_t)n) == cudaSuccess ? 0 : -2;
}
#endif

size_t select_v6_dyn_smem(int m_max, bool sms, int cand) {
  const int W = zb_words(m_max);
  const size_t hdr = cand <= 512 ? sizeof(Sel6Smem<512>) : sizeof(Sel6Smem<2048>);
  return ((hdr + 15) & ~(size_t)15) + (size_t)(sms ? ((m_max + 3) & ~3) : 0) * 4 + (size_t)2 * W * 4;
}

// GM: head slots of the unit union (4 for G <= 4, else 8)
template __global__ void select_v6_kernel<512, true, 4>(IndexView, StepView, SelParams);
template __global__ void select_v6_kernel<512, false, 4>(IndexView, StepView, SelParams);
template __global__ void select_v6_kernel<2048, false, 4>(IndexView, StepView, SelParams);
template __global__ void select_v6_kernel<512, true, 8>(IndexView, StepView, SelParams);
template __global__ void select_v6_kernel<512, false, 8>(IndexView, StepView, SelParams);
template __global__ void select_v6_kernel<2048, false, 8>(IndexView, StepView, SelParams);

}  // namespace wk
