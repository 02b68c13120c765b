// attend_v4.cu -- fused tripartite decode attention (attention.py:67-148,
// engine.py:150-172), persistent flat schedule, CUDA cores: the fp32-store
// path (HeadEngine's exact drop-in).  bf16 stores run attend_v5.cu (tensor
// cores) and share att4_merge_kernel below.
//
// Work is a flat list of CHUNKS over all units: per unit u, first the steady
// zone (sinks + decode buffer, engine.py:87-96) in runs of RG contiguous rows,
// then the retrieval pieces built by select_v6 (runs of <= RG contiguous store
// rows of one cluster; the store is cluster-contiguous, store.py:51-54), then
// the estimation rows (fp32 value sums of the union estimation clusters) RG at
// a time.  A persistent grid of P CTAs x 8 warps splits the list evenly; each
// warp streams its contiguous chunk range through a private ring of NST
// shared-memory stages filled by 1-D bulk copies (cp.async.bulk / TMA): a
// chunk is 2 copies (K run, V run) plus zero-row tail copies, so the HBM reads
// are whole contiguous runs.  The warp flushes an online-softmax partial
// (max, denominator, numerator[d] per head) to global memory whenever the
// (unit, kind) of its chunks changes; att4_merge_kernel folds the partials of
// each (unit, head) with the log-sum-exp merge (attention.py:115-148) and the
// eq2 / tail modes of _final_output (engine.py:150-172).
//
// Inner loop (per chunk of RG = 32/HS rows): lanes 0-15 take even rows, lanes
// 16-31 odd rows, each lane owns DPL = d/16 contiguous dims; q.k partials of
// RG/2 rows x HS heads are reduced over the 16 lanes of a half with a
// transposed shuffle reduction; packed FFMA2 for q.k and p.v.
#include <cuda_bf16.h>

#include "common.cuh"
#include "decode_internal.h"

namespace wk {

__device__ __align__(128) unsigned char g_zero4[8192];

template <typename T, int DPL> struct Row4;
template <> struct Row4<__nv_bfloat16, 8> {
  static WK_DEVINL void ld(const unsigned char* p, float2 (&o)[4]) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    o[0] = make_float2(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xffff0000u));
    o[1] = make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xffff0000u));
    o[2] = make_float2(__uint_as_float(r.z << 16), __uint_as_float(r.z & 0xffff0000u));
    o[3] = make_float2(__uint_as_float(r.w << 16), __uint_as_float(r.w & 0xffff0000u));
  }
};
template <> struct Row4<__nv_bfloat16, 4> {
  static WK_DEVINL void ld(const unsigned char* p, float2 (&o)[2]) {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    o[0] = make_float2(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xffff0000u));
    o[1] = make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xffff0000u));
  }
};
template <> struct Row4<float, 8> {
  static WK_DEVINL void ld(const unsigned char* p, float2 (&o)[4]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    o[0] = make_float2(a.x, a.y); o[1] = make_float2(a.z, a.w); o[2] = make_float2(b.x, b.y); o[3] = make_float2(b.z, b.w);
  }
};
template <> struct Row4<float, 4> {
  static WK_DEVINL void ld(const unsigned char* p, float2 (&o)[2]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    o[0] = make_float2(a.x, a.y); o[1] = make_float2(a.z, a.w);
  }
};

// 16 values summed over the 16 lanes of each half-warp; lane keeps index lane&15
WK_DEVINL float att4_treduce16(float (&v)[16]) {
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

template <typename T, int DPL, int HS>
struct Att4Cfg {
  static constexpr int RG = HS == 4 ? 16 : 8;      // rows per chunk
  static constexpr int NL = (RG / 2) * HS / 16;    // (row, head) logits per lane after the reduction
  static constexpr int NST = RG == 16 ? 2 : 3;     // ring stages per warp
  static constexpr int D = 16 * DPL;
  static constexpr int ROWT = D * (int)sizeof(T);  // K or V row bytes
  static constexpr int ROWV = D * 4;               // value-sum row bytes
  static constexpr int SB = ((2 * RG * ROWT > RG * ROWV ? 2 * RG * ROWT : RG * ROWV) + 127) / 128 * 128;
  // one CTA per SM: 12 warps when the ring fits (<= 168 registers, no spills)
  static constexpr int WARPS = HS == 8 ? 8 : (SB <= 8192 ? 12 : 6);
  static constexpr int MAXU = 1024;                // units per launch (smem chunk prefix)
  // per warp: stage tags + per-stage estimation inputs (x, w per lane slot) + p broadcast buffer
  static constexpr int META = NST * (16 + NL * 32 * 8) + RG * HS * 4;
  static constexpr size_t SMEM = (size_t)WARPS * NST * SB + (size_t)WARPS * NST * 8 + (size_t)WARPS * META +
                                 (size_t)(MAXU + 1) * 4 + 64;
};

// chunk counts of unit u
template <int RG>
WK_DEVINL void att4_counts(const SteadyView& st, const StepView& sv, const int32_t* n_store, bool full, int u,
                           int& c0, int& c1, int& c2) {
  const int n_st = st.n[u];
  c0 = (n_st + RG - 1) / RG;
  if (full) {
    c1 = (n_store[u] + RG - 1) / RG;
    c2 = 0;
  } else {
    c1 = sv.cnt[u * 4 + 3];
    c2 = (sv.cnt[u * 4 + 2] + RG - 1) / RG;
  }
}

// first warp (of W) whose balanced range [N w / W, N (w+1) / W) holds chunk c
WK_DEVINL int att4_warp_of(long long c, long long N, long long W) { return (int)(((c + 1) * W + N - 1) / N - 1); }

template <typename T, int DPL, int HS, bool FULL, bool OFF>
__global__ void __launch_bounds__(Att4Cfg<T, DPL, HS>::WARPS * 32, 1) attend_v4_kernel(IndexView ix, SteadyView st, StepView sv, AttnParams p,
                                                            const int32_t* __restrict__ n_store, int U) {
  using CF = Att4Cfg<T, DPL, HS>;
  constexpr int RG = CF::RG, NST = CF::NST, ROWT = CF::ROWT, ROWV = CF::ROWV, SB = CF::SB, NL = CF::NL;
  constexpr int D = CF::D, RH = RG / 2, DP2 = DPL / 2;
  pdl_wait();
  const int G = p.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, sub = lane & 15;
  extern __shared__ __align__(128) unsigned char a4s[];
  unsigned char* ring = a4s + (size_t)warp * NST * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(a4s + (size_t)CF::WARPS * NST * SB) + warp * NST;
  unsigned char* meta = a4s + (size_t)CF::WARPS * NST * SB + (size_t)CF::WARPS * NST * 8 + (size_t)warp * CF::META;
  int4* stag = reinterpret_cast<int4*>(meta);                          // [NST] chunk tags
  float* sx = reinterpret_cast<float*>(meta + NST * 16);               // [NST][NL][32] estimation logits
  float* sw = sx + NST * NL * 32;                                      // [NST][NL][32] their weights
  float* pbuf = reinterpret_cast<float*>(meta + NST * (16 + NL * 32 * 8));  // [RG][HS] chunk weights
  int* woff = reinterpret_cast<int*>(a4s + (size_t)CF::WARPS * NST * SB + (size_t)CF::WARPS * NST * 8 +
                                     (size_t)CF::WARPS * CF::META);

  // ---- chunk prefix over units (every CTA; U <= MAXU) ----
  {
    int carry = 0;
    for (int base = 0; base < U; base += blockDim.x) {
      const int u = base + threadIdx.x;
      int c = 0;
      if (u < U) {
        int c0, c1, c2;
        att4_counts<RG>(st, sv, n_store, FULL, u, c0, c1, c2);
        c = c0 + c1 + c2;
      }
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int* ws = woff + CF::MAXU + 1;  // <= 16 ints of scratch past woff (within the +64 pad)
      if (lane == 31) ws[warp] = x;
      __syncthreads();
      int wbase = 0;
      for (int w = 0; w < warp; w++) wbase += ws[w];
      int tot = 0;
      for (int w = 0; w < CF::WARPS; w++) tot += ws[w];
      if (u < U) woff[u] = carry + wbase + x - c;
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) woff[U] = carry;
    __syncthreads();
  }
  const long long Ntot = woff[U];
  const long long Wtot = (long long)gridDim.x * CF::WARPS;
  const int wg = blockIdx.x * CF::WARPS + warp;
  if (blockIdx.x == 0 && sv.woff)
    for (int i = threadIdx.x; i <= U; i += blockDim.x) sv.woff[i] = woff[i];
  const long long ca = Ntot * wg / Wtot, cb = Ntot * (wg + 1) / Wtot;

  if (lane == 0) {
    for (int i = 0; i < NST; i++) mbar_init(bars + i, 1);
    fence_mbar_init();
  }
  __syncwarp();

  const float isd = p.inv_sqrt_d;
  const int allmask = (1 << G) - 1;
  // after the reduction lane (half, sub) holds the logits of (row jl(l), head h_own), l < NL
  const int h_own = sub % HS;
  auto jl = [&](int l) { return half + 2 * ((l * 16 + sub) / HS); };

  // ---- issue cursor: (unit, kind, local chunk) of chunk ci ----
  int iu = 0;
  {
    // binary search: last u with woff[u] <= ca
    int lo = 0, hi = U - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (woff[mid] <= ca) lo = mid; else hi = mid - 1;
    }
    iu = lo;
  }
  int ic0 = 0, ic1 = 0, ic2 = 0;
  if (ca < cb) att4_counts<RG>(st, sv, n_store, FULL, iu, ic0, ic1, ic2);

  // chunk metadata is loaded one chunk ahead of its bulk-copy issue so the
  // loads (piece words, estimation inputs) are in flight during a compute
  int in_st = 0;  // steady rows of the cursor's unit
  if (ca < cb) in_st = st.n[iu];
  struct Meta {
    int h;  // unit (bits 0-19) | kind + 1 (20-21) | n (22-26)
    int a;  // first row (kinds 0/1) or the lane's estimation cluster (kind 2)
    int mk; // head mask (kinds 0/1)
    float x[NL], w[NL];  // kind 2: lane slots' logits / weights; offload kind 1: cluster, first token
  };
  auto chunk_meta = [&](long long ci) {
    Meta m;
    m.h = 0; m.a = 0; m.mk = 0;
#pragma unroll
    for (int l = 0; l < NL; l++) { m.x[l] = -INFINITY; m.w[l] = 0.f; }
    if (ci >= cb) return m;
    while (ci >= woff[iu + 1]) {
      iu++;
      att4_counts<RG>(st, sv, n_store, FULL, iu, ic0, ic1, ic2);
      in_st = st.n[iu];
    }
    int lc = (int)(ci - woff[iu]);
    const int u = iu;
    int kind, n;
    if (lc < ic0) {
      kind = 0;
      m.a = lc * RG;
      n = min(RG, in_st - m.a);
      m.mk = allmask;
    } else if (lc < ic0 + ic1) {
      kind = 1;
      lc -= ic0;
      if (FULL) {
        m.a = lc * RG;
        n = min(RG, n_store[u] - m.a);
        m.mk = allmask;
      } else if (OFF) {
        // offload piece: (row, n | mask << 8 | flags << 16, cluster, first token)
        const int4 pc = __ldcg(reinterpret_cast<const int4*>(sv.pieces) + (size_t)u * sv.pc_cap + lc);
        m.a = pc.x;
        n = -1;
        m.mk = pc.y;
        m.x[0] = __int_as_float(pc.z);
        m.w[0] = __int_as_float(pc.w);
      } else {
        const int2 pc = __ldcg(reinterpret_cast<const int2*>(sv.pieces) + (size_t)u * sv.pc_cap + lc);
        m.a = pc.x;
        n = -1;        // decoded at issue (pc.y in mk)
        m.mk = pc.y;
      }
    } else {
      kind = 2;
      lc -= ic0 + ic1;
      const int e0 = lc * RG;
      n = min(RG, sv.cnt[u * 4 + 2] - e0);
      if (lane < n) m.a = __ldcg(sv.eu_ids + (size_t)u * sv.eu_cap + e0 + lane);
      // lane slot (row jl, head h_own): logit sigma * q.C and cluster size
      // (select_v6's cluster union)
#pragma unroll
      for (int l = 0; l < NL; l++)
        if (jl(l) < n && h_own < G) {
          m.x[l] = __ldcg(sv.eu_x + ((size_t)u * sv.eu_cap + e0 + jl(l)) * G + h_own);
          m.w[l] = __ldcg(sv.eu_sz + (size_t)u * sv.eu_cap + e0 + jl(l));
        }
    }
    m.h = u | ((kind + 1) << 20) | ((n & 31) << 22);
    return m;
  };
  auto issue = [&](int sti, const Meta& m) {
    const int u = m.h & 0xfffff, kind = ((m.h >> 20) & 3) - 1;
    int n = (m.h >> 22) & 31, mk = m.mk, flags = 0;
    if (kind == 1 && !FULL) { n = m.mk & 0xff; mk = (m.mk >> 8) & 0xff; flags = OFF ? (m.mk >> 16) & 3 : 0; }
    unsigned char* stage = ring + sti * SB;
    if (kind < 2) {
      const unsigned char* srck;
      const unsigned char* srcv;
      if (kind == 0) {
        srck = (const unsigned char*)st.k + ((size_t)u * st.t_cap + m.a) * ROWT;
        srcv = (const unsigned char*)st.v + ((size_t)u * st.t_cap + m.a) * ROWT;
      } else if (OFF && (flags & 1)) {  // offload hit: the HBM slot arena
        srck = (const unsigned char*)sv.arena_k + ((size_t)u * sv.arena_rows + m.a) * ROWT;
        srcv = (const unsigned char*)sv.arena_v + ((size_t)u * sv.arena_rows + m.a) * ROWT;
      } else {  // in-HBM store, or an offload miss: the pinned host store (zero-copy TMA)
        srck = (const unsigned char*)ix.store_k + ((size_t)u * ix.s_cap + m.a) * ROWT;
        srcv = (const unsigned char*)ix.store_v + ((size_t)u * ix.s_cap + m.a) * ROWT;
      }
      // K rows >= n stay stale (their logits are masked to -inf); V rows >= n are
      // zero-filled so p = 0 never meets a non-finite stale value
      if (lane == 0) {
        mbar_arrive_expect_tx(bars + sti, (uint32_t)((n + RG) * ROWT));
        bulk_g2s(stage, srck, (uint32_t)(n * ROWT), bars + sti);
        bulk_g2s(stage + RG * ROWT, srcv, (uint32_t)(n * ROWT), bars + sti);
        if (n < RG) bulk_g2s(stage + RG * ROWT + n * ROWT, g_zero4, (uint32_t)((RG - n) * ROWT), bars + sti);
      }
    } else {
      if (lane == 0) mbar_arrive_expect_tx(bars + sti, (uint32_t)(RG * ROWV));
      __syncwarp();
      if (lane < n)
        bulk_g2s(stage + lane * ROWV, ix.VS32 + ((size_t)u * ix.m_cap + m.a) * D, (uint32_t)ROWV, bars + sti);
      if (lane == 0 && n < RG) bulk_g2s(stage + n * ROWV, g_zero4, (uint32_t)((RG - n) * ROWV), bars + sti);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        sx[(sti * NL + l) * 32 + lane] = m.x[l];
        sw[(sti * NL + l) * 32 + lane] = m.w[l];
      }
    }
    // tag: (unit, kind + 1 | rows << 8 | head mask << 16, cluster, first token | write-through << 31)
    if (lane == 0)
      stag[sti] = make_int4(u, (kind + 1) | (n << 8) | (mk << 16),
                            (OFF && kind == 1 && (flags & 2)) ? __float_as_int(m.x[0]) : 0,
                            (OFF && kind == 1 && (flags & 2)) ? ((__float_as_int(m.w[0]) & 0xffffff) | (int)0x80000000) : 0);
  };

  // ---- q of the current unit (pre-scaled), softmax state, accumulators ----
  float2 qv[HS][DP2];
  int qu = -1;
  auto load_q = [&](int u) {
#pragma unroll
    for (int h = 0; h < HS; h++)
#pragma unroll
      for (int k = 0; k < DP2; k++) {
        const float* qp = sv.q + ((size_t)u * G + (h < G ? h : 0)) * D + sub * DPL + 2 * k;
        qv[h][k] = h < G ? make_float2(__ldg(qp) * isd, __ldg(qp + 1) * isd) : make_float2(0.f, 0.f);
      }
    qu = u;
  };
  // Lazily rescaled online softmax: per head a reference mref (uniform over
  // the warp); weights p = exp(x - mref) <= e^10 are accumulated without
  // rescaling, and the accumulators are rescaled only when some logit exceeds
  // its head's reference by more than 10 (a warp vote).  Each lane keeps the
  // denominator partial of its own (row, head) slot; partials are reduced
  // over the lanes of a head at flush.  The merge is exact for any reference.
  float mref[HS];
  float dl;
  float2 acc[HS][DP2];
  auto reset = [&]() {
    dl = 0.f;
#pragma unroll
    for (int h = 0; h < HS; h++) {
      mref[h] = -INFINITY;
#pragma unroll
      for (int k = 0; k < DP2; k++) acc[h][k] = make_float2(0.f, 0.f);
    }
  };
  reset();
  int cu = -1, ck = -1;  // (unit, kind) of the open partial
  auto flush = [&]() {
    if (cu < 0) return;
#pragma unroll
    for (int h = 0; h < HS; h++)
#pragma unroll
      for (int k = 0; k < DP2; k++) {
        acc[h][k].x += __shfl_xor_sync(0xffffffffu, acc[h][k].x, 16);
        acc[h][k].y += __shfl_xor_sync(0xffffffffu, acc[h][k].y, 16);
      }
    float dsum = dl;
#pragma unroll
    for (int off = HS; off < 32; off <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
    const size_t slot = (size_t)(wg + cu);
    if (half == 0) {
#pragma unroll
      for (int h = 0; h < HS; h++) {
        if (h < G) {
          float* dst = sv.part + ((slot * 3 + ck) * G + h) * (size_t)(4 + D);  // (M, D, -, -, num[D])
          if (sub == h) { dst[0] = mref[h]; dst[1] = dsum; }
#pragma unroll
          for (int k = 0; k < DP2; k++) *reinterpret_cast<float2*>(dst + 4 + sub * DPL + 2 * k) = acc[h][k];
        }
      }
    }
    reset();
  };

  // tg = the stage's tag: kind + 1 | rows << 8 | head mask << 16
  auto compute = [&](int sti, int tagw) {
    const int kind = (tagw & 0xff) - 1, nrow = (tagw >> 8) & 0xff, hmask = (tagw >> 16) & 0xff;
    const unsigned char* stage = ring + sti * SB;
    float x[NL], wz[NL];
    if (kind < 2) {
      float v[NL][16];
#pragma unroll
      for (int jj = 0; jj < RH; jj++) {
        const int j = half + 2 * jj;
        float2 kf[DP2];
        Row4<T, DPL>::ld(stage + j * ROWT + sub * DPL * (int)sizeof(T), kf);
#pragma unroll
        for (int h = 0; h < HS; h++) {
          float2 a2 = __fmul2_rn(kf[0], qv[h][0]);
#pragma unroll
          for (int k = 1; k < DP2; k++) a2 = __ffma2_rn(kf[k], qv[h][k], a2);
          const int idx = jj * HS + h;
          v[idx >> 4][idx & 15] = a2.x + a2.y;
        }
      }
      const bool hon = (hmask >> h_own) & 1;
#pragma unroll
      for (int l = 0; l < NL; l++) {
        x[l] = att4_treduce16(v[l]);
        if (!(hon && jl(l) < nrow)) x[l] = -INFINITY;
        wz[l] = 1.f;
      }
    } else {
#pragma unroll
      for (int l = 0; l < NL; l++) {
        x[l] = sx[(sti * NL + l) * 32 + lane];
        wz[l] = sw[(sti * NL + l) * 32 + lane];
      }
    }
    float mo = mref[0];
#pragma unroll
    for (int h = 1; h < HS; h++)
      if (h == h_own) mo = mref[h];
    float xm = x[0];
#pragma unroll
    for (int l = 1; l < NL; l++) xm = fmaxf(xm, x[l]);
    if (__any_sync(0xffffffffu, xm > mo + 10.f)) {
      // raise the references of the heads whose chunk max exceeds them
      float mx = xm;
#pragma unroll
      for (int off = HS; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
#pragma unroll
      for (int h = 0; h < HS; h++) {
        const float mh = __shfl_sync(0xffffffffu, mx, h);
        if (mh > mref[h]) {
          const float alpha = mref[h] == -INFINITY ? 0.f : __expf(mref[h] - mh);
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int k = 0; k < DP2; k++) acc[h][k] = __fmul2_rn(acc[h][k], a2);
          if (h == h_own) dl *= alpha;
          mref[h] = mh;
        }
      }
      mo = mref[0];
#pragma unroll
      for (int h = 1; h < HS; h++)
        if (h == h_own) mo = mref[h];
    }
#pragma unroll
    for (int l = 0; l < NL; l++) {
      const float pw = x[l] == -INFINITY ? 0.f : __expf(x[l] - mo);
      dl = fmaf(pw, wz[l], dl);
      pbuf[jl(l) * HS + h_own] = pw;
    }
    __syncwarp();
#pragma unroll
    for (int jj = 0; jj < RH; jj++) {
      const int j = half + 2 * jj;
      float2 vf[DP2];
      if (kind < 2) Row4<T, DPL>::ld(stage + RG * ROWT + j * ROWT + sub * DPL * (int)sizeof(T), vf);
      else Row4<float, DPL>::ld(stage + j * ROWV + sub * DPL * 4, vf);
      float pj[HS];
#pragma unroll
      for (int h4 = 0; h4 < HS; h4 += 4) {
        const float4 p4 = *reinterpret_cast<const float4*>(pbuf + j * HS + h4);
        pj[h4] = p4.x; pj[h4 + 1] = p4.y; pj[h4 + 2] = p4.z; pj[h4 + 3] = p4.w;
      }
#pragma unroll
      for (int h = 0; h < HS; h++) {
        const float2 p2 = make_float2(pj[h], pj[h]);
#pragma unroll
        for (int k = 0; k < DP2; k++) acc[h][k] = __ffma2_rn(p2, vf[k], acc[h][k]);
      }
    }
  };

  const int nch = (int)(cb - ca);
  if (nch > 0) {
#pragma unroll
    for (int i = 0; i < NST - 1; i++)
      if (i < nch) issue(i, chunk_meta(ca + i));
    Meta mnext = chunk_meta(ca + NST - 1);
    for (int k = 0; k < nch; k++) {
      const int sti = k % NST;
      if (k + NST - 1 < nch) {
        fence_proxy_async();
        __syncwarp();
        issue((k + NST - 1) % NST, mnext);
        mnext = chunk_meta(ca + k + NST);
      }
      __syncwarp();
      const int4 tg = stag[sti];
      const int tkind = (tg.y & 0xff) - 1;
      if (tg.x != cu || tkind != ck) {
        flush();
        cu = tg.x;
        ck = tkind;
        if (qu != cu) load_q(cu);
      }
      mbar_wait(bars + sti, (uint32_t)((k / NST) & 1));
      compute(sti, tg.y);
      if (OFF && tg.w < 0) {
        // admitted offload miss: write its rows through into the new slots
        const int cl = tg.z, j0 = tg.w & 0xffffff, nrow = (tg.y >> 8) & 0xff;
        const int bt = sv.block_tokens;
        const int32_t* sl = sv.slot_ids + (size_t)cu * sv.slot_cap;
        const int so = __ldg(sv.slot_off + (size_t)cu * ix.m_cap + cl);
        const unsigned char* stage = ring + sti * SB;
        for (int i = half; i < nrow; i += 2) {
          const int tok = j0 + i;
          const size_t arow = (size_t)cu * sv.arena_rows + (size_t)__ldcg(sl + so + tok / bt) * bt + tok % bt;
          for (int o = sub * 16; o < ROWT; o += 256) {
            *reinterpret_cast<uint4*>((unsigned char*)sv.arena_k + arow * ROWT + o) =
                *reinterpret_cast<const uint4*>(stage + i * ROWT + o);
            *reinterpret_cast<uint4*>((unsigned char*)sv.arena_v + arow * ROWT + o) =
                *reinterpret_cast<const uint4*>(stage + RG * ROWT + i * ROWT + o);
          }
        }
      }
      __syncwarp();
    }
    pdl_trigger<4>();
    flush();
  }
}

// ---------------------------------------------------------------------------
// merge: one warp per (unit, head); lane owns d/32 dims
// ---------------------------------------------------------------------------
template <bool FULL, int DL>
__global__ void __launch_bounds__(128) att4_merge_kernel(SteadyView st, StepView sv, AttnParams p,
                                                          const int32_t* __restrict__ n_store, int U, int Wtot,
                                                          int RG, int rows_mode) {
  // one CTA (4 warps) per (unit, head): the partial records are split over
  // the warps so ~4x more loads are in flight than with one warp per head
  pdl_wait();
  pdl_trigger<8>();
  const int G = p.G, d = p.d, D2 = 4 + d;  // partial record: (M, D, -, -, num[d])
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, t = threadIdx.x;
  __shared__ float s_m[3][4];
  __shared__ float s_d[3][4];
  __shared__ float s_n[3][4][128];
  const long long N = sv.woff[U];
  int c0, c1, c2;
  {
    const int n_st = st.n[u];
    c0 = (n_st + RG - 1) / RG;
    if (FULL) { c1 = (n_store[u] + RG - 1) / RG; c2 = 0; }
    else {
      // retrieval chunks: the pieces, or (attend_v5 row mode) RG retrieved rows each
      c1 = rows_mode ? (sv.cnt[u * 4 + 1] + RG - 1) / RG : sv.cnt[u * 4 + 3];
      c2 = (sv.cnt[u * 4 + 2] + RG - 1) / RG;
    }
  }
  const long long ub = sv.woff[u];
  const long long kb[4] = {ub, ub + c0, ub + c0 + c1, ub + c0 + c1 + c2};
  int nk[3], wk0[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    nk[k] = 0;
    wk0[k] = 0;
    if (kb[k + 1] > kb[k]) {
      wk0[k] = att4_warp_of(kb[k], N, Wtot);
      nk[k] = att4_warp_of(kb[k + 1] - 1, N, Wtot) - wk0[k] + 1;
    }
  }
  const int S = nk[0] + nk[1] + nk[2];
  auto item = [&](int i, int& k, int& w) {
    k = i < nk[0] ? 0 : (i < nk[0] + nk[1] ? 1 : 2);
    w = wk0[k] + i - (k == 0 ? 0 : (k == 1 ? nk[0] : nk[0] + nk[1]));
  };
  auto rec = [&](int k, int w) { return sv.part + (((size_t)(w + u) * 3 + k) * G + g) * (size_t)D2; };
  // empty ranges wrote nothing; with at least one chunk per warp every range is live (no division)
  const bool all_live = N >= (long long)Wtot;
  auto live_w = [&](int w) { return all_live || N * w / Wtot < N * (w + 1) / Wtot; };
  // one pass: warp w folds its items i = w, w + 4, ... against per-warp, per-kind
  // maxima (the value rows of the first 8 items are loaded together with the
  // (M, D) words -- one round trip); warps are combined in shared memory.
  const int Sw = (S - warp + 3) / 4;  // items of this warp
  float mw[3] = {-INFINITY, -INFINITY, -INFINITY}, dw3[3] = {0.f, 0.f, 0.f};
  float nacc[3][DL];
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int j = 0; j < DL; j++) nacc[k][j] = 0.f;
  auto vload = [&](int i, float (&v)[DL]) {
    int k, w;
    item(i, k, w);
    const float* src = rec(k, w) + 4 + lane * DL;
    if (DL == 4) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
      v[0] = x.x; v[1] = x.y; v[2 % DL] = x.z; v[3 % DL] = x.w;
    } else {
      const float2 x = __ldcg(reinterpret_cast<const float2*>(src));
      v[0] = x.x; v[1 % DL] = x.y;
    }
  };
  constexpr int PF = 8;
  for (int i0 = 0; i0 < Sw; i0 += 32) {
    const int nw = min(32, Sw - i0);
    float pv[PF][DL];
#pragma unroll
    for (int j = 0; j < PF; j++)
      if (j < nw) vload(warp + 4 * (i0 + j), pv[j]);
    float M = -INFINITY, Dw = 0.f;
    int kl = 0;
    if (lane < nw) {
      int w;
      item(warp + 4 * (i0 + lane), kl, w);
      if (live_w(w)) {
        const float* r = rec(kl, w);
        Dw = __ldcg(r + 1);
        M = Dw > 0.f ? __ldcg(r) : -INFINITY;
      }
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const float bm = warp_max(kl == k ? M : -INFINITY);
      if (bm > mw[k]) {  // raise the running maximum of kind k (first batch: from -inf)
        const float alpha = mw[k] == -INFINITY ? 0.f : expf(mw[k] - bm);
        dw3[k] *= alpha;
#pragma unroll
        for (int j = 0; j < DL; j++) nacc[k][j] *= alpha;
        mw[k] = bm;
      }
    }
    const float mk = kl == 0 ? mw[0] : (kl == 1 ? mw[1] : mw[2]);
    const float sc = Dw > 0.f ? __expf(M - mk) : 0.f;
    if (kl == 0) dw3[0] += Dw * sc; else if (kl == 1) dw3[1] += Dw * sc; else dw3[2] += Dw * sc;
    auto fold = [&](int j, const float (&v)[DL]) {
      const float swt = __shfl_sync(0xffffffffu, sc, j);
      const int kj = __shfl_sync(0xffffffffu, kl, j);
      // partials of empty-range warps may hold stale bits: weight 0 selects them out
#pragma unroll
      for (int jj = 0; jj < DL; jj++) {
        const float add = swt != 0.f ? v[jj] * swt : 0.f;
        nacc[0][jj] += kj == 0 ? add : 0.f;
        nacc[1][jj] += kj == 1 ? add : 0.f;
        nacc[2][jj] += kj == 2 ? add : 0.f;
      }
    };
#pragma unroll
    for (int j = 0; j < PF; j++)
      if (j < nw) fold(j, pv[j]);
    for (int j = PF; j < nw; j++) {
      float v[DL];
      vload(warp + 4 * (i0 + j), v);
      fold(j, v);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; k++) dw3[k] = warp_sum(dw3[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 3; k++) { s_m[k][warp] = mw[k]; s_d[k][warp] = dw3[k]; }
  }
#pragma unroll
  for (int jj = 0; jj < DL; jj++) {
    s_n[0][warp][lane * DL + jj] = nacc[0][jj];
    s_n[1][warp][lane * DL + jj] = nacc[1][jj];
    s_n[2][warp][lane * DL + jj] = nacc[2][jj];
  }
  __syncthreads();
  if (warp != 0) return;
  double kM[3];
  double kD[3];
  float num[3][DL];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const float m = fmaxf(fmaxf(s_m[k][0], s_m[k][1]), fmaxf(s_m[k][2], s_m[k][3]));
    kM[k] = m;
    float f[4];
#pragma unroll
    for (int w = 0; w < 4; w++) f[w] = s_m[k][w] == -INFINITY ? 0.f : expf(s_m[k][w] - m);
    kD[k] = (double)(s_d[k][0] * f[0]) + s_d[k][1] * f[1] + s_d[k][2] * f[2] + s_d[k][3] * f[3];
#pragma unroll
    for (int jj = 0; jj < DL; jj++) {
      const int o = lane * DL + jj;
      num[k][jj] = ((s_n[k][0][o] * f[0] + s_n[k][1][o] * f[1]) + (s_n[k][2][o] * f[2] + s_n[k][3][o] * f[3]));
    }
  }
  const float zero4[4] = {-INFINITY, 0.f, -INFINITY, 0.f};
  const float* tl = (!FULL && sv.tail) ? sv.tail + ((size_t)u * G + g) * 4 : zero4;
  const bool live0 = kD[0] > 0, live1 = kD[1] > 0, live2 = kD[2] > 0;
  const bool live3 = p.tail_denominator_only && tl[1] > 0.f;
  double gmax = -INFINITY;
  if (live0) gmax = fmax(gmax, kM[0]);
  if (live1) gmax = fmax(gmax, kM[1]);
  if (live2) gmax = fmax(gmax, kM[2]);
  if (live3) gmax = fmax(gmax, (double)tl[0]);
  if (gmax == -INFINITY) {  // merge requires a non-empty partial (attention.py:117-119)
    if (lane == 0) set_status(sv.status, kErrEmptyMerge);
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
  float* out = sv.out + ((size_t)u * G + g) * d;
#pragma unroll
  for (int i = 0; i < DL; i++) {
    const double v = (double)num[0][i] * sc0 + (double)num[1][i] * sc1 + (double)num[2][i] * sc2;
    out[lane * DL + i] = (float)(v * out_scale);
  }
  if (lane == 0) {
    sv.logden[(size_t)u * G + g] = (float)logden;
    sv.cov[(size_t)u * G + g] = (float)cov;
  }
}

template <typename T, int DPL, int HS, bool FULL>
size_t attend_v4_smem() { return Att4Cfg<T, DPL, HS>::SMEM; }
template <typename T, int DPL, int HS>
int attend_v4_warps() { return Att4Cfg<T, DPL, HS>::WARPS; }

#define WK_INST_ATT4(T, DL, HS)                                                                                   \
  template __global__ void attend_v4_kernel<T, DL, HS, false, false>(IndexView, SteadyView, StepView, AttnParams,   \
                                                                    const int32_t*, int);                          \
  template __global__ void attend_v4_kernel<T, DL, HS, false, true>(IndexView, SteadyView, StepView, AttnParams,    \
                                                                   const int32_t*, int);                           \
  template __global__ void attend_v4_kernel<T, DL, HS, true, false>(IndexView, SteadyView, StepView, AttnParams,    \
                                                                   const int32_t*, int);                           \
  template size_t attend_v4_smem<T, DL, HS, false>();                                                              \
  template size_t attend_v4_smem<T, DL, HS, true>();                                                               \
  template int attend_v4_warps<T, DL, HS>();
WK_INST_ATT4(float, 8, 4)
WK_INST_ATT4(float, 8, 8)
WK_INST_ATT4(float, 4, 4)
WK_INST_ATT4(float, 4, 8)
template __global__ void att4_merge_kernel<false, 4>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int);
template __global__ void att4_merge_kernel<true, 4>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int);
template __global__ void att4_merge_kernel<false, 2>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int);
template __global__ void att4_merge_kernel<true, 2>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int);

}  // namespace wk
