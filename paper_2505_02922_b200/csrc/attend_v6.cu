// attend_v6.cu -- fused tripartite decode attention (attention.py:67-148,
// engine.py:150-172) for bf16 K/V stores, warp-specialised.
//
// The arithmetic is attend_v5's (q.k and p.v of the exact zones on the bf16
// tensor cores with an exact three-term split of q and of the softmax weights,
// estimation rows on the FP32 pipes; see attend_v5.cu).  What changes is the
// pipeline: attend_v5 gave every warp a private 2-stage ring and made it issue
// its own copies and decode its own chunk descriptors, so each warp handled
// one 16-row chunk every ~5,000 cycles (~580 instructions, mostly bookkeeping
// and copy issue) and the kernel was bound by that serial chain at ~5 TB/s
// (tools/tma_stream_probe.cu: the same staging pattern with no compute streams
// at 6.9-7.1 TB/s).  Here each CTA runs
//   * NP producer warps: walk the CTA's contiguous range of the flat chunk
//     list (producer p takes chunks p, p + NP, ...), prefetch each chunk's row
//     ids L chunks ahead (cp.async into a small per-producer ring), and fill a
//     CTA-wide ring of S stages: one TMA bulk copy per contiguous run of K / V
//     rows (the bf16 rows are stored swizzled, common.cuh swz_col, so unpadded
//     rows read conflict-free with ldmatrix), TMA gather4 of the estimation
//     rows' fp32 value sums (4 arbitrary rows per instruction, out-of-range
//     rows zero-filled) plus bulk copies of their logits and sizes;
//   * NC consumer warps: consumer c takes chunks c, c + NC, ..., waits on the
//     stage's full barrier, accumulates, releases the stage.
// Partials (M, D, num[d]) are flushed per (consumer, unit, kind) and folded
// by att6_merge_kernel (same LSE merge as att4_merge_kernel, with the
// consumer round-robin schedule).
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_mma.cuh"
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

__device__ __align__(128) unsigned char g_zero6[8192];
#ifdef ATT6_DEBUG  // hang / accounting diagnostics (experiment builds only)
}  // namespace wk
#include <cstdio>
namespace wk {
WK_DEVINL void dbg_wait(uint32_t bar, uint32_t phase, int tag, int i) {
  long long spins = 0;
  while (true) {
    uint32_t ok;
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
    if (ok) return;
    if (++spins == (1ll << 22)) {
      printf("att6 hang: block %d warp %d %s chunk %d phase %u\n", blockIdx.x, threadIdx.x >> 5, tag ? "full" : "empty", i, phase);
      asm volatile("trap;");
    }
  }
}
#endif
#ifdef ATT6_TIMING  // tools/att6_timing.py: per-warp cycles waiting vs working (experiment builds only)
__device__ long long g_att6_ts[148 * 16 * 4];
extern "C" int wk_att6_timing(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_att6_ts, sizeof(long long) * (size_t)n) == cudaSuccess ? 0 : -2;
}
#define A6_T(v) long long v = clock64()
#define A6_ADD(acc, t0) acc += clock64() - (t0)
#else
#define A6_T(v) do {} while (0)
#define A6_ADD(acc, t0) do {} while (0)
#endif

#ifdef WK_EXP_ACC_EXP  // accuracy experiment only (tools/exp_bench.py): full-precision exp
#define A6_EXP expf
#else
#define A6_EXP __expf
#endif

template <int D, int HS>
struct Att6Cfg {
#ifndef ATT6_CH
#define ATT6_CH 16  // 32-row chunks (8 stages) measured no faster
#endif
  static constexpr int CH = ATT6_CH;          // rows per chunk (producer / ring granularity)
  static constexpr int RG = 16;               // rows per consumer sub-chunk (mma K of p.v)
  static constexpr int KS = D / 16;           // q.k k-steps == p.v m-tiles
  static constexpr int NT = HS == 4 ? 2 : 3;  // q.k n-tiles (head x split columns)
  static constexpr int NL = HS == 4 ? 2 : 4;  // (row, head) logit slots per lane
  static constexpr int NH = HS == 4 ? 1 : 2;  // logit heads per lane
  static constexpr int NA = KS * 4;           // accumulator floats per lane
  static constexpr int ROWT = D * 2;          // bf16 K / V row bytes
  static constexpr int ROWV = D * 4;          // fp32 value-sum row bytes
  static constexpr int SB = 2 * CH * ROWT > CH * ROWV ? 2 * CH * ROWT : CH * ROWV;  // stage bytes
#ifndef ATT6_NP
#define ATT6_NP 4  // tuning experiments only (tools/att6_sweep.sh)
#endif
#ifndef ATT6_NC
#define ATT6_NC 8
#endif
  static constexpr int NP = ATT6_NP;          // producer warps
  static constexpr int NC = ATT6_NC;          // consumer warps
  static constexpr int WARPS = NP + NC;
#ifndef ATT6_L
#define ATT6_L 8
#endif
  static constexpr int L = ATT6_L;            // producer meta lookahead (chunks)
  // stage meta (producer -> consumers): tag int4 | (mask | key << 8) u16[CH] |
  // estimation logits f32[CH][8] | sizes f32[CH]
  static constexpr int SM_TAG = 0, SM_MK = 16, SM_EX = (16 + 2 * CH + 15) / 16 * 16, SM_ESZ = SM_EX + CH * 8 * 4;
  static constexpr int SM = ((SM_ESZ + 4 * CH) + 127) / 128 * 128;
  static constexpr int CS = 3 * 8 * RG * 2 + RG * HS * 4;  // consumer scratch: split weights | fp32 weights
  static constexpr int PR = L * (16 + 4 * CH);             // producer ring: desc int4 + CH row ids
  static constexpr int MAXU = 1024;
  static constexpr int FIXED = NC * CS + NP * PR + (MAXU + 1) * 4 + 64 + 128;
  static constexpr int S_FIT = (227 * 1024 - FIXED) / (SB + SM + 16);
#ifndef ATT6_SMAX
#define ATT6_SMAX 24
#endif
  // ring stages per CTA, a multiple of NC and of NP.  The stage barriers are
  // waited on by phase parity, which only tells the last two phases apart:
  // the consumer of chunk i must not reach stage i % S before chunk i - S's
  // phase completed, which holds when chunk i - S went to the same consumer
  // (S % NC == 0); likewise the producer of chunk i must already have waited
  // for the release of chunk i - 2S (S % NP == 0).  Other S let a fast
  // consumer / producer pass a barrier one phase early (the CH = 32 faults and
  // NC = 10 hangs of the tuning builds).
  static constexpr int gcd(int a, int b) { return b == 0 ? a : gcd(b, a % b); }
  static constexpr int LCM_PC = NC / gcd(NC, NP) * NP;
  static constexpr int S_CAP = S_FIT > ATT6_SMAX ? ATT6_SMAX : S_FIT;
  static constexpr int S = S_CAP / LCM_PC * LCM_PC;
  static_assert(S >= LCM_PC && S % NC == 0 && S % NP == 0, "ring stages must be a multiple of NC and NP");
  static constexpr size_t SMEM = (size_t)S * (SB + SM + 16) + FIXED;
};

template <int RG, bool FULL, bool ROWS>
WK_DEVINL void att6_counts(const SteadyView& st, const StepView& sv, const int32_t* n_store, int u, int& c0,
                           int& c1, int& c2) {
  c0 = (st.n[u] + RG - 1) / RG;
  if (FULL) {
    c1 = (n_store[u] + RG - 1) / RG;
    c2 = 0;
  } else {
    c1 = ROWS ? (sv.cnt[u * 4 + 1] + RG - 1) / RG : sv.cnt[u * 4 + 3];
    c2 = (sv.cnt[u * 4 + 2] + RG - 1) / RG;
  }
#ifdef ATT6_SKIP  // timing experiments only: 1 = no estimation chunks, 2 = no exact chunks
  if (ATT6_SKIP == 1) c2 = 0;
  if (ATT6_SKIP == 2) { c0 = 0; c1 = 0; }
#endif
}

template <int D, int HS, bool FULL, bool OFF, bool ROWS>
__global__ void __launch_bounds__(Att6Cfg<D, HS>::WARPS * 32, 1)
    attend_v6_kernel(IndexView ix, SteadyView st, StepView sv, AttnParams p, const int32_t* __restrict__ n_store,
                     int U, const __grid_constant__ CUtensorMap tm_vs) {
  using CF = Att6Cfg<D, HS>;
  constexpr int CH = CF::CH, RG = CF::RG, KS = CF::KS, NT = CF::NT, NL = CF::NL, NH = CF::NH, NA = CF::NA;
  constexpr int ROWT = CF::ROWT, ROWV = CF::ROWV, SB = CF::SB, SMT = CF::SM, S = CF::S, NP = CF::NP,
                NC = CF::NC, L = CF::L;
  constexpr int DL = D / 16;  // estimation mode: dims per lane
  pdl_wait();
  const int G = p.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(128) unsigned char a6s[];
  unsigned char* sdata = a6s;                                   // [S][SB]
  unsigned char* smeta = a6s + (size_t)S * SB;                  // [S][SMT]
  uint64_t* fullb = reinterpret_cast<uint64_t*>(smeta + (size_t)S * SMT);  // [S]
  uint64_t* emptyb = fullb + S;                                 // [S]
  unsigned char* cscr = reinterpret_cast<unsigned char*>(emptyb + S);  // [NC][CS]
  unsigned char* pring = cscr + NC * CF::CS;                    // [NP][L][16 + 64]
  int* woff = reinterpret_cast<int*>(pring + NP * CF::PR);      // [MAXU + 1] (+ 16 scratch)
  const uint32_t sdata_s = smem_u32(sdata), smeta_s = smem_u32(smeta);
  const uint32_t full_s = smem_u32(fullb), empty_s = smem_u32(emptyb);

  // ---- chunk prefix over units (every CTA; U <= MAXU) ----
  {
    int carry = 0;
    for (int base = 0; base < U; base += blockDim.x) {
      const int u = base + threadIdx.x;
      int c = 0;
      if (u < U) {
        int c0, c1, c2;
        att6_counts<CH, FULL, ROWS>(st, sv, n_store, u, c0, c1, c2);
        c = c0 + c1 + c2;
      }
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int* ws = woff + CF::MAXU + 1;
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
    if (threadIdx.x == 0) {
      woff[U] = carry;
      for (int i = 0; i < S; i++) {
        mbar_init(fullb + i, 1);
        mbar_init(emptyb + i, 1);
      }
      fence_mbar_init();
    }
    __syncthreads();
  }
  const long long Ntot = woff[U];
  if (blockIdx.x == 0 && sv.woff)
    for (int i = threadIdx.x; i <= U; i += blockDim.x) sv.woff[i] = woff[i];
  const long long ca = Ntot * blockIdx.x / gridDim.x, cb = Ntot * (blockIdx.x + 1) / gridDim.x;
  const int ncta = (int)(cb - ca);

  if (warp < NP) {
    // =========================== producer ===========================
    const int pw = warp;
#ifdef ATT6_TIMING
    long long tw_acc = 0;
    const long long tp0 = clock64();
#endif
    unsigned char* ring = pring + pw * CF::PR;
    int4* rdesc = reinterpret_cast<int4*>(ring);            // [L] (u, kind + 1 | n << 8, a, lc)
    int* rids = reinterpret_cast<int*>(ring + L * 16);      // [L][CH]
    const uint32_t rids_s = smem_u32(rids);
    // cursor over units (chunk indices visited in increasing order); the unit's
    // sizes stay in registers (no global load per chunk on the producer's chain)
    int iu = 0, ic0 = 0, ic1 = 0, ic2 = 0, in_st = 0, in_x = 0, in_e = 0;
    auto unit_sizes = [&]() {
      att6_counts<CH, FULL, ROWS>(st, sv, n_store, iu, ic0, ic1, ic2);
      in_st = st.n[iu];
      in_x = FULL ? n_store[iu] : (ROWS ? sv.cnt[iu * 4 + 1] : 0);
      in_e = FULL ? 0 : sv.cnt[iu * 4 + 2];
    };
    {
      int lo = 0, hi = U - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (woff[mid] <= ca) lo = mid; else hi = mid - 1;
      }
      iu = lo;
      unit_sizes();
    }
    const int allmask = (1 << G) - 1;
    auto prefetch = [&](int k) {
      const int i = pw + NP * k;
      if (i < ncta) {
        const long long ci = ca + i;
        while (ci >= woff[iu + 1]) {
          iu++;
          unit_sizes();
        }
        const int u = iu;
        int lc = (int)(ci - woff[u]);
        int kind, n, a = 0;
        if (lc < ic0) {
          kind = 0;
          a = lc * CH;
          n = min(CH, in_st - a);
        } else if (lc < ic0 + ic1) {
          kind = 1;
          lc -= ic0;
          if (FULL) {
            a = lc * CH;
            n = min(CH, in_x - a);
          } else if (ROWS) {
            a = lc * CH;
            n = min(CH, in_x - a);
            if (lane < n) cp_async4(rids_s + ((k % L) * CH + lane) * 4, sv.rtok_row + (size_t)u * sv.rt_cap + a + lane);
          } else {  // offload piece (row, n | mask << 8 | flags << 16, cluster, first token)
            n = 0;    // from the piece
            if (lane == 0)
              cp_async16_ca(rids_s + (k % L) * CH * 4, reinterpret_cast<const int4*>(sv.pieces) + (size_t)u * sv.pc_cap + lc);
          }
        } else {
          kind = 2;
          lc -= ic0 + ic1;
          a = lc * CH;
          n = min(CH, in_e - a);
          if (lane < n) cp_async4(rids_s + ((k % L) * CH + lane) * 4, sv.eu_ids + (size_t)u * sv.eu_cap + a + lane);
        }
        if (lane == 0) rdesc[k % L] = make_int4(u, (kind + 1) | (n << 8), a, lc);
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int k = 0; k < L; k++) prefetch(k);
#pragma unroll 1
    for (int k = 0; pw + NP * k < ncta; k++) {
      const int i = pw + NP * k, s = i % S, slot = k % L;
      cp_async_wait<L - 1>();
      __syncwarp();
      const int4 dsc = rdesc[slot];
      const int u = dsc.x, kind = (dsc.y & 0xff) - 1;
      int n = (dsc.y >> 8) & 0xff;
#ifdef ATT6_TIMING
      const long long tw0 = clock64();
#endif
#ifdef ATT6_DEBUG
      if (i >= S) dbg_wait(empty_s + s * 8, (uint32_t)(((i / S) - 1) & 1), 0, i);
#else
      if (i >= S) mbar_wait_s(empty_s + s * 8, (uint32_t)(((i / S) - 1) & 1));
#endif
#ifdef ATT6_TIMING
      tw_acc += clock64() - tw0;
#endif
      const uint32_t stg = sdata_s + s * SB, bar = full_s + s * 8;
      unsigned char* meta = smeta + (size_t)s * SMT;
      int wt_z = 0, wt_w = 0;
      if (kind < 2) {
        int row, mk;
        const unsigned char* bk;
        const unsigned char* bv;
        const int j = lane;  // chunk row (CH == 32) / lanes >= n: unused
        if (kind == 0) {
          row = dsc.z + j;
          mk = allmask;
          bk = (const unsigned char*)st.k + (size_t)u * st.t_cap * ROWT;
          bv = (const unsigned char*)st.v + (size_t)u * st.t_cap * ROWT;
        } else if (FULL) {
          row = dsc.z + j;
          mk = allmask;
          bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
          bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
        } else if (ROWS) {
          const int w = rids[slot * CH + (j & (CH - 1))];
          row = w & 0xffffff;
          mk = (int)((unsigned)w >> 24);
          bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
          bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
        } else {
          const int4 pc = reinterpret_cast<const int4*>(rids)[slot * CH / 4];
          n = pc.y & 0xff;
          row = pc.x + j;
          mk = (pc.y >> 8) & 0xff;
          const int flags = (pc.y >> 16) & 3;
          if (flags & 1) {
            bk = (const unsigned char*)sv.arena_k + (size_t)u * sv.arena_rows * ROWT;
            bv = (const unsigned char*)sv.arena_v + (size_t)u * sv.arena_rows * ROWT;
          } else {
            bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
            bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
          }
          if (flags & 2) { wt_z = pc.z; wt_w = (pc.w & 0xffffff) | (int)0x80000000; }
        }
        const bool live = lane < n;
        // meta first (generic stores), then the barrier's expect_tx, then the copies
        if (lane < CH)
          reinterpret_cast<unsigned short*>(meta + CF::SM_MK)[lane] =
              (unsigned short)(live ? (mk | ((row & 7) << 8)) : ((lane & 7) << 8));
        if (lane == 0) *reinterpret_cast<int4*>(meta + CF::SM_TAG) = make_int4(u, (kind + 1) | (n << 8), wt_z, wt_w);
        const int prev = __shfl_up_sync(0xffffffffu, row, 1);
        const bool start = live && (lane == 0 || row != prev + 1);
        const unsigned starts = __ballot_sync(0xffffffffu, start);
        __syncwarp();
        if (lane == 0) mbar_expect_s(bar, (uint32_t)((n + CH) * ROWT));
        __syncwarp();
#ifdef ATT6_DEBUG
        {
          int lsum = 0;
          if (start) { const unsigned later = starts & ~((2u << lane) - 1u); lsum = (later ? __ffs(later) - 1 : n) - lane; }
          for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
          if (lane == 0 && (lsum != n || n <= 0 || n > CH))
            printf("att6 runs: block %d chunk %d kind %d n %d sum %d\n", blockIdx.x, i, kind, n, lsum);
        }
#endif
        if (start) {
          const unsigned later = starts & ~((2u << lane) - 1u);
          const int len = (later ? __ffs(later) - 1 : n) - lane;
          bulk_g2s_s(stg + lane * ROWT, bk + (size_t)row * ROWT, (uint32_t)(len * ROWT), bar);
          bulk_g2s_s(stg + CH * ROWT + lane * ROWT, bv + (size_t)row * ROWT, (uint32_t)(len * ROWT), bar);
        }
        // V rows >= n zero-filled (a zero weight never meets a stale non-finite value)
        if (lane == 0 && n < CH) bulk_g2s_s(stg + CH * ROWT + n * ROWT, g_zero6, (uint32_t)((CH - n) * ROWT), bar);
      } else {
        if (lane == 0) *reinterpret_cast<int4*>(meta + CF::SM_TAG) = make_int4(u, (kind + 1) | (n << 8), 0, 0);
        __syncwarp();
        if (lane == 0) {
          const uint32_t exb = (uint32_t)(CH * G * 4);
          mbar_expect_s(bar, (uint32_t)(CH * ROWV) + exb + 4u * CH);
          const int4* id4 = reinterpret_cast<const int4*>(rids + slot * CH);
          const int rb = u * (int)ix.m_cap;
#pragma unroll
          for (int g4 = 0; g4 < CH / 4; g4++) {
            const int4 c = id4[g4];
            const int b = 4 * g4;
            tma_gather4(stg + b * ROWV, &tm_vs, 0, b < n ? rb + c.x : -1, b + 1 < n ? rb + c.y : -1,
                        b + 2 < n ? rb + c.z : -1, b + 3 < n ? rb + c.w : -1, bar);
          }
          // logits [16][G] and sizes [16] of the rows (rows >= n: ignored by the consumers)
          bulk_g2s_s(smeta_s + s * SMT + CF::SM_EX, sv.eu_x + ((size_t)u * sv.eu_cap + dsc.z) * G, exb, bar);
          bulk_g2s_s(smeta_s + s * SMT + CF::SM_ESZ, sv.eu_sz + (size_t)u * sv.eu_cap + dsc.z, 4u * CH, bar);
        }
      }
      __syncwarp();  // this ring slot is consumed: reuse it for chunk k + L
      prefetch(k + L);
    }
    cp_async_wait<0>();
#ifdef ATT6_TIMING
    if (lane == 0 && blockIdx.x < 148) {
      g_att6_ts[(blockIdx.x * 16 + warp) * 4 + 0] = tw_acc;
      g_att6_ts[(blockIdx.x * 16 + warp) * 4 + 1] = clock64() - tp0;
    }
#endif
    return;
  }

  // =========================== consumers ===========================
  const int cw = warp - NP;
  const int g8 = lane >> 2, t4 = lane & 3;      // mma fragment coordinates
  const int half = lane >> 4, sub = lane & 15;  // estimation mode coordinates
  unsigned short* pb = reinterpret_cast<unsigned short*>(cscr + cw * CF::CS);  // [3][8][RG] bf16
  float* pe = reinterpret_cast<float*>(pb + 3 * 8 * RG);                      // [RG][HS]
  const uint32_t pb_s = smem_u32(pb);
  for (int i = lane; i < 3 * 8 * RG / 2; i += 32) reinterpret_cast<uint32_t*>(pb)[i] = 0u;
  __syncwarp();
  const int gw = blockIdx.x * NC + cw;
  const float isd = p.inv_sqrt_d;
#ifdef ATT6_TIMING
  long long tw_acc = 0;
  const long long tp0 = clock64();
#endif
  auto slot_row = [&](int l) { return g8 + 8 * (HS == 4 ? l : (l >> 1)); };
  auto slot_head = [&](int l) { return HS == 4 ? t4 : 2 * t4 + (l & 1); };

  uint32_t qb[KS][NT][2];
  int qu = -1;
  auto load_q = [&](int u) {
    const int hq = HS == 4 ? (g8 >> 1) : g8;
    int sp[NT];
#pragma unroll
    for (int nt = 0; nt < NT; nt++) {
      sp[nt] = HS == 4 ? (nt == 0 ? (g8 & 1) : ((g8 & 1) ? -1 : 2)) : nt;
      if (hq >= G) sp[nt] = -1;
    }
    const float* qrow = sv.q + ((size_t)u * G + (hq < G ? hq : 0)) * D;
#pragma unroll
    for (int kk = 0; kk < KS; kk++) {
#pragma unroll
      for (int hf = 0; hf < 2; hf++) {
        const float2 qv = *reinterpret_cast<const float2*>(qrow + kk * 16 + 2 * t4 + 8 * hf);
        uint32_t s0[3], s1[3];
        split3(qv.x * isd, s0[0], s0[1], s0[2]);
        split3(qv.y * isd, s1[0], s1[1], s1[2]);
#pragma unroll
        for (int nt = 0; nt < NT; nt++) {
          uint32_t w = 0;
#pragma unroll
          for (int s = 0; s < 3; s++)
            if (sp[nt] == s) w = s0[s] | (s1[s] << 16);
          qb[kk][nt][hf] = w;
        }
      }
    }
    qu = u;
  };

  float mo[NH], dl[NH], acc[NA];
  auto reset = [&]() {
#pragma unroll
    for (int i = 0; i < NH; i++) { mo[i] = -INFINITY; dl[i] = 0.f; }
#pragma unroll
    for (int i = 0; i < NA; i++) acc[i] = 0.f;
  };
  reset();
  int cu = -1, ck = -1;
  auto dim_e = [&](int j) { return j < 4 ? sub * 4 + j : 64 + sub * 4 + (j - 4); };
  auto flush = [&]() {
    if (cu < 0) return;
    float ds[NH];
#pragma unroll
    for (int i = 0; i < NH; i++) {
      float v = dl[i];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      ds[i] = v;
    }
    // record key gw + NC * u = NC * (CTA + u) + consumer: unique, since a
    // CTA's units start at or after the previous CTA's last unit (a consumer
    // takes chunks of several units round-robin, so gw + u would collide)
    float* base = sv.part + ((size_t)(gw + NC * cu) * 3 + ck) * (size_t)G * (4 + D);
    if (g8 == 0) {
#pragma unroll
      for (int i = 0; i < NH; i++) {
        const int h = HS == 4 ? t4 : 2 * t4 + i;
        if (h < G) { base[(size_t)h * (4 + D)] = mo[i]; base[(size_t)h * (4 + D) + 1] = ds[i]; }
      }
    }
    if (ck < 2) {
#pragma unroll
      for (int mt = 0; mt < KS; mt++)
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int h = 2 * t4 + (r & 1), dim = mt * 16 + g8 + 8 * (r >> 1);
          if (h < G) base[(size_t)h * (4 + D) + 4 + dim] = acc[mt * 4 + r];
        }
    } else {
      if (HS == 4) {
#pragma unroll
        for (int i = 0; i < NA; i++) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
      }
      if (HS == 8 || half == 0) {
#pragma unroll
        for (int h4 = 0; h4 < 4; h4++) {
          const int h = (HS == 8 ? 4 * half : 0) + h4;
          if (h < G) {
            float* dst = base + (size_t)h * (4 + D) + 4;
#pragma unroll
            for (int j = 0; j < DL; j += 4)
              *reinterpret_cast<float4*>(dst + dim_e(j)) =
                  make_float4(acc[h4 * DL + j], acc[h4 * DL + j + 1], acc[h4 * DL + j + 2], acc[h4 * DL + j + 3]);
          }
        }
      }
    }
    reset();
  };
  // lazily rescaled online softmax (attend_v5)
  auto softmax = [&](const float (&x)[NL], bool est_mode) {
    bool up = false;
#pragma unroll
    for (int l = 0; l < NL; l++) up |= x[l] > mo[HS == 4 ? 0 : (l & 1)] + 10.f;
    if (__any_sync(0xffffffffu, up)) {
      float al[NH];
#pragma unroll
      for (int i = 0; i < NH; i++) {
        float mx = HS == 4 ? fmaxf(x[0], x[1]) : fmaxf(x[i], x[i + 2 < NL ? i + 2 : i]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        al[i] = 1.f;
        if (mx > mo[i]) {
          al[i] = mo[i] == -INFINITY ? 0.f : A6_EXP(mo[i] - mx);
          mo[i] = mx;
        }
        dl[i] *= al[i];
      }
      if (!est_mode) {
        float a0, a1;
        if (HS == 4) {
          a0 = __shfl_sync(0xffffffffu, al[0], (2 * t4) & 3);
          a1 = __shfl_sync(0xffffffffu, al[0], (2 * t4 + 1) & 3);
        } else {
          a0 = __shfl_sync(0xffffffffu, al[0], t4);
          a1 = __shfl_sync(0xffffffffu, al[NH - 1], t4);
        }
#pragma unroll
        for (int i = 0; i < NA; i++) acc[i] *= (i & 1) ? a1 : a0;
      } else {
#pragma unroll
        for (int h4 = 0; h4 < 4; h4++) {
          float a;
          if (HS == 4) {
            a = __shfl_sync(0xffffffffu, al[0], h4);
          } else {
            const float a_e = __shfl_sync(0xffffffffu, al[0], 2 * half + (h4 >> 1));
            const float a_o = __shfl_sync(0xffffffffu, al[NH - 1], 2 * half + (h4 >> 1));
            a = (h4 & 1) ? a_o : a_e;
          }
#pragma unroll
          for (int j = 0; j < DL; j++) acc[h4 * DL + j] *= a;
        }
      }
    }
  };

  // one 16-row sub-chunk (rows r0 .. r0 + 15 of the stage's chunk)
  auto compute = [&](int s, int kind, int n, int r0) {
    const uint32_t stg = sdata_s + s * SB;
    const unsigned char* meta = smeta + (size_t)s * SMT;
    const unsigned short* mk16 = reinterpret_cast<const unsigned short*>(meta + CF::SM_MK) + r0;
    n -= r0;
    float x[NL], pw[NL];
    if (kind < 2) {
      // q.k: S^T = K . Qs^T (two accumulator sets halve the dependent MMA chain)
      float c[NT][4], c2[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; nt++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[nt][i] = c2[nt][i] = 0.f;
      const int jk = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int kbk = ((mk16[jk] >> 8) & 7) ^ (lane >> 4);
      const uint32_t aK = stg + (r0 + jk) * ROWT;
      uint32_t ak[KS][4];
#pragma unroll
      for (int kk = 0; kk < KS; kk++)
        ldsm_x4(aK + (((2 * kk) ^ kbk) << 4), ak[kk][0], ak[kk][1], ak[kk][2], ak[kk][3]);
#pragma unroll
      for (int kk = 0; kk < KS; kk++)
#pragma unroll
        for (int nt = 0; nt < NT; nt++)
          mma_bf16((kk & 1) ? c2[nt] : c[nt], ak[kk][0], ak[kk][1], ak[kk][2], ak[kk][3], qb[kk][nt][0],
                   qb[kk][nt][1]);
#pragma unroll
      for (int nt = 0; nt < NT; nt++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[nt][i] += c2[nt][i];
      const int mk_lo = mk16[g8] & 0xff, mk_hi = mk16[g8 + 8] & 0xff;
#pragma unroll
      for (int l = 0; l < NL; l++) {
        float sc;
        if (HS == 4) {
          const int ci = 2 * l;
          sc = (c[0][ci] + c[0][ci + 1]) + c[1][ci];
        } else {
          const int ci = 2 * (l >> 1) + (l & 1);
          sc = (c[0][ci] + c[1][ci]) + c[2][ci];
        }
        const int mk = (HS == 4 ? l : (l >> 1)) ? mk_hi : mk_lo;
        x[l] = ((mk >> slot_head(l)) & 1) ? sc : -INFINITY;
      }
      softmax(x, false);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int i = HS == 4 ? 0 : (l & 1);
        pw[l] = x[l] == -INFINITY ? 0.f : A6_EXP(x[l] - mo[i]);
        dl[i] += pw[l];
        uint32_t sh, sm, sl;
        split3(pw[l], sh, sm, sl);
        const int idx = slot_head(l) * RG + slot_row(l);
        pb[idx] = (unsigned short)sh;
        pb[8 * RG + idx] = (unsigned short)sm;
        pb[16 * RG + idx] = (unsigned short)sl;
      }
      __syncwarp();
      // p.v: O^T += V^T . P_s, all V fragments first, then split-major MMAs
      uint32_t b[3][2];
      {
        const int mi = lane >> 3, r = lane & 7;
        ldsm_x4(pb_s + (((mi >> 1) * 8 + r) * RG + (mi & 1) * 8) * 2, b[0][0], b[0][1], b[1][0], b[1][1]);
        ldsm_x2(pb_s + ((16 + r) * RG + (mi & 1) * 8) * 2, b[2][0], b[2][1]);
      }
      const int jv = (lane & 7) + 8 * (lane >> 4);
      const int kbv = ((mk16[jv] >> 8) & 7) ^ ((lane >> 3) & 1);
      const uint32_t aV = stg + CH * ROWT + (r0 + jv) * ROWT;
      uint32_t av[KS][4];
#pragma unroll
      for (int mt = 0; mt < KS; mt++)
        ldsm_x4_t(aV + (((2 * mt) ^ kbv) << 4), av[mt][0], av[mt][1], av[mt][2], av[mt][3]);
      // the chunk's p.v in a fresh accumulator, added to the running one by
      // IEEE fp32 adds: the tensor-core accumulate truncates, which biases a
      // large running sum fed many small chunk terms (rank-ordered pieces)
#pragma unroll
      for (int mt = 0; mt < KS; mt++) {
        float cc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int sp = 2; sp >= 0; sp--)
          mma_bf16(cc, av[mt][0], av[mt][1], av[mt][2], av[mt][3], b[sp][0], b[sp][1]);
#pragma unroll
        for (int i = 0; i < 4; i++) acc[mt * 4 + i] += cc[i];
      }
    } else {
      // estimation rows: fp32 value sums on the FP32 pipes
      const float* ex = reinterpret_cast<const float*>(meta + CF::SM_EX) + r0 * G;
      const float* esz = reinterpret_cast<const float*>(meta + CF::SM_ESZ) + r0;
      float wz[NL];
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int r = slot_row(l), h = slot_head(l);
        const bool ok = r < n && h < G;
        x[l] = ok ? ex[r * G + h] : -INFINITY;
        wz[l] = ok ? esz[r] : 0.f;
      }
      softmax(x, true);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int i = HS == 4 ? 0 : (l & 1);
        pw[l] = x[l] == -INFINITY ? 0.f : A6_EXP(x[l] - mo[i]);
        dl[i] = fmaf(pw[l], wz[l], dl[i]);
        pe[slot_row(l) * HS + slot_head(l)] = pw[l];
      }
      __syncwarp();
      const unsigned char* stage = sdata + (size_t)s * SB + (size_t)r0 * ROWV;
      constexpr int RSTEP = HS == 4 ? 2 : 1;
#pragma unroll 4
      for (int j = (HS == 4 ? half : 0); j < RG; j += RSTEP) {
        const float* row = reinterpret_cast<const float*>(stage + j * ROWV);
        float2 v2[DL / 2];
        {
          const float4 lo = *reinterpret_cast<const float4*>(row + sub * 4);
          v2[0] = make_float2(lo.x, lo.y);
          v2[1] = make_float2(lo.z, lo.w);
          if (DL == 8) {
            const float4 hi = *reinterpret_cast<const float4*>(row + 64 + sub * 4);
            v2[2 % (DL / 2)] = make_float2(hi.x, hi.y);
            v2[3 % (DL / 2)] = make_float2(hi.z, hi.w);
          }
        }
        const float4 p4 = *reinterpret_cast<const float4*>(pe + j * HS + (HS == 8 ? 4 * half : 0));
        const float pj[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int h4 = 0; h4 < 4; h4++) {
          const float2 p2 = make_float2(pj[h4], pj[h4]);
#pragma unroll
          for (int k = 0; k < DL / 2; k++) {
            float2 a = make_float2(acc[h4 * DL + 2 * k], acc[h4 * DL + 2 * k + 1]);
            a = __ffma2_rn(p2, v2[k], a);
            acc[h4 * DL + 2 * k] = a.x;
            acc[h4 * DL + 2 * k + 1] = a.y;
          }
        }
      }
    }
  };

#pragma unroll 1
  for (int i = cw; i < ncta; i += NC) {
    const int s = i % S;
#ifdef ATT6_TIMING
    const long long tw0 = clock64();
#endif
#ifdef ATT6_DEBUG
    dbg_wait(full_s + s * 8, (uint32_t)((i / S) & 1), 1, i);
#else
    mbar_wait_s(full_s + s * 8, (uint32_t)((i / S) & 1));
#endif
#ifdef ATT6_TIMING
    tw_acc += clock64() - tw0;
#endif
    const int4 tg = *reinterpret_cast<const int4*>(smeta + (size_t)s * SMT + CF::SM_TAG);
    const int kind = (tg.y & 0xff) - 1, n = (tg.y >> 8) & 0xff;
    if (tg.x != cu || kind != ck) {
      flush();
      cu = tg.x;
      ck = kind;
      if (qu != cu) load_q(cu);
    }
    for (int r0 = 0; r0 < n; r0 += RG) {
      if (r0) __syncwarp();  // the split / fp32 weight scratch is rewritten
      compute(s, kind, n, r0);
    }
    if (OFF && tg.w < 0) {
      // admitted offload miss: write its rows through into the new slots (re-keyed)
      const int cl = tg.z, j0 = tg.w & 0xffffff;
      const int bt = sv.block_tokens;
      const int32_t* sl = sv.slot_ids + (size_t)cu * sv.slot_cap;
      const int so = __ldg(sv.slot_off + (size_t)cu * ix.m_cap + cl);
      const unsigned char* stage = sdata + (size_t)s * SB;
      const unsigned short* mk16 = reinterpret_cast<const unsigned short*>(smeta + (size_t)s * SMT + CF::SM_MK);
      for (int r = half; r < n; r += 2) {
        const int tok = j0 + r;
        const size_t ar = (size_t)__ldcg(sl + so + tok / bt) * bt + tok % bt;
        const size_t arow = (size_t)cu * sv.arena_rows + ar;
        const int ks = (mk16[r] >> 8) & 7, ka = (int)(ar & 7);
        if (sub < ROWT / 16) {
          *reinterpret_cast<uint4*>((unsigned char*)sv.arena_k + arow * ROWT + ((sub ^ ka) << 4)) =
              *reinterpret_cast<const uint4*>(stage + r * ROWT + ((sub ^ ks) << 4));
          *reinterpret_cast<uint4*>((unsigned char*)sv.arena_v + arow * ROWT + ((sub ^ ka) << 4)) =
              *reinterpret_cast<const uint4*>(stage + CH * ROWT + r * ROWT + ((sub ^ ks) << 4));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(empty_s + s * 8);
  }
  pdl_trigger<4>();
  flush();
#ifdef ATT6_TIMING
  if (lane == 0 && blockIdx.x < 148) {
    g_att6_ts[(blockIdx.x * 16 + warp) * 4 + 0] = tw_acc;
    g_att6_ts[(blockIdx.x * 16 + warp) * 4 + 1] = clock64() - tp0;
  }
#endif
}

// ---------------------------------------------------------------------------
// merge: one CTA (4 warps) per (unit, head); the partial records of a (unit,
// kind) are those of the consumer warps that took at least one of its chunks
// (CTA ranges are contiguous, consumers round-robin within a CTA)
// ---------------------------------------------------------------------------
template <bool FULL, int DL>
__global__ void __launch_bounds__(128, 4) att6_merge_kernel(SteadyView st, StepView sv, AttnParams p,
                                                          const int32_t* __restrict__ n_store, int U, int P,
                                                          int NC, int rows_mode, int RG) {
  pdl_wait();
  pdl_trigger<8>();
#ifdef WK_EXP_MERGE_EMPTY  // timing experiment only (tools/exp_bench.py): the merge launch's fixed cost
  return;
#endif
  const int G = p.G, d = p.d, D2 = 4 + d;
  const int u = blockIdx.x / G, g = blockIdx.x % G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the tail partial (m, D, eq2 m, eq2 D) loaded up front, off the merge's chain
  const float4 tl4 = (!FULL && sv.tail) ? __ldcg(reinterpret_cast<const float4*>(sv.tail + ((size_t)u * G + g) * 4))
                                        : make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
  __shared__ float s_m[3][4];
  __shared__ float s_d[3][4];
  __shared__ float s_n[3][4][128];
  const long long N = sv.woff[U];
  int c0, c1, c2;
  {
    c0 = (st.n[u] + RG - 1) / RG;
    if (FULL) { c1 = (n_store[u] + RG - 1) / RG; c2 = 0; }
    else {
      c1 = rows_mode ? (sv.cnt[u * 4 + 1] + RG - 1) / RG : sv.cnt[u * 4 + 3];
      c2 = (sv.cnt[u * 4 + 2] + RG - 1) / RG;
    }
  }
  const long long ub = sv.woff[u];
  const long long kb[4] = {ub, ub + c0, ub + c0 + c1, ub + c0 + c1 + c2};
  // the CTA-range arithmetic in 32 bits when (N + 1) P fits (every realistic
  // size; the 64-bit divisions dominated this kernel's instruction count)
  const bool i32 = (N + 1) * (long long)(P + 1) < (1ll << 31);
  const int N32 = (int)N;
  auto cta_of = [&](long long c) {
    return i32 ? (((int)c + 1) * P + N32 - 1) / N32 - 1 : (int)(((c + 1) * P + N - 1) / N - 1);
  };
  int nb[3], b0[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    nb[k] = 0;
    b0[k] = 0;
    if (kb[k + 1] > kb[k]) {
      b0[k] = cta_of(kb[k]);
      nb[k] = cta_of(kb[k + 1] - 1) - b0[k] + 1;
    }
  }
  const int S = (nb[0] + nb[1] + nb[2]) * NC;
  // item i -> (kind, consumer warp id); live iff that consumer took a chunk of the kind's range
  auto item = [&](int i, int& k, int& gwi) {
    int b = i / NC;
    const int c = i % NC;
    k = b < nb[0] ? 0 : (b < nb[0] + nb[1] ? 1 : 2);
    b = b0[k] + b - (k == 0 ? 0 : (k == 1 ? nb[0] : nb[0] + nb[1]));
    gwi = b * NC + c;
    if (i32) {
      const int A = N32 * b / P, B = N32 * (b + 1) / P;
      const int x = (int)(kb[k] > A ? kb[k] : A) - A, y = (int)(kb[k + 1] < B ? kb[k + 1] : B) - A;
      const int j0 = x + ((c - x) % NC + NC) % NC;
      return j0 < y;
    }
    const long long A = N * b / P, B = N * (b + 1) / P;
    const long long x = (kb[k] > A ? kb[k] : A) - A, y = (kb[k + 1] < B ? kb[k + 1] : B) - A;
    const long long j0 = x + ((c - x) % NC + NC) % NC;
    return j0 < y;
  };
  auto rec = [&](int k, int gwi) { return sv.part + (((size_t)(gwi + NC * u) * 3 + k) * G + g) * (size_t)D2; };
  const int Sw = (S - warp + 3) / 4;
  float mw[3] = {-INFINITY, -INFINITY, -INFINITY}, dw3[3] = {0.f, 0.f, 0.f};
  float nacc[3][DL];
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int j = 0; j < DL; j++) nacc[k][j] = 0.f;
  for (int i0 = 0; i0 < Sw; i0 += 32) {
    const int nw = min(32, Sw - i0);
    float M = -INFINITY, Dw = 0.f;
    int kl = 0, gl = 0;
    bool lv = false;
    if (lane < nw) {
      lv = item(warp + 4 * (i0 + lane), kl, gl);
      if (lv) {
        const float* r = rec(kl, gl);
        Dw = __ldcg(r + 1);
        M = Dw > 0.f ? __ldcg(r) : -INFINITY;
      }
    }
    constexpr int PF = 8;
    auto vload = [&](int j, float (&v)[DL]) {
      const int kj = __shfl_sync(0xffffffffu, kl, j);
      const int gj = __shfl_sync(0xffffffffu, gl, j);
      const bool lj = __shfl_sync(0xffffffffu, (int)lv, j) != 0;
      const float* src = rec(kj, gj) + 4 + lane * DL;
      if (!lj) {
#pragma unroll
        for (int jj = 0; jj < DL; jj++) v[jj] = 0.f;
      } else if (DL == 4) {
        const float4 q4 = __ldcg(reinterpret_cast<const float4*>(src));
        v[0] = q4.x; v[1] = q4.y; v[2 % DL] = q4.z; v[3 % DL] = q4.w;
      } else {
        const float2 q2 = __ldcg(reinterpret_cast<const float2*>(src));
        v[0] = q2.x; v[1 % DL] = q2.y;
      }
    };
    // the first batch's value loads are in flight with the (M, D) loads;
    // batches of PF items, folds in item order
    float pv[PF][DL];
#pragma unroll
    for (int j = 0; j < PF; j++)
      if (j < nw) vload(j, pv[j]);
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const float bm = warp_max(kl == k ? M : -INFINITY);
      if (bm > mw[k]) {
        const float alpha = mw[k] == -INFINITY ? 0.f : expf(mw[k] - bm);
        dw3[k] *= alpha;
#pragma unroll
        for (int j = 0; j < DL; j++) nacc[k][j] *= alpha;
        mw[k] = bm;
      }
    }
    const float mk = kl == 0 ? mw[0] : (kl == 1 ? mw[1] : mw[2]);
    const float sc = Dw > 0.f ? A6_EXP(M - mk) : 0.f;
    if (kl == 0) dw3[0] += Dw * sc; else if (kl == 1) dw3[1] += Dw * sc; else dw3[2] += Dw * sc;
    auto fold = [&](int j, const float (&v)[DL]) {
      const float swt = __shfl_sync(0xffffffffu, sc, j);
      const int kj = __shfl_sync(0xffffffffu, kl, j);
      // dead or empty records (may hold stale bits): weight 0 selects them out
      // kj is warp-uniform: one accumulator row per item
#pragma unroll
      for (int k = 0; k < 3; k++)
        if (kj == k) {
#pragma unroll
          for (int jj = 0; jj < DL; jj++) nacc[k][jj] += swt != 0.f ? v[jj] * swt : 0.f;
        }
    };
    for (int j0 = 0; j0 < nw; j0 += PF) {
      if (j0 > 0) {
#pragma unroll
        for (int j = 0; j < PF; j++)
          if (j0 + j < nw) vload(j0 + j, pv[j]);
      }
#pragma unroll
      for (int j = 0; j < PF; j++)
        if (j0 + j < nw) fold(j0 + j, pv[j]);
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
  const float tl[4] = {tl4.x, tl4.y, tl4.z, tl4.w};
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

template <int D, int HS>
size_t attend_v6_smem() { return Att6Cfg<D, HS>::SMEM; }
template <int D, int HS>
int attend_v6_warps() { return Att6Cfg<D, HS>::WARPS; }
template <int D, int HS>
int attend_v6_consumers() { return Att6Cfg<D, HS>::NC; }
template <int D, int HS>
int attend_v6_chunk_rows() { return Att6Cfg<D, HS>::CH; }

#define WK_INST_ATT6(D, HS)                                                                                   \
  template __global__ void attend_v6_kernel<D, HS, false, false, true>(                                        \
      IndexView, SteadyView, StepView, AttnParams, const int32_t*, int, const __grid_constant__ CUtensorMap);  \
  template __global__ void attend_v6_kernel<D, HS, false, true, false>(                                        \
      IndexView, SteadyView, StepView, AttnParams, const int32_t*, int, const __grid_constant__ CUtensorMap);  \
  template __global__ void attend_v6_kernel<D, HS, true, false, false>(                                        \
      IndexView, SteadyView, StepView, AttnParams, const int32_t*, int, const __grid_constant__ CUtensorMap);  \
  template size_t attend_v6_smem<D, HS>();                                                                    \
  template int attend_v6_warps<D, HS>();                                                                      \
  template int attend_v6_consumers<D, HS>();                                                                  \
  template int attend_v6_chunk_rows<D, HS>();
WK_INST_ATT6(128, 4)
WK_INST_ATT6(128, 8)
WK_INST_ATT6(64, 4)
WK_INST_ATT6(64, 8)
template __global__ void att6_merge_kernel<false, 4>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int, int);
template __global__ void att6_merge_kernel<true, 4>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int, int);
template __global__ void att6_merge_kernel<false, 2>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int, int);
template __global__ void att6_merge_kernel<true, 2>(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int, int);

}  // namespace wk
