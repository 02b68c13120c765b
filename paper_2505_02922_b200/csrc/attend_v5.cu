// attend_v5.cu -- fused tripartite decode attention (attention.py:67-148,
// engine.py:150-172) for bf16 K/V stores: the exact zones (steady tokens and
// retrieved clusters) run their q.k and p.v contractions on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32), the estimation zone on the FP32 pipes.
//
// Why tensor cores here: per token the step does 2 G FMAs per 2 bytes of K/V
// (G <= 8), far below any compute roofline, but on the CUDA cores every FMA,
// every bf16 -> fp32 unpack and every shuffle of the q.k reduction is an
// issued instruction; attend_v4 (CUDA cores) issued ~890 warp instructions per
// 16-row chunk and stalled on issue at 4 TB/s (profiles/r1_attend_v4_*).
// One m16n8k16 does 2048 multiply-adds from registers, so a 16-token chunk is
// 16 ldmatrix + 40 MMAs + a short softmax and the warp goes back to waiting
// on HBM.
//
// fp32-equivalent arithmetic on bf16 tensor cores: the keys and values are
// bf16 (the store's own format, exact); the query and the softmax weights are
// fp32 and are split exactly into three bf16 terms x = hi + mid + lo
// (hi = bf16(x), mid = bf16(x - hi), lo = bf16(x - hi - mid): 24 mantissa
// bits).  Every product of two bf16 numbers is exact in fp32 and the tensor
// core accumulates in fp32, so q.k and sum p v carry fp32-level error like the
// CUDA-core path (tolerance rel-L2 1e-5 vs the fp64 oracle).
//
//   q.k:  S^T[token][col] = K[token][:] . Qs^T[:][col]   (M = 16 tokens, K = d,
//         N = head x split columns: G <= 4 -> 2 n-tiles (hi|mid interleaved,
//         lo), G <= 8 -> 3 n-tiles (one per split)); the three split columns
//         of a head are summed in registers (no shuffles).
//   p.v:  O^T[dim][head] += V^T[dim][tokens] . P_s[tokens][head]  for s in
//         {lo, mid, hi}  (M = 16 dims per tile, K = 16 tokens, N = 8 heads);
//         O^T stays in the accumulator fragments for the whole (unit, kind)
//         run of the warp.
//
// Schedule (shared with att4_merge_kernel): a flat list of chunks over all
// units -- steady runs of 16 rows, the retrieved tokens 16 at a time (row
// mode: select_v6 wrote every retrieved token's store row + head mask, so the
// clusters' runs are packed into full chunks; offload: the cache's pieces),
// the estimation rows 16 at a time -- split evenly over a persistent grid of
// P CTAs x WARPS warps.  Each warp streams its range through a 2-stage ring
// filled by 1-D bulk copies (TMA), one per contiguous run of store rows (a
// 16-row chunk of retrieved tokens is ~2 cluster runs); the bf16 rows are
// stored swizzled (common.cuh swz_col: 16-byte piece c of row r at c ^ (r & 7)),
// so the 8 row addresses of an ldmatrix hit 8 distinct bank groups without
// padding.  Measured alternatives: one bulk copy per row into padded rows
// (a bulk copy takes warp-uniform operands, so 16 lanes' row addresses go
// through a serialising R2UR loop, ~6 instructions per row: the top stall of
// that version, 81 us/layer) and cp.async (LDGSTS) per 16 bytes (123 us).
// Partials (M, D, num[d]) are flushed per (unit, kind) and folded by
// att4_merge_kernel.
#include <cuda_bf16.h>

#include "common.cuh"
#include "decode_internal.h"

namespace wk {

__device__ __align__(128) unsigned char g_zero5[8192];

template <int D, int HS>
struct Att5Cfg {
  static constexpr int RG = 16;                    // rows per chunk (mma K for p.v)
  static constexpr int KS = D / 16;                // q.k k-steps == p.v m-tiles
  static constexpr int NT = HS == 4 ? 2 : 3;       // q.k n-tiles
  static constexpr int NL = HS == 4 ? 2 : 4;       // (row, head) logit slots per lane
  static constexpr int NH = HS == 4 ? 1 : 2;       // logit heads per lane
  static constexpr int NA = KS * 4;                // accumulator floats per lane
#ifndef ATT5_NST
#define ATT5_NST 2  // tuning experiments only (tools/att5_sweep.sh)
#endif
#ifndef ATT5_WMAX
#define ATT5_WMAX 12
#endif
  static constexpr int NST = ATT5_NST;             // ring stages per warp
  static constexpr int ROWT = D * 2;               // bf16 K or V row bytes
  static constexpr int ROWV = D * 4;               // fp32 value-sum row bytes
  static constexpr int SB = ((2 * RG * ROWT > RG * ROWV ? 2 * RG * ROWT : RG * ROWV) + 127) / 128 * 128;
  // per warp: stage tags + row (head mask | swizzle key << 8), per-stage estimation inputs (logit
  // + weight per lane slot), bf16 split weights [3][8 heads][16 tokens], fp32
  // weights [16][HS]
  static constexpr int META = NST * 48 + NST * NL * 32 * 8 + 3 * 8 * RG * 2 + RG * HS * 4;
  static constexpr int MAXU = 1024;
  static constexpr int WPB = NST * SB + NST * 8 + META;  // bytes per warp
  static constexpr int FIT = (227 * 1024 - (MAXU + 1) * 4 - 64) / WPB;
  static constexpr int WARPS = FIT > ATT5_WMAX ? ATT5_WMAX : FIT;
  static constexpr size_t SMEM = (size_t)WARPS * WPB + (size_t)(MAXU + 1) * 4 + 64;
};

WK_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
WK_DEVINL void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
WK_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
WK_DEVINL void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                        uint32_t b1) {
  // not volatile: a pure register operation the compiler may interleave
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// mbarrier wait on a 32-bit shared-window address
WK_DEVINL void mbar_wait_s(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
// exact split x = hi + mid + lo into bf16 terms (bits of each term)
WK_DEVINL void split3(float x, uint32_t& hi, uint32_t& mid, uint32_t& lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(m);
  const __nv_bfloat16 l = __float2bfloat16_rn(r2);
  hi = __bfloat16_as_ushort(h);
  mid = __bfloat16_as_ushort(m);
  lo = __bfloat16_as_ushort(l);
}

// chunk counts of unit u: steady, retrieval (pieces / RG-row groups / store
// runs), estimation
template <int RG, bool FULL, bool ROWS>
WK_DEVINL void att5_counts(const SteadyView& st, const StepView& sv, const int32_t* n_store, int u, int& c0,
                           int& c1, int& c2) {
  c0 = (st.n[u] + RG - 1) / RG;
  if (FULL) {
    c1 = (n_store[u] + RG - 1) / RG;
    c2 = 0;
  } else {
    c1 = ROWS ? (sv.cnt[u * 4 + 1] + RG - 1) / RG : sv.cnt[u * 4 + 3];
    c2 = (sv.cnt[u * 4 + 2] + RG - 1) / RG;
  }
#ifdef ATT5_SKIP  // timing experiments only: 1 = no estimation chunks, 2 = no exact chunks
  if (ATT5_SKIP == 1) c2 = 0;
  if (ATT5_SKIP == 2) { c0 = 0; c1 = 0; }
#endif
}

template <int D, int HS, bool FULL, bool OFF, bool ROWS>
__global__ void __launch_bounds__(Att5Cfg<D, HS>::WARPS * 32, 1)
    attend_v5_kernel(IndexView ix, SteadyView st, StepView sv, AttnParams p, const int32_t* __restrict__ n_store,
                     int U) {
  using CF = Att5Cfg<D, HS>;
  constexpr int RG = CF::RG, KS = CF::KS, NT = CF::NT, NL = CF::NL, NH = CF::NH, NA = CF::NA, NST = CF::NST;
  constexpr int ROWT = CF::ROWT, ROWV = CF::ROWV, SB = CF::SB;
  constexpr int DL = D / 16;  // estimation mode: dims per lane
  pdl_wait();
  const int G = p.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;      // mma fragment coordinates
  const int half = lane >> 4, sub = lane & 15;  // estimation mode coordinates
  extern __shared__ __align__(128) unsigned char a5s[];
  unsigned char* ring = a5s + (size_t)warp * NST * SB;
  const uint32_t ring_s = smem_u32(ring);
  uint64_t* bars = reinterpret_cast<uint64_t*>(a5s + (size_t)CF::WARPS * NST * SB) + warp * NST;
  const uint32_t bars_s = smem_u32(bars);
  unsigned char* meta = a5s + (size_t)CF::WARPS * NST * (SB + 8) + (size_t)warp * CF::META;
  int4* stag = reinterpret_cast<int4*>(meta);                                 // [NST] chunk tags
  unsigned short* smk = reinterpret_cast<unsigned short*>(meta + NST * 16);   // [NST][16] mask | key << 8
  float* sx = reinterpret_cast<float*>(meta + NST * 48);                      // [NST][NL][32]
  float* sw = sx + NST * NL * 32;                                             // [NST][NL][32]
  unsigned short* pb = reinterpret_cast<unsigned short*>(sw + NST * NL * 32);  // [3][8][RG] bf16
  float* pe = reinterpret_cast<float*>(pb + 3 * 8 * RG);                      // [RG][HS]
  const uint32_t pb_s = smem_u32(pb);
  int* woff = reinterpret_cast<int*>(a5s + (size_t)CF::WARPS * (NST * (SB + 8) + CF::META));

  // ---- chunk prefix over units (every CTA; U <= MAXU) ----
  {
    int carry = 0;
    for (int base = 0; base < U; base += blockDim.x) {
      const int u = base + threadIdx.x;
      int c = 0;
      if (u < U) {
        int c0, c1, c2;
        att5_counts<RG, FULL, ROWS>(st, sv, n_store, u, c0, c1, c2);
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
  // split-weight rows of the unused head slots stay zero
  for (int i = lane; i < 3 * 8 * RG / 2; i += 32) reinterpret_cast<uint32_t*>(pb)[i] = 0u;
  __syncwarp();

  const float isd = p.inv_sqrt_d;
  const int allmask = (1 << G) - 1;
  // logit slot l of this lane: (row, head); head index within the lane: hs(l)
  auto slot_row = [&](int l) { return g8 + 8 * (HS == 4 ? l : (l >> 1)); };
  auto slot_head = [&](int l) { return HS == 4 ? t4 : 2 * t4 + (l & 1); };

  // ---- issue cursor ----
  int iu = 0;
  {
    int lo = 0, hi = U - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (woff[mid] <= ca) lo = mid; else hi = mid - 1;
    }
    iu = lo;
  }
  int ic0 = 0, ic1 = 0, ic2 = 0;
  if (ca < cb) att5_counts<RG, FULL, ROWS>(st, sv, n_store, iu, ic0, ic1, ic2);
  int in_st = 0, in_x = 0;  // steady rows / retrieved rows (ROWS) or store rows (FULL) of the cursor's unit
  auto unit_sizes = [&]() {
    in_st = st.n[iu];
    in_x = FULL ? n_store[iu] : (ROWS ? sv.cnt[iu * 4 + 1] : 0);
  };
  if (ca < cb) unit_sizes();
  struct Meta {
    int h;   // unit (bits 0-19) | kind + 1 (20-21) | n (22-26)
    int a;   // first row (steady / FULL / offload piece), the lane's row | mask << 24 (ROWS),
             // or the lane's estimation cluster
    int mk;  // head mask (steady / FULL), piece word (offload)
    float x[NL], w[NL];  // kind 2: lane slots' logits / weights; offload: cluster, first token
  };
  auto chunk_meta = [&](long long ci) {
    Meta m;
    m.h = 0; m.a = 0; m.mk = 0;
#pragma unroll
    for (int l = 0; l < NL; l++) { m.x[l] = -INFINITY; m.w[l] = 0.f; }
    if (ci >= cb) return m;
    while (ci >= woff[iu + 1]) {
      iu++;
      att5_counts<RG, FULL, ROWS>(st, sv, n_store, iu, ic0, ic1, ic2);
      unit_sizes();
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
        n = min(RG, in_x - m.a);
        m.mk = allmask;
      } else if (ROWS) {
        const int r0 = lc * RG;
        n = min(RG, in_x - r0);
        if ((lane & 15) < n) m.a = __ldcg(sv.rtok_row + (size_t)u * sv.rt_cap + r0 + (lane & 15));
      } else {  // offload piece: (row, n | mask << 8 | flags << 16, cluster, first token)
        const int4 pc = __ldcg(reinterpret_cast<const int4*>(sv.pieces) + (size_t)u * sv.pc_cap + lc);
        m.a = pc.x;
        n = pc.y & 0xff;
        m.mk = pc.y;
        m.x[0] = __int_as_float(pc.z);
        m.w[0] = __int_as_float(pc.w);
      }
    } else {
      kind = 2;
      lc -= ic0 + ic1;
      const int e0 = lc * RG;
      n = min(RG, sv.cnt[u * 4 + 2] - e0);
      if ((lane & 15) < n) m.a = __ldcg(sv.eu_ids + (size_t)u * sv.eu_cap + e0 + (lane & 15));
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int r = slot_row(l), h = slot_head(l);
        if (r < n && h < G) {
          m.x[l] = __ldcg(sv.eu_x + ((size_t)u * sv.eu_cap + e0 + r) * G + h);
          m.w[l] = __ldcg(sv.eu_sz + (size_t)u * sv.eu_cap + e0 + r);
        }
      }
    }
    m.h = u | ((kind + 1) << 20) | ((n & 31) << 22);
    return m;
  };
  // Copies (TMA 1-D bulk): the K and V rows of a chunk arrive as one bulk copy
  // per contiguous run of store rows (row mode: a cluster's members are
  // contiguous, so a 16-row chunk is ~2 runs), issued by the run's first lane;
  // bf16 rows are stored swizzled (common.cuh swz_col), so the unpadded rows
  // read conflict-free with ldmatrix.  Estimation rows: one copy per row.
  auto issue = [&](int sti, const Meta& m) {
    const int u = m.h & 0xfffff, kind = ((m.h >> 20) & 3) - 1, n = (m.h >> 22) & 31;
    const uint32_t stage_s = ring_s + sti * SB, bar = bars_s + sti * 8;
    const int j = lane & 15;
    const bool live = lane < n;
    int flags = 0;
    if (kind < 2) {
      int row, mk;
      const unsigned char* bk;
      const unsigned char* bv;
      if (kind == 0) {
        row = m.a + j;
        mk = m.mk;
        bk = (const unsigned char*)st.k + (size_t)u * st.t_cap * ROWT;
        bv = (const unsigned char*)st.v + (size_t)u * st.t_cap * ROWT;
      } else if (FULL) {
        row = m.a + j;
        mk = m.mk;
        bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
        bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
      } else if (ROWS) {
        row = m.a & 0xffffff;
        mk = (int)((unsigned)m.a >> 24);
        bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
        bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
      } else {  // offload piece: hit -> the HBM slot arena, miss -> the pinned host store (zero-copy TMA)
        row = m.a + j;
        mk = (m.mk >> 8) & 0xff;
        flags = (m.mk >> 16) & 3;
        if (flags & 1) {
          bk = (const unsigned char*)sv.arena_k + (size_t)u * sv.arena_rows * ROWT;
          bv = (const unsigned char*)sv.arena_v + (size_t)u * sv.arena_rows * ROWT;
        } else {
          bk = (const unsigned char*)ix.store_k + (size_t)u * ix.s_cap * ROWT;
          bv = (const unsigned char*)ix.store_v + (size_t)u * ix.s_cap * ROWT;
        }
      }
      // runs of consecutive rows among lanes 0..n-1
      const int prev = __shfl_up_sync(0xffffffffu, row, 1);
      const bool start = live && (lane == 0 || row != prev + 1);
      const unsigned starts = __ballot_sync(0xffffffffu, start);
      if (lane == 0) mbar_arrive_expect_tx(bars + sti, (uint32_t)((n + RG) * ROWT));
      __syncwarp();
      if (start) {
        const unsigned later = starts & ~((2u << lane) - 1u);
        const int len = (later ? __ffs(later) - 1 : n) - lane;
        bulk_g2s(ring + sti * SB + lane * ROWT, bk + (size_t)row * ROWT, (uint32_t)(len * ROWT), bars + sti);
        bulk_g2s(ring + sti * SB + RG * ROWT + lane * ROWT, bv + (size_t)row * ROWT, (uint32_t)(len * ROWT),
                 bars + sti);
      }
      // V rows >= n zero-filled (a zero weight never meets a stale non-finite
      // value); K rows >= n stay stale (head mask 0: logits masked by selection)
      if (lane == 0 && n < RG)
        bulk_g2s(ring + sti * SB + RG * ROWT + n * ROWT, g_zero5, (uint32_t)((RG - n) * ROWT), bars + sti);
      if (lane < RG) smk[sti * 16 + lane] = (unsigned short)(live ? (mk | ((row & 7) << 8)) : ((lane & 7) << 8));
    } else {
      if (lane == 0) mbar_arrive_expect_tx(bars + sti, (uint32_t)(RG * ROWV));
      __syncwarp();
      if (live)
        bulk_g2s(ring + sti * SB + lane * ROWV, ix.VS32 + ((size_t)u * ix.m_cap + m.a) * D, (uint32_t)ROWV,
                 bars + sti);
      if (lane == 0 && n < RG) bulk_g2s(ring + sti * SB + n * ROWV, g_zero5, (uint32_t)((RG - n) * ROWV), bars + sti);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        sx[(sti * NL + l) * 32 + lane] = m.x[l];
        sw[(sti * NL + l) * 32 + lane] = m.w[l];
      }
    }
    (void)bar;
    (void)stage_s;
    // tag: (unit, kind + 1 | rows << 8, offload write-through: cluster, first token | 1 << 31)
    if (lane == 0)
      stag[sti] = make_int4(u, (kind + 1) | (n << 8),
                            (OFF && kind == 1 && (flags & 2)) ? __float_as_int(m.x[0]) : 0,
                            (OFF && kind == 1 && (flags & 2)) ? ((__float_as_int(m.w[0]) & 0xffffff) | (int)0x80000000) : 0);
  };

  // ---- q of the current unit as the split B fragments of the q.k MMAs ----
  // column c of n-tile nt: G <= 4: nt 0 -> (head c/2, split c&1), nt 1 -> (head
  // c/2, split 2) for even c, zero for odd c; G <= 8: (head c, split nt)
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

  // ---- softmax state: per lane, the references and denominator partials of
  // its logit heads (uniform over the 8 lanes sharing t4); accumulators ----
  float mo[NH], dl[NH], acc[NA];
  auto reset = [&]() {
#pragma unroll
    for (int i = 0; i < NH; i++) { mo[i] = -INFINITY; dl[i] = 0.f; }
#pragma unroll
    for (int i = 0; i < NA; i++) acc[i] = 0.f;
  };
  reset();
  int cu = -1, ck = -1;  // (unit, kind) of the open partial
  // estimation-mode layout: lane (half, sub) owns dims dim_e(j) of heads
  // hb + 0..3 (G <= 4: hb = 0, rows of parity `half`; G <= 8: hb = 4 half, all
  // rows); acc[h4 * DL + j]
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
    float* base = sv.part + ((size_t)(wg + cu) * 3 + ck) * (size_t)G * (4 + D);
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

  // Lazily rescaled online softmax (as attend_v4): weights exp(x - ref) <= e^10
  // accumulate unscaled; a head's reference moves only when one of its logits
  // exceeds it by > 10 (warp vote), rescaling that head's accumulators.
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
          al[i] = mo[i] == -INFINITY ? 0.f : __expf(mo[i] - mx);
          mo[i] = mx;
        }
        dl[i] *= al[i];
      }
      // the accumulators' heads: alphas from the lanes owning them (head h:
      // lane h (G <= 4), lane h / 2 slot h & 1 (G <= 8))
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

  auto compute = [&](int sti, int tagw) {
    const int kind = (tagw & 0xff) - 1;
    const uint32_t stage_s = ring_s + sti * SB;
    float x[NL], pw[NL];
    if (kind < 2) {
      // ---- q.k on the tensor cores: S^T = K . Qs^T ----
      // two accumulator sets (even / odd k-steps) halve the dependent MMA chain
      float c[NT][4], c2[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; nt++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[nt][i] = c2[nt][i] = 0.f;
      // swizzled rows: piece c of chunk row r sits at piece c ^ key(r)
      const int jk = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int kbk = ((smk[sti * 16 + jk] >> 8) & 7) ^ (lane >> 4);
      const uint32_t aK = stage_s + jk * ROWT;
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
      const int mk_lo = smk[sti * 16 + g8] & 0xff, mk_hi = smk[sti * 16 + g8 + 8] & 0xff;
#pragma unroll
      for (int l = 0; l < NL; l++) {
        float s;
        if (HS == 4) {
          const int ci = 2 * l;  // row g8 (l = 0) -> c[.][0..1]; row g8 + 8 -> c[.][2..3]
          s = (c[0][ci] + c[0][ci + 1]) + c[1][ci];
        } else {
          const int ci = 2 * (l >> 1) + (l & 1);
          s = (c[0][ci] + c[1][ci]) + c[2][ci];
        }
        const int mk = (HS == 4 ? l : (l >> 1)) ? mk_hi : mk_lo;
        x[l] = ((mk >> slot_head(l)) & 1) ? s : -INFINITY;
      }
      softmax(x, false);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int i = HS == 4 ? 0 : (l & 1);
        pw[l] = x[l] == -INFINITY ? 0.f : __expf(x[l] - mo[i]);
        dl[i] += pw[l];
        uint32_t sh, sm, sl;
        split3(pw[l], sh, sm, sl);
        const int idx = slot_head(l) * RG + slot_row(l);
        pb[idx] = (unsigned short)sh;
        pb[8 * RG + idx] = (unsigned short)sm;
        pb[16 * RG + idx] = (unsigned short)sl;
      }
      __syncwarp();
      // ---- p.v on the tensor cores: O^T += V^T . P_s ----
      uint32_t b[3][2];
      {
        const int mi = lane >> 3, r = lane & 7;
        ldsm_x4(pb_s + (((mi >> 1) * 8 + r) * RG + (mi & 1) * 8) * 2, b[0][0], b[0][1], b[1][0], b[1][1]);
        ldsm_x2(pb_s + ((16 + r) * RG + (mi & 1) * 8) * 2, b[2][0], b[2][1]);
      }
      const int jv = (lane & 7) + 8 * (lane >> 4);
      const int kbv = ((smk[sti * 16 + jv] >> 8) & 7) ^ ((lane >> 3) & 1);
      const uint32_t aV = stage_s + RG * ROWT + jv * ROWT;
      // all V fragments first, then the MMAs split-major (lo, mid, hi) so
      // consecutive MMAs update different accumulator tiles
      uint32_t av[KS][4];
#pragma unroll
      for (int mt = 0; mt < KS; mt++)
        ldsm_x4_t(aV + (((2 * mt) ^ kbv) << 4), av[mt][0], av[mt][1], av[mt][2], av[mt][3]);
#pragma unroll
      for (int s = 2; s >= 0; s--)
#pragma unroll
        for (int mt = 0; mt < KS; mt++) {
          float (&cc)[4] = *reinterpret_cast<float(*)[4]>(&acc[mt * 4]);
          mma_bf16(cc, av[mt][0], av[mt][1], av[mt][2], av[mt][3], b[s][0], b[s][1]);
        }
    } else {
      // ---- estimation rows: fp32 value sums on the FP32 pipes ----
      float wz[NL];
#pragma unroll
      for (int l = 0; l < NL; l++) {
        x[l] = sx[(sti * NL + l) * 32 + lane];
        wz[l] = sw[(sti * NL + l) * 32 + lane];
      }
      softmax(x, true);
#pragma unroll
      for (int l = 0; l < NL; l++) {
        const int i = HS == 4 ? 0 : (l & 1);
        pw[l] = x[l] == -INFINITY ? 0.f : __expf(x[l] - mo[i]);
        dl[i] = fmaf(pw[l], wz[l], dl[i]);
        pe[slot_row(l) * HS + slot_head(l)] = pw[l];
      }
      __syncwarp();
      const unsigned char* stage = ring + sti * SB;
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
      mbar_wait_s(bars_s + sti * 8, (uint32_t)((k / NST) & 1));
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
          const size_t ar = (size_t)__ldcg(sl + so + tok / bt) * bt + tok % bt;  // the unit's arena row
          const size_t arow = (size_t)cu * sv.arena_rows + ar;
          const int ks = (smk[sti * 16 + i] >> 8) & 7, ka = (int)(ar & 7);  // re-swizzle: store key -> arena key
          if (sub < ROWT / 16) {
            *reinterpret_cast<uint4*>((unsigned char*)sv.arena_k + arow * ROWT + ((sub ^ ka) << 4)) =
                *reinterpret_cast<const uint4*>(stage + i * ROWT + ((sub ^ ks) << 4));
            *reinterpret_cast<uint4*>((unsigned char*)sv.arena_v + arow * ROWT + ((sub ^ ka) << 4)) =
                *reinterpret_cast<const uint4*>(stage + RG * ROWT + i * ROWT + ((sub ^ ks) << 4));
          }
        }
      }
      __syncwarp();
    }
    pdl_trigger<4>();
    flush();
  }
}

template <int D, int HS>
size_t attend_v5_smem() { return Att5Cfg<D, HS>::SMEM; }
template <int D, int HS>
int attend_v5_warps() { return Att5Cfg<D, HS>::WARPS; }

#define WK_INST_ATT5(D, HS)                                                                                     \
  template __global__ void attend_v5_kernel<D, HS, false, false, true>(IndexView, SteadyView, StepView,          \
                                                                       AttnParams, const int32_t*, int);        \
  template __global__ void attend_v5_kernel<D, HS, false, true, false>(IndexView, SteadyView, StepView,          \
                                                                       AttnParams, const int32_t*, int);        \
  template __global__ void attend_v5_kernel<D, HS, true, false, false>(IndexView, SteadyView, StepView,          \
                                                                       AttnParams, const int32_t*, int);        \
  template size_t attend_v5_smem<D, HS>();                                                                      \
  template int attend_v5_warps<D, HS>();
WK_INST_ATT5(128, 4)
WK_INST_ATT5(128, 8)
WK_INST_ATT5(64, 4)
WK_INST_ATT5(64, 8)

}  // namespace wk
