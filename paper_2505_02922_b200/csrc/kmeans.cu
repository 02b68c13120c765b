// kmeans.cu -- segmented spherical k-means on B200 (prefill index build and
// decode-time index updates).  Restates tierkv clustering.py:66-101 and
// index.py:43-58 / 143-186 bit-exactly: the CPU reference's fp32/fp64
// evaluation orders are reproduced with round-to-nearest intrinsics (see
// common.cuh).  All segments of all (request, kv-head) units of a layer are
// processed by one launch per phase.
#include <type_traits>

#include "common.cuh"
#include "wavekv_internal.h"

namespace wk {

// ---------------------------------------------------------------------------
// phase 1: centre by the fp32 column mean (sequential over rows, then / n)
// and normalize rows (clustering.py:82, :16-23).
// grid = n_segments, block = 256
// ---------------------------------------------------------------------------
__global__ void km_prep_kernel(const SegDesc* __restrict__ segs, float* __restrict__ P_all, int d,
                               __half* __restrict__ P16_all) {
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  extern __shared__ float sm_mean[];
  const float* keys = sg.keys;
  float* P = P_all + (size_t)sg.p_off * d;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < sg.L; i++) s = __fadd_rn(s, keys[(size_t)i * sg.key_stride + t]);
    sm_mean[t] = __fdiv_rn(s, (float)sg.L);
  }
  __syncthreads();
  for (size_t idx = threadIdx.x; idx < (size_t)sg.L * d; idx += blockDim.x) {
    size_t i = idx / d, t = idx % d;
    P[idx] = __fsub_rn(keys[i * sg.key_stride + t], sm_mean[t]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < sg.L; i += blockDim.x) {
    float* row = P + (size_t)i * d;
    float nr = row_norm_f32(row, d);
    if (nr != 0.0f) {
      for (int t = 0; t < d; t++) row[t] = __fdiv_rn(row[t], nr);
    } else {
      for (int t = 0; t < d; t++) row[t] = 0.f;
      row[0] = 1.0f;
    }
    if (P16_all) {
      __half* r16 = P16_all + ((size_t)sg.p_off + i) * d;
      for (int t = 0; t < d; t++) r16[t] = __float2half_rn(row[t]);
    }
  }
}

// v2 of the prep for d = 32 EPL (32 / 64 / 128): the column means keep the
// sequential fp32 chain of np.mean(axis=0) with 8 loads in flight per column;
// then one warp per row (lane = EPL contiguous dims, coalesced): centre, square
// into smem, the 8 pairwise-sum chains of np.linalg.norm on lanes 0-7 (one
// block of 8 per step, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by shuffles),
// divide, write P and P16 in the same pass.  Bit-identical to km_prep_kernel.
template <int EPL>
__global__ void __launch_bounds__(512) km_prep_v2_kernel(const SegDesc* __restrict__ segs, float* __restrict__ P_all,
                                                         __half* __restrict__ P16_all) {
  constexpr int D = 32 * EPL;
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  __shared__ float mean[D];
  __shared__ float sq[16][D];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, NW = blockDim.x >> 5;
  const float* keys = sg.keys;
  if (t < D) {
    float sum = 0.f;
    int i = 0;
    for (; i + 8 <= sg.L; i += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] = __ldg(keys + (size_t)(i + k) * sg.key_stride + t);
#pragma unroll
      for (int k = 0; k < 8; k++) sum = __fadd_rn(sum, v[k]);
    }
    for (; i < sg.L; i++) sum = __fadd_rn(sum, __ldg(keys + (size_t)i * sg.key_stride + t));
    mean[t] = __fdiv_rn(sum, (float)sg.L);
  }
  __syncthreads();
  float mu[EPL];
#pragma unroll
  for (int e = 0; e < EPL; e++) mu[e] = mean[lane * EPL + e];
  float* P = P_all + (size_t)sg.p_off * D;
  __half* P16 = P16_all ? P16_all + (size_t)sg.p_off * D : nullptr;
  float* sw = sq[warp];
  for (int i = warp; i < sg.L; i += NW) {
    const float* kr = keys + (size_t)i * sg.key_stride + lane * EPL;
    float x[EPL];
    if (EPL == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(kr));
      x[0] = v.x; x[1 % EPL] = v.y; x[2 % EPL] = v.z; x[3 % EPL] = v.w;
    } else if (EPL == 2) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(kr));
      x[0] = v.x; x[1 % EPL] = v.y;
    } else {
      x[0] = __ldg(kr);
    }
#pragma unroll
    for (int e = 0; e < EPL; e++) {
      x[e] = __fsub_rn(x[e], mu[e]);
      sw[lane * EPL + e] = __fmul_rn(x[e], x[e]);
    }
    __syncwarp();
    float r = 0.f;
    if (lane < 8) {
      r = sw[lane];
#pragma unroll
      for (int j = 8; j < D; j += 8) r = __fadd_rn(r, sw[j + lane]);
    }
    r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));
    r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 2));
    r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 4));
    const float nr = __fsqrt_rn(__shfl_sync(0xffffffffu, r, 0));
    __syncwarp();
    float y[EPL];
#pragma unroll
    for (int e = 0; e < EPL; e++) y[e] = nr != 0.f ? __fdiv_rn(x[e], nr) : (lane * EPL + e == 0 ? 1.f : 0.f);
    float* pr = P + (size_t)i * D + lane * EPL;
    if (EPL == 4) *reinterpret_cast<float4*>(pr) = make_float4(y[0], y[1 % EPL], y[2 % EPL], y[3 % EPL]);
    else if (EPL == 2) *reinterpret_cast<float2*>(pr) = make_float2(y[0], y[1 % EPL]);
    else pr[0] = y[0];
    if (P16) {
      __half* hr = P16 + (size_t)i * D + lane * EPL;
#pragma unroll
      for (int e = 0; e < EPL; e++) hr[e] = __float2half_rn(y[e]);
    }
  }
}
template __global__ void km_prep_v2_kernel<1>(const SegDesc*, float*, __half*);
template __global__ void km_prep_v2_kernel<2>(const SegDesc*, float*, __half*);
template __global__ void km_prep_v2_kernel<4>(const SegDesc*, float*, __half*);

// ---------------------------------------------------------------------------
// phase 2: k-means++ seeding under cosine distance (clustering.py:26-43).
// One CTA per segment runs the k-1 sequential steps; the sgemv of each step
// is spread over the CTA with the OpenBLAS row recipe, the fp32 cumsum is the
// reference's sequential chain (thread 0), the draw is numpy's PCG64 stream.
// grid = n_segments, block = 512, dyn smem = d floats (+2L floats if it fits)
// ---------------------------------------------------------------------------
__global__ void km_seed_kernel(const SegDesc* __restrict__ segs, const float* __restrict__ P_all,
                               float* __restrict__ C_all, float* __restrict__ scratch_all,
                               int d, int blas_threads, int smem_rows) {
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  extern __shared__ float sm[];
  float* cent = sm;  // d floats: current centroid
  const int L = sg.L;
  float *md, *cdf;
  if (L <= smem_rows) {
    md = sm + d;
    cdf = md + L;
  } else {
    md = scratch_all + (size_t)sg.p_off * 2;
    cdf = md + L;
  }
  const float* P = P_all + (size_t)sg.p_off * d;
  float* C = C_all + (size_t)sg.c_off * d;
  __shared__ Pcg64 g;
  __shared__ long long s_idx;
  if (threadIdx.x == 0) {
    g.hi = sg.rng[0]; g.lo = sg.rng[1]; g.ihi = sg.rng[2]; g.ilo = sg.rng[3];
    g.has32 = 0; g.u32 = 0;
    s_idx = pcg_integers(g, L);
  }
  __syncthreads();
  for (int c = 0; c < sg.k; c++) {
    const long long idx = s_idx;
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
      float v = P[(size_t)idx * d + t];
      cent[t] = v;
      C[(size_t)c * d + t] = v;
    }
    __syncthreads();
    if (c == sg.k - 1) break;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      int cls = gemv_row_class(i, L, d, blas_threads);
      float dot = sgemv_row(P + (size_t)i * d, cent, d, cls);
      float v = __fsub_rn(1.0f, dot);
      v = v < 0.f ? 0.f : v;
      if (c == 0) md[i] = v;
      else if (!(md[i] <= v)) md[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = md[0];
      cdf[0] = s;
      for (int i = 1; i < L; i++) { s = __fadd_rn(s, md[i]); cdf[i] = s; }
      long long nidx;
      if (s <= 0.0f) {
        nidx = pcg_integers(g, L);
      } else {
        float u = (float)pcg_next_double(g);
        float thr = __fmul_rn(u, s);
        int lo = 0, hi = L;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (cdf[mid] <= thr) lo = mid + 1; else hi = mid; }
        nidx = lo > L - 1 ? L - 1 : lo;
      }
      s_idx = nidx;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// phase 2 (v2): the same k-means++ steps with a coalesced, recipe-exact sgemv.
// A main row (OpenBLAS group-of-4 row, gemv_row_class 0) is served by two
// lanes: lane h owns the accumulators a[4h .. 4h+3] of the reference's 8-way
// FMA split (t mod 8) and streams its 16-byte slices t = 8s + 4h; the two
// halves are combined in the recipe order ((a_l + a_{l+4}), then
// (s0+s1)+(s2+s3)).  A warp covers 16 rows per 16-byte load instruction
// (512 contiguous-row bytes).  Chunk-tail rows (classes 1, 2) keep the
// per-thread recipe.  The fp32 cumsum stays the reference's sequential chain
// (recomputed in a second pass up to the drawn index instead of being stored).
// Rows the new centre provably cannot improve are skipped before any load
// (triangle inequality on the unit sphere, rigorous margin KS_EPS covering the
// fp32 evaluation): with b = the row's current best centre,
//   ||p - c|| >= ||c_b - c|| - ||p - c_b||,  ||p - c_b||^2 <= 2 (md + eps),
// so if (D_lo - r_hi)^2 / 2 >= md + eps the computed 1 - p.c is >= md and
// min(md, .) keeps md -- the same bits as evaluating the row.
// grid = n_segments, block = 256
// ---------------------------------------------------------------------------
constexpr float KS_EPS = 1e-4f;
constexpr int KS_CKS = 32;                 // cumsum checkpoint stride (elements)
constexpr int KS_CK = 8192 / KS_CKS + 4;   // checkpoint slots (stride grows with L past 8192)
// per-phase cycle totals of km_seed_v2 for tools/seed_timing.py (a separate
// -DWK_SEED_TIMING build; compiled out of the product library)
#ifdef WK_SEED_TIMING
__device__ long long g_seed_ts[8192 * 4];
extern "C" int wk_seed_timing(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_seed_ts, sizeof(long long) * (size_t)n) == cudaSuccess ? 0 : -2;
}
#define KS_T0() long long ks_t = clock64()
#define KS_LAP(i) do { if (threadIdx.x == 0) { const long long n_ = clock64(); ks_acc[i] += n_ - ks_t; ks_t = n_; } } while (0)
#else
#define KS_T0() do {} while (0)
#define KS_LAP(i) do {} while (0)
#endif
#ifndef KS_MINB
#define KS_MINB 4  // 4 segments per SM (64 registers): the seeding is latency-bound
#endif
__global__ void __launch_bounds__(256, KS_MINB) km_seed_v2_kernel(const SegDesc* __restrict__ segs, const float* __restrict__ P_all,
                                                         float* __restrict__ C_all, float* __restrict__ scratch_all,
                                                         int d, int blas_threads, int in_smem,
                                                         const __half* __restrict__ P16_all, int max_k) {
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  extern __shared__ __align__(16) float sm2[];
  float* cent = sm2;          // d floats: current centroid
  float* ccd = sm2 + d;       // max_k floats: lower bounds of ||C[a] - cent||
  float* ck = ccd + ((max_k + 3) & ~3);  // KS_CK cumsum checkpoints
  const int L = sg.L;
  float* md;
  unsigned short* best;       // the centre each row's md was last set by
  unsigned short* lst;        // rows the new centre may improve (compacted), global scratch
  const int L4 = (L + 3) & ~3;
  if (in_smem) {
    md = ck + KS_CK;
    best = reinterpret_cast<unsigned short*>(md + L4);
    lst = reinterpret_cast<unsigned short*>(scratch_all + (size_t)sg.p_off * 2);
  } else {
    md = scratch_all + (size_t)sg.p_off * 2;
    best = reinterpret_cast<unsigned short*>(md + L);
    lst = best + L;
  }
  __shared__ int s_nact;
  const float* P = P_all + (size_t)sg.p_off * d;
  const __half* P16 = P16_all ? P16_all + (size_t)sg.p_off * d : nullptr;
  float* C = C_all + (size_t)sg.c_off * d;
  __shared__ Pcg64 g;
  __shared__ long long s_idx;
  if (threadIdx.x == 0) {
    g.hi = sg.rng[0]; g.lo = sg.rng[1]; g.ihi = sg.rng[2]; g.ilo = sg.rng[3];
    g.has32 = 0; g.u32 = 0;
    s_idx = pcg_integers(g, L);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int h = lane & 1, rsub = lane >> 1;  // 16 rows per warp, 2 lanes per row
  const int nq = d >> 3;                     // 16-byte slices per lane (d % 8 == 0)
#ifdef WK_SEED_TIMING
  long long ks_acc[4] = {0, 0, 0, 0};
  long long ks_nact = 0;
#endif
  KS_T0();
  // rows [0, main_end) of every chunk are class 0; find the first non-main row
  for (int c = 0; c < sg.k; c++) {
    const long long idx = s_idx;
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
      const float v = P[(size_t)idx * d + t];
      cent[t] = v;
      C[(size_t)c * d + t] = v;
    }
    __syncthreads();
    if (c == sg.k - 1) break;
    // lower bounds of the distances from the earlier centres to the new one:
    // one thread per earlier centre, the row's 16-byte slices loaded together
    // (independent rows in flight instead of a serial warp reduction per row)
    for (int a = threadIdx.x; a < c; a += blockDim.x) {
      const float4* cr = reinterpret_cast<const float4*>(C + (size_t)a * d);
      float dp0 = 0.f, dp1 = 0.f;
      for (int q0 = 0; q0 < (d >> 2); q0 += 8) {
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; j++) x[j] = q0 + j < (d >> 2) ? __ldcg(cr + q0 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; j++) {
          if (q0 + j >= (d >> 2)) break;
          const float4 y = reinterpret_cast<const float4*>(cent)[q0 + j];
          dp0 = fmaf(x[j].x, y.x, dp0); dp1 = fmaf(x[j].y, y.y, dp1);
          dp0 = fmaf(x[j].z, y.z, dp0); dp1 = fmaf(x[j].w, y.w, dp1);
        }
      }
      ccd[a] = sqrtf(fmaxf(0.f, 2.f * (1.f - (dp0 + dp1) - KS_EPS)));
    }
    if (threadIdx.x == 0) s_nact = 0;
    __syncthreads();
    KS_LAP(0);
    // compaction: the rows the new centre may improve (the triangle test
    // fails); the row pass below then keeps every lane busy on those only
    for (int i0 = 0; i0 < L; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      bool act = i < L;
      if (act && c > 0) {
        const float m = md[i];
        const float rh = sqrtf(2.f * (m + KS_EPS)), dl = ccd[best[i]];
        if (dl > rh && 0.5f * (dl - rh) * (dl - rh) >= m + KS_EPS) act = false;
      }
      const unsigned am = __ballot_sync(0xffffffffu, act);
      if (am) {
        int b = 0;
        if (lane == 0) b = atomicAdd(&s_nact, __popc(am));
        b = __shfl_sync(0xffffffffu, b, 0);
        if (act) lst[b + __popc(am & ((1u << lane) - 1u))] = (unsigned short)i;
      }
    }
    __syncthreads();
    KS_LAP(3);
    const int nact = s_nact;
#ifdef WK_SEED_TIMING
    if (threadIdx.x == 0) ks_nact += nact;
#endif
    for (int base = warp * 16; base < nact; base += nwarp * 16) {
      const int j = base + rsub;
      bool act = j < nact;
      const int i = act ? (int)lst[j] : 0;
      if (act && c > 0 && P16) {
        // first pass on the fp16 copy: |dot' - dot| <= 2^-11 + 2 gamma_d for
        // unit rows, so v' - 1e-3 >= md[i] proves min(md, v) == md (no update)
        const uint4* r16 = reinterpret_cast<const uint4*>(P16 + (size_t)i * d) + h * (nq / 2);
        float a = 0.f;
        uint4 wv[8];
#pragma unroll
        for (int q = 0; q < 8; q++) wv[q] = q < nq / 2 ? __ldcg(r16 + q) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if (q >= nq / 2) break;
          const uint4 w = wv[q];
          const __half2* hh = reinterpret_cast<const __half2*>(&w);
          const float* cc = cent + h * (d / 2) + 8 * q;
#pragma unroll
          for (int e2 = 0; e2 < 4; e2++) {
            const float2 f = __half22float2(hh[e2]);
            a = fmaf(f.x, cc[2 * e2], a);
            a = fmaf(f.y, cc[2 * e2 + 1], a);
          }
        }
        const unsigned pm16 = __activemask() & (0x3u << (lane & ~1));
        a += __shfl_xor_sync(pm16, a, 1);
        const float vq = 1.0f - a;
        if (vq - 1e-3f >= md[i]) act = false;
      }
      const int cls = act ? gemv_row_class(i, L, d, blas_threads) : 0;
      float dot = 0.f;
      const unsigned both = __ballot_sync(0xffffffffu, act && cls == 0);
      if (act && cls == 0) {
        const float4* row = reinterpret_cast<const float4*>(P + (size_t)i * d) + h;
        const float4* cv = reinterpret_cast<const float4*>(cent) + h;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        // two batches of 8 slices in flight (16 at once spilled to local
        // memory under the 64-register budget of 4 segments per SM)
#pragma unroll
        for (int q0 = 0; q0 < 16; q0 += 8) {
          if (q0 >= nq) break;
          float4 xv[8];
#pragma unroll
          for (int q = 0; q < 8; q++)
            xv[q] = q0 + q < nq ? __ldcg(row + 2 * (q0 + q)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (q0 + q >= nq) break;
            const float4 x = xv[q], y = cv[2 * (q0 + q)];
            a0 = __fmaf_rn(x.x, y.x, a0);
            a1 = __fmaf_rn(x.y, y.y, a1);
            a2 = __fmaf_rn(x.z, y.z, a2);
            a3 = __fmaf_rn(x.w, y.w, a3);
          }
        }
        // lane h = 0 holds a0..a3, h = 1 holds a4..a7: s_l = a_l + a_{l+4}
        const unsigned pm = both & (0x3u << (lane & ~1));
        const float b0 = __shfl_xor_sync(pm, a0, 1), b1 = __shfl_xor_sync(pm, a1, 1);
        const float b2 = __shfl_xor_sync(pm, a2, 1), b3 = __shfl_xor_sync(pm, a3, 1);
        const float s0 = __fadd_rn(a0, b0), s1 = __fadd_rn(a1, b1), s2 = __fadd_rn(a2, b2), s3 = __fadd_rn(a3, b3);
        dot = __fadd_rn(0.f, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
      } else if (act && h == 0) {
        dot = sgemv_row(P + (size_t)i * d, cent, d, cls);
      }
      if (act && h == 0) {
        float v = __fsub_rn(1.0f, dot);
        v = v < 0.f ? 0.f : v;
        if (c == 0 || !(md[i] <= v)) { md[i] = v; best[i] = (unsigned short)c; }
      }
    }
    __syncthreads();
    KS_LAP(1);
    if (threadIdx.x == 0) {
      // the reference's sequential fp32 cumsum (clustering.py:35): one pass
      // with batched loads (the chain runs at the FADD latency) storing the
      // running sum every KS_CKS elements; searchsorted('right') then
      // re-walks the same chain from the last checkpoint <= threshold (the
      // cumsum is non-decreasing: md >= 0 and rounding is monotone)
      float sacc = 0.f;  // 0 + md[0] == md[0] (md >= +0)
      const int cks = KS_CKS * ((L + 8191) / 8192);  // checkpoint stride: <= KS_CK checkpoints
      const int nfull = (L / KS_CKS) * KS_CKS;
      // full blocks: unpredicated 16-byte loads issued before the FADD chain
      // (shared or global md; the serial thread competes for issue slots)
      auto blocks = [&](const float* mdp, auto vec) {
        int ci = 0;
        for (int i0 = 0; i0 < nfull; i0 += KS_CKS) {
          if (i0 == ci * cks) { ck[ci] = sacc; ci++; }
          float v[KS_CKS];
          if (vec) {
#pragma unroll
            for (int q = 0; q < KS_CKS / 4; q++) {
              const float4 x = reinterpret_cast<const float4*>(mdp + i0)[q];
              v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < KS_CKS; q++) v[q] = mdp[i0 + q];
          }
#pragma unroll
          for (int q = 0; q < KS_CKS; q++) sacc = __fadd_rn(sacc, v[q]);
        }
        if (nfull < L && nfull == ci * cks) ck[ci] = sacc;
        for (int i = nfull; i < L; i++) sacc = __fadd_rn(sacc, mdp[i]);
      };
      // md in shared memory is 16-byte aligned (d, K4, KS_CK multiples of 4)
      if (in_smem) blocks(ck + KS_CK, std::true_type{});
      else blocks(md, std::false_type{});
      long long nidx;
      if (sacc <= 0.0f) {
        nidx = pcg_integers(g, L);
      } else {
        const float u = (float)pcg_next_double(g);
        const float thr = __fmul_rn(u, sacc);
        int lo = 0, hi = (L - 1) / cks;  // last checkpoint <= thr (ck[0] = 0 <= thr)
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ck[mid] <= thr) lo = mid; else hi = mid - 1;
        }
        float s2 = ck[lo];
        int i = lo * cks;
        for (; i < L; i++) {
          s2 = __fadd_rn(s2, md[i]);
          if (s2 > thr) break;
        }
        nidx = i > L - 1 ? L - 1 : i;
      }
      s_idx = nidx;
    }
    __syncthreads();
    KS_LAP(2);
  }
#ifdef WK_SEED_TIMING
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; i++) g_seed_ts[blockIdx.x * 4 + i] = ks_acc[i];
  if (threadIdx.x == 0) g_seed_ts[8192 * 4 - 1 - blockIdx.x] = ks_nact;
#endif
}

// ---------------------------------------------------------------------------
// phase 2 (v3): k-means++ seeding with ONE WARP per segment.  The 511 steps of
// a segment are a serial chain whose floor is the reference's sequential fp32
// cumsum (8,124 dependent FADDs per step, clustering.py:35); v2 gave every
// segment a 256-thread CTA, so only 4 chains ran per SM and each step paid ~5
// block barriers plus their memory round trips (343 ms for the 1,920 segments
// of a 120K-context layer).  Here the segments run side by side (a 120K layer
// is one wave of ~13 warps per SM), every phase is warp-synchronous, and the
// arithmetic is v2's exactly (same bounds, same fp16 first pass, same recipe
// dots, same checkpointed cumsum / searchsorted):
//   * centre: one 16-byte slice per lane; earlier-centre distance bounds: one
//     lane per earlier centre;
//   * triangle test over all rows (lane-strided), survivors compacted by ballot;
//   * row pass: 16 rows per warp iteration, 2 lanes per row (the recipe split);
//   * cumsum: the warp stages 256 md values at a time into shared memory
//     (coalesced, the next block's loads in flight while lane 0 adds the
//     current one) and lane 0 runs the FADD chain from 16-byte smem reads.
// md / best / the compacted list live in the global scratch (L2-resident).
// grid = ceil(n_segments / KS3_W), block = 32 KS3_W, dyn smem = KS3_W * (d + K4 + KS_CK + 256) floats
// ---------------------------------------------------------------------------
constexpr int KS3_W = 4;  // segments (warps) per CTA
__global__ void __launch_bounds__(KS3_W * 32, 4) km_seed_v3_kernel(const SegDesc* __restrict__ segs, int n_segs,
                                                                    const float* __restrict__ P_all,
                                                                    float* __restrict__ C_all,
                                                                    float* __restrict__ scratch_all, int d,
                                                                    int blas_threads,
                                                                    const __half* __restrict__ P16_all, int max_k) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K4 = (max_k + 3) & ~3;
  extern __shared__ __align__(16) float sm3[];
  float* cent = sm3 + (size_t)warp * (d + K4 + KS_CK + 256);
  float* ccd = cent + d;
  float* ck = ccd + K4;
  float* stg = ck + KS_CK;  // 256 staged md values
  const int sgi = blockIdx.x * KS3_W + warp;
  if (sgi >= n_segs) return;
  const SegDesc sg = segs[sgi];
  if (sg.k <= 1) return;
  const int L = sg.L;
  float* md = scratch_all + (size_t)sg.p_off * 2;
  unsigned short* best = reinterpret_cast<unsigned short*>(md + L);
  unsigned short* lst = best + L;
  const float* P = P_all + (size_t)sg.p_off * d;
  const __half* P16 = P16_all ? P16_all + (size_t)sg.p_off * d : nullptr;
  float* C = C_all + (size_t)sg.c_off * d;
  Pcg64 g;
  long long idx = 0;
  if (lane == 0) {
    g.hi = sg.rng[0]; g.lo = sg.rng[1]; g.ihi = sg.rng[2]; g.ilo = sg.rng[3];
    g.has32 = 0; g.u32 = 0;
    idx = pcg_integers(g, L);
  }
  idx = __shfl_sync(0xffffffffu, idx, 0);
  const int h = lane & 1, rsub = lane >> 1;
  const int nq = d >> 3;
  const unsigned lt = (1u << lane) - 1u;
#ifdef WK_SEED_TIMING
  long long ks_acc[4] = {0, 0, 0, 0}, ks_t = clock64();
#define KS3_LAP(q) do { const long long n_ = clock64(); ks_acc[q] += n_ - ks_t; ks_t = n_; } while (0)
#else
#define KS3_LAP(q) do {} while (0)
#endif
  for (int c = 0; c < sg.k; c++) {
    for (int t = lane * 4; t < d; t += 128) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(P + (size_t)idx * d + t));
      *reinterpret_cast<float4*>(cent + t) = v;
      *reinterpret_cast<float4*>(C + (size_t)c * d + t) = v;
    }
    __syncwarp();
    if (c == sg.k - 1) break;
    // lower bounds of ||C[a] - cent|| (v2's formula and margin)
    for (int a = lane; a < c; a += 32) {
      const float4* cr = reinterpret_cast<const float4*>(C + (size_t)a * d);
      float dp0 = 0.f, dp1 = 0.f;
      for (int q0 = 0; q0 < (d >> 2); q0 += 8) {
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; j++) x[j] = q0 + j < (d >> 2) ? __ldcg(cr + q0 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; j++) {
          if (q0 + j >= (d >> 2)) break;
          const float4 y = reinterpret_cast<const float4*>(cent)[q0 + j];
          dp0 = fmaf(x[j].x, y.x, dp0); dp1 = fmaf(x[j].y, y.y, dp1);
          dp0 = fmaf(x[j].z, y.z, dp0); dp1 = fmaf(x[j].w, y.w, dp1);
        }
      }
      ccd[a] = sqrtf(fmaxf(0.f, 2.f * (1.f - (dp0 + dp1) - KS_EPS)));
    }
    __syncwarp();
    KS3_LAP(0);
    // triangle test over every row; survivors compacted (ascending order)
    // (order of the survivors is irrelevant: each row's update is its own).
    // Batches of 16 rows per lane with every load issued first: the loop is
    // bound by load latency otherwise (one L2 round trip per 32 rows).
    int nact = 0;
    constexpr int CB = 16;
    for (int i0 = 0; i0 < L; i0 += 32 * CB) {
      float m[CB];
      unsigned short bb[CB];
#pragma unroll
      for (int q = 0; q < CB; q++) {
        const int i = i0 + 32 * q + lane;
        m[q] = 0.f;
        bb[q] = 0;
        if (i < L && c > 0) { m[q] = __ldcg(md + i); bb[q] = __ldcg(best + i); }
      }
#pragma unroll
      for (int q = 0; q < CB; q++) {
        const int i = i0 + 32 * q + lane;
        bool act = i < L;
        if (act && c > 0) {
          const float rh = sqrtf(2.f * (m[q] + KS_EPS)), dl = ccd[bb[q]];
          if (dl > rh && 0.5f * (dl - rh) * (dl - rh) >= m[q] + KS_EPS) act = false;
        }
        const unsigned am = __ballot_sync(0xffffffffu, act);
        if (act) {
          lst[nact + __popc(am & lt)] = (unsigned short)i;
#ifdef KS3_PF16  // experiment: L2 prefetch of the survivors' fp16 rows
          const char* r16 = reinterpret_cast<const char*>(P16 ? (const void*)(P16 + (size_t)i * d)
                                                              : (const void*)(P + (size_t)i * d));
          for (int o = 0; o < (P16 ? 2 : 4) * d; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(r16 + o));
#endif
        }
        nact += __popc(am);
      }
    }
    __syncwarp();
    KS3_LAP(1);
    // row pass (v2's arithmetic), in two sweeps so the fp32 rows are fetched
    // to L2 while the fp16 filter runs: (1) fp16 first pass over the active
    // rows, survivors re-compacted into lst (positions already consumed) with
    // an L2 prefetch of their fp32 rows; (2) the recipe-exact dot + update
    int n2 = nact;
    if (c > 0 && P16) {
      n2 = 0;
      int inext = rsub < nact ? (int)__ldcg(lst + rsub) : 0;
      for (int base = 0; base < nact; base += 16) {
        const int j = base + rsub;
        bool act = j < nact;
        const int i = inext;
        inext = j + 16 < nact ? (int)__ldcg(lst + j + 16) : 0;
        // the next iteration's fp16 rows to L2 (each lane of a pair: its half)
        if (j + 16 < nact)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(P16 + (size_t)inext * d) + h * d));
        float mdi = 0.f;
        if (act) {
          mdi = __ldcg(md + i);
          const uint4* r16 = reinterpret_cast<const uint4*>(P16 + (size_t)i * d) + h * (nq / 2);
          float a = 0.f;
          uint4 wv[8];
#pragma unroll
          for (int q = 0; q < 8; q++) wv[q] = q < nq / 2 ? __ldcg(r16 + q) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (q >= nq / 2) break;
            const uint4 w = wv[q];
            const __half2* hh = reinterpret_cast<const __half2*>(&w);
            const float* cc = cent + h * (d / 2) + 8 * q;
#pragma unroll
            for (int e2 = 0; e2 < 4; e2++) {
              const float2 f = __half22float2(hh[e2]);
              a = fmaf(f.x, cc[2 * e2], a);
              a = fmaf(f.y, cc[2 * e2 + 1], a);
            }
          }
          const unsigned pm16 = __activemask() & (0x3u << (lane & ~1));
          a += __shfl_xor_sync(pm16, a, 1);
          const float vq = 1.0f - a;
          // v' - 1e-3 >= md proves min(md, v) == md (no update)
          if (vq - 1e-3f >= mdi) act = false;
        }
        const bool keep = act && h == 0;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          lst[n2 + __popc(km & lt)] = (unsigned short)i;
          const char* rp = reinterpret_cast<const char*>(P + (size_t)i * d);
          for (int o = 0; o < 4 * d; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + o));
        }
        n2 += __popc(km);
      }
      __syncwarp();
    }
    {
      int inext = rsub < n2 ? (int)__ldcg(lst + rsub) : 0;
      for (int base = 0; base < n2; base += 16) {
        const int j = base + rsub;
        const bool act = j < n2;
        const int i = inext;
        inext = j + 16 < n2 ? (int)__ldcg(lst + j + 16) : 0;
        const int cls = act ? gemv_row_class(i, L, d, blas_threads) : 0;
        float dot = 0.f;
        const unsigned both = __ballot_sync(0xffffffffu, act && cls == 0);
        if (act && cls == 0) {
          const float4* row = reinterpret_cast<const float4*>(P + (size_t)i * d) + h;
          const float4* cv = reinterpret_cast<const float4*>(cent) + h;
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int q0 = 0; q0 < 16; q0 += 8) {
            if (q0 >= nq) break;
            float4 xv[8];
#pragma unroll
            for (int q = 0; q < 8; q++)
              xv[q] = q0 + q < nq ? __ldcg(row + 2 * (q0 + q)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              if (q0 + q >= nq) break;
              const float4 x = xv[q], y = cv[2 * (q0 + q)];
              a0 = __fmaf_rn(x.x, y.x, a0);
              a1 = __fmaf_rn(x.y, y.y, a1);
              a2 = __fmaf_rn(x.z, y.z, a2);
              a3 = __fmaf_rn(x.w, y.w, a3);
            }
          }
          const unsigned pm = both & (0x3u << (lane & ~1));
          const float b0 = __shfl_xor_sync(pm, a0, 1), b1 = __shfl_xor_sync(pm, a1, 1);
          const float b2 = __shfl_xor_sync(pm, a2, 1), b3 = __shfl_xor_sync(pm, a3, 1);
          const float s0 = __fadd_rn(a0, b0), s1 = __fadd_rn(a1, b1), s2 = __fadd_rn(a2, b2), s3 = __fadd_rn(a3, b3);
          dot = __fadd_rn(0.f, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
        } else if (act && h == 0) {
          dot = sgemv_row(P + (size_t)i * d, cent, d, cls);
        }
        if (act && h == 0) {
          float v = __fsub_rn(1.0f, dot);
          v = v < 0.f ? 0.f : v;
          if (c == 0 || !(__ldcg(md + i) <= v)) { md[i] = v; best[i] = (unsigned short)c; }
        }
      }
    }
    __syncwarp();
    KS3_LAP(2);
    // the sequential fp32 cumsum (clustering.py:35), checkpoint every KS_CKS
    // elements; blocks of 256 staged through shared memory by the whole warp
    // (the next block's loads in flight while lane 0 adds the current one)
    const int cks = KS_CKS * ((L + 8191) / 8192);
    float sacc = 0.f;
    {
      float nxt[8];
      auto fetch = [&](int b0) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const int i = b0 + lane + 32 * q;
          nxt[q] = i < L ? __ldcg(md + i) : 0.f;
        }
      };
      fetch(0);
      for (int b0 = 0; b0 < L; b0 += 256) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; q++) stg[lane + 32 * q] = nxt[q];
        __syncwarp();
        if (b0 + 256 < L) fetch(b0 + 256);
        if (lane == 0) {
          const int nb = min(256, L - b0);
          if (nb == 256 && (cks % 4) == 0) {
#pragma unroll 2
            for (int q = 0; q < 256; q += KS_CKS) {
              if (((b0 + q) % cks) == 0) ck[(b0 + q) / cks] = sacc;
              float v[KS_CKS];
#pragma unroll
              for (int e = 0; e < KS_CKS / 4; e++) {
                const float4 x = reinterpret_cast<const float4*>(stg + q)[e];
                v[4 * e] = x.x; v[4 * e + 1] = x.y; v[4 * e + 2] = x.z; v[4 * e + 3] = x.w;
              }
#pragma unroll
              for (int e = 0; e < KS_CKS; e++) sacc = __fadd_rn(sacc, v[e]);
            }
          } else {
            for (int q = 0; q < nb; q++) {
              if (((b0 + q) % cks) == 0) ck[(b0 + q) / cks] = sacc;
              sacc = __fadd_rn(sacc, stg[q]);
            }
          }
        }
      }
    }
    if (lane == 0) {
      long long nidx;
      if (sacc <= 0.0f) {
        nidx = pcg_integers(g, L);
      } else {
        const float u = (float)pcg_next_double(g);
        const float thr = __fmul_rn(u, sacc);
        int lo = 0, hi = (L - 1) / cks;  // last checkpoint <= thr (ck[0] = 0 <= thr)
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ck[mid] <= thr) lo = mid; else hi = mid - 1;
        }
        float s2 = ck[lo];
        int i = lo * cks;
        for (; i < L; i++) {
          s2 = __fadd_rn(s2, __ldcg(md + i));
          if (s2 > thr) break;
        }
        nidx = i > L - 1 ? L - 1 : i;
      }
      idx = nidx;
    }
    idx = __shfl_sync(0xffffffffu, idx, 0);
    KS3_LAP(3);
  }
#ifdef WK_SEED_TIMING
  if (lane == 0)
    for (int q = 0; q < 4; q++) g_seed_ts[sgi * 4 + q] = ks_acc[q];
#endif
}

// ---------------------------------------------------------------------------
// phase 3 (tensor cores): assignment = argmax(points @ centroids.T), the
// reference's sequential fp32 FMA chain per score (clustering.py:85,96), via
// a tensor-core first pass + exact verification.
//   * first pass: bf16x3 split products (p_hi c_hi + p_hi c_lo + p_lo c_hi) on
//     mma.sync.m16n8k16 with fp32 accumulation; rows are unit vectors, so
//     |s' - s_exact| <= B = 1e-4 for every (point, centroid) (split residuals
//     3 * 2^-18, accumulation 384 * 2^-23, the reference chain's own gamma_128);
//   * each lane keeps the top 4 s' of its rows; the quad merges them;
//   * every centroid within 2B of the best s' is re-scored with the exact
//     fp32 chain and the first index of the exact max wins (np.argmax); if
//     the 4th candidate is still within 2B the point falls back to an exact
//     scan of all centroids.
// grid = (ceil(Lmax / 64), n_segments), block = 128 (4 warps x 16 points);
// smem: a chunk of 64 centroids as bf16 hi / lo rows padded to 136 elements.
// ---------------------------------------------------------------------------
constexpr int KTC_CH = 64;     // centroids per smem chunk
constexpr int KTC_PAD = 136;   // padded bf16 row (conflict-free B fragment loads)
constexpr float KTC_B = 1e-4f;

WK_DEVINL void ktc_mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
WK_DEVINL uint32_t ktc_pack(float x, float y) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(y)) << 16);
}
WK_DEVINL void ktc_split(float x, float y, uint32_t& hi, uint32_t& lo) {
  const float hx = __bfloat162float(__float2bfloat16_rn(x)), hy = __bfloat162float(__float2bfloat16_rn(y));
  hi = ktc_pack(hx, hy);
  lo = ktc_pack(x - hx, y - hy);
}
// insert (v, i) into a descending top-4 list
WK_DEVINL void ktc_ins(float (&tv)[4], int (&ti)[4], float v, int i) {
  if (!(v > tv[3])) return;
  if (v > tv[2]) { tv[3] = tv[2]; ti[3] = ti[2]; } else { tv[3] = v; ti[3] = i; return; }
  if (v > tv[1]) { tv[2] = tv[1]; ti[2] = ti[1]; } else { tv[2] = v; ti[2] = i; return; }
  if (v > tv[0]) { tv[1] = tv[0]; ti[1] = ti[0]; tv[0] = v; ti[0] = i; } else { tv[1] = v; ti[1] = i; }
}
WK_DEVINL float ktc_exact(const float* __restrict__ p, const float* __restrict__ c, int d) {
  float acc = 0.f;
#pragma unroll 16
  for (int t = 0; t < d; t++) acc = __fmaf_rn(__ldg(p + t), __ldg(c + t), acc);
  return acc;
}
// four candidates' sequential fp32 FMA chains side by side (the same bits as
// ktc_exact per candidate; the chains' latencies overlap instead of adding up)
WK_DEVINL void ktc_exact4(const float* __restrict__ p, const float* __restrict__ c0, const float* __restrict__ c1,
                          const float* __restrict__ c2, const float* __restrict__ c3, int d, float (&out)[4]) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  for (int t0 = 0; t0 < d; t0 += 4) {
    const float4 pv = __ldg(reinterpret_cast<const float4*>(p + t0));
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(c0 + t0));
    const float4 x1 = __ldg(reinterpret_cast<const float4*>(c1 + t0));
    const float4 x2 = __ldg(reinterpret_cast<const float4*>(c2 + t0));
    const float4 x3 = __ldg(reinterpret_cast<const float4*>(c3 + t0));
    a0 = __fmaf_rn(pv.x, x0.x, a0); a1 = __fmaf_rn(pv.x, x1.x, a1); a2 = __fmaf_rn(pv.x, x2.x, a2); a3 = __fmaf_rn(pv.x, x3.x, a3);
    a0 = __fmaf_rn(pv.y, x0.y, a0); a1 = __fmaf_rn(pv.y, x1.y, a1); a2 = __fmaf_rn(pv.y, x2.y, a2); a3 = __fmaf_rn(pv.y, x3.y, a3);
    a0 = __fmaf_rn(pv.z, x0.z, a0); a1 = __fmaf_rn(pv.z, x1.z, a1); a2 = __fmaf_rn(pv.z, x2.z, a2); a3 = __fmaf_rn(pv.z, x3.z, a3);
    a0 = __fmaf_rn(pv.w, x0.w, a0); a1 = __fmaf_rn(pv.w, x1.w, a1); a2 = __fmaf_rn(pv.w, x2.w, a2); a3 = __fmaf_rn(pv.w, x3.w, a3);
  }
  out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3;
}

template <int KS>
__global__ void __launch_bounds__(128) km_assign_tc_kernel(const SegDesc* __restrict__ segs,
                                                            const float* __restrict__ P_all,
                                                            const float* __restrict__ C_all,
                                                            int32_t* __restrict__ A_all) {
  constexpr int d = KS * 16;
  const SegDesc sg = segs[blockIdx.y];
  if (sg.k <= 1) return;
  if ((long long)sg.L * sg.k <= 1200) return;  // OpenBLAS small-kernel shapes: km_assign_small_kernel
  const int p0 = blockIdx.x * 64;
  if (p0 >= sg.L) return;
  __shared__ __align__(16) __nv_bfloat16 csh[2][KTC_CH][KTC_PAD];  // [hi/lo][centroid][dim]
  const float* P = P_all + (size_t)sg.p_off * d;
  const float* C = C_all + (size_t)sg.c_off * d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = p0 + warp * 16 + g, r1 = r0 + 8;  // this lane's two point rows
  // A fragments (points, hi / lo), resident for the whole centroid loop
  uint32_t ah[KS][4], al[KS][4];
  {
    const float* pr0 = P + (size_t)min(r0, sg.L - 1) * d;
    const float* pr1 = P + (size_t)min(r1, sg.L - 1) * d;
#pragma unroll
    for (int s = 0; s < KS; s++) {
      const int k0 = 16 * s + 2 * t;
      const float2 x00 = *reinterpret_cast<const float2*>(pr0 + k0), x10 = *reinterpret_cast<const float2*>(pr1 + k0);
      const float2 x01 = *reinterpret_cast<const float2*>(pr0 + k0 + 8), x11 = *reinterpret_cast<const float2*>(pr1 + k0 + 8);
      ktc_split(x00.x, x00.y, ah[s][0], al[s][0]);
      ktc_split(x10.x, x10.y, ah[s][1], al[s][1]);
      ktc_split(x01.x, x01.y, ah[s][2], al[s][2]);
      ktc_split(x11.x, x11.y, ah[s][3], al[s][3]);
    }
  }
  float tv0[4], tv1[4];
  int ti0[4], ti1[4];
#pragma unroll
  for (int i = 0; i < 4; i++) { tv0[i] = tv1[i] = -INFINITY; ti0[i] = ti1[i] = 0x7fffffff; }
  for (int c0 = 0; c0 < sg.k; c0 += KTC_CH) {
    const int nc = min(KTC_CH, sg.k - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < KTC_CH * (d / 2); idx += blockDim.x) {
      const int c = idx / (d / 2), t2 = (idx % (d / 2)) * 2;
      float2 x = make_float2(0.f, 0.f);
      if (c < nc) x = *reinterpret_cast<const float2*>(C + (size_t)(c0 + c) * d + t2);
      uint32_t hi, lo;
      ktc_split(x.x, x.y, hi, lo);
      *reinterpret_cast<uint32_t*>(&csh[0][c][t2]) = hi;
      *reinterpret_cast<uint32_t*>(&csh[1][c][t2]) = lo;
    }
    __syncthreads();
#pragma unroll 2
    for (int nt = 0; nt < KTC_CH / 8; nt++) {
      if (nt * 8 >= nc) break;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int cn = nt * 8 + g;
#pragma unroll
      for (int s = 0; s < KS; s++) {
        const int k0 = 16 * s + 2 * t;
        const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(&csh[0][cn][k0]);
        const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(&csh[0][cn][k0 + 8]);
        const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(&csh[1][cn][k0]);
        const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(&csh[1][cn][k0 + 8]);
        ktc_mma(acc, ah[s], bh0, bh1);
        ktc_mma(acc, ah[s], bl0, bl1);
        ktc_mma(acc, al[s], bh0, bh1);
      }
      const int ca = c0 + nt * 8 + 2 * t;
      if (nt * 8 + 2 * t < nc) { ktc_ins(tv0, ti0, acc[0], ca); ktc_ins(tv1, ti1, acc[2], ca); }
      if (nt * 8 + 2 * t + 1 < nc) { ktc_ins(tv0, ti0, acc[1], ca + 1); ktc_ins(tv1, ti1, acc[3], ca + 1); }
    }
  }
  // merge the quad's lists: every lane ends with the top 4 of its two rows
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    float ov0[4], ov1[4];
    int oi0[4], oi1[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      ov0[i] = __shfl_xor_sync(0xffffffffu, tv0[i], o); oi0[i] = __shfl_xor_sync(0xffffffffu, ti0[i], o);
      ov1[i] = __shfl_xor_sync(0xffffffffu, tv1[i], o); oi1[i] = __shfl_xor_sync(0xffffffffu, ti1[i], o);
    }
#pragma unroll
    for (int i = 0; i < 4; i++) { ktc_ins(tv0, ti0, ov0[i], oi0[i]); ktc_ins(tv1, ti1, ov1[i], oi1[i]); }
  }
  // exact verification: lane t takes row r0 (t < 2) or r1 (t >= 2)
  const int r = t < 2 ? r0 : r1;
  if (r >= sg.L) return;
  float tv[4];
  int ti[4];
#pragma unroll
  for (int i = 0; i < 4; i++) { tv[i] = t < 2 ? tv0[i] : tv1[i]; ti[i] = t < 2 ? ti0[i] : ti1[i]; }
  if ((t & 1) == 1) return;  // one lane per row
  const float* pr = P + (size_t)r * d;
  const float lim = tv[0] - 2.f * KTC_B;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  if (tv[3] >= lim) {
    // too many near-ties for the list: exact scan of every centroid
    for (int c = 0; c < sg.k; c++) {
      const float v = ktc_exact(pr, C + (size_t)c * d, d);
      if (v > best) { best = v; bi = c; }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      if (!(tv[i] >= lim)) break;
      const float v = ktc_exact(pr, C + (size_t)ti[i] * d, d);
      if (v > best || (v == best && ti[i] < bi)) { best = v; bi = ti[i]; }
    }
    if (bi == 0x7fffffff) bi = ti[0];  // non-finite scores: keep the first-pass winner
  }
  A_all[sg.p_off + r] = bi;
}
template __global__ void km_assign_tc_kernel<8>(const SegDesc*, const float*, const float*, int32_t*);
template __global__ void km_assign_tc_kernel<4>(const SegDesc*, const float*, const float*, int32_t*);
template __global__ void km_assign_tc_kernel<2>(const SegDesc*, const float*, const float*, int32_t*);

// ---------------------------------------------------------------------------
// phase 3 on the 5th-generation tensor cores (d = 128): the same bf16x3 first
// pass + exact verification as km_assign_tc_kernel, with the contraction on
// tcgen05.mma and the scores in TMEM.
//   * one CTA = 128 points of a segment, 4 warps; points (hi / lo bf16) and a
//     chunk of 256 centroids (hi / lo) are staged in smem in the K-major,
//     no-swizzle UMMA layout (8-row x 16-byte core matrices; LBO = 128 B along
//     K, SBO = 2 KB along M/N);
//   * thread 0 issues M128 x N256 x K16 MMAs: 3 split products x 8 K-steps per
//     centroid chunk into TMEM columns [256 j, 256 j + 256), then commits to an
//     mbarrier; the chunk buffer is refilled once the MMAs have read it;
//   * thread r owns TMEM lane r (= point r): tcgen05.ld 32 columns at a time,
//     top-4 insertion, then the exact fp32 chain for the candidates within 2B.
// grid = (ceil(Lmax / 128), n_segments), block = 128, dyn smem = 192 KB + 64.
// ---------------------------------------------------------------------------
constexpr int K5_M = 128, K5_N = 256, K5_D = 128;
constexpr uint32_t K5_A_BYTES = K5_M * K5_D * 2, K5_B_BYTES = K5_N * K5_D * 2;
constexpr size_t K5_SMEM = 2 * (size_t)K5_A_BYTES + 2 * (size_t)K5_B_BYTES + 64;  // + top-4 exchange aliases B

WK_DEVINL uint32_t k5_off(int r, int k) {  // byte offset of (row r, dim k) in a K-major no-swizzle operand
  return (uint32_t)((((r >> 3) * (K5_D / 8) + (k >> 3)) << 7) + ((r & 7) << 4) + ((k & 7) << 1));
}
WK_DEVINL uint64_t k5_desc(uint32_t saddr) {  // UMMA shared-memory descriptor, SWIZZLE_NONE
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);             // start address
  d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;        // LBO: next core matrix along K
  d |= (uint64_t)((2048u >> 4) & 0x3FFF) << 32;       // SBO: next 8-row group
  d |= (uint64_t)1 << 46;                              // descriptor version (sm_100)
  return d;                                            // base offset 0, layout type 0
}
// instruction descriptor: f32 accumulate, bf16 x bf16, both K-major, M = 128, N = 256
constexpr uint32_t K5_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(K5_N >> 3) << 17) |
                              ((uint32_t)(K5_M >> 4) << 24);

WK_DEVINL void k5_mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(K5_IDESC), "r"(acc));
}
WK_DEVINL void k5_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
WK_DEVINL void k5_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// centroids of every segment split to bf16 hi / lo once per Lloyd round, in the
// UMMA operand layout (rows beyond k zero, k rounded up to 8): segment s at
// element offset (c_off + 8 s) * 2 * d of `pk`, hi rows then lo rows, so a chunk
// of 256 rows is one contiguous 64 KB run for a bulk copy.
__global__ void km_pack_c5_kernel(const SegDesc* __restrict__ segs, const float* __restrict__ C_all,
                                  __nv_bfloat16* __restrict__ pk) {
  constexpr int d = K5_D;
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1 || (long long)sg.L * sg.k <= 1200) return;
  const int k8 = (sg.k + 7) & ~7;
  unsigned char* hi = reinterpret_cast<unsigned char*>(pk + ((size_t)sg.c_off + 8 * (size_t)blockIdx.x) * 2 * d);
  unsigned char* lo = hi + (size_t)k8 * d * 2;
  const float* C = C_all + (size_t)sg.c_off * d;
  for (int idx = threadIdx.x; idx < k8 * (d / 8); idx += blockDim.x) {
    const int c = idx / (d / 8), kg = idx % (d / 8);
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (c < sg.k) {
      a = *reinterpret_cast<const float4*>(C + (size_t)c * d + 8 * kg);
      b = *reinterpret_cast<const float4*>(C + (size_t)c * d + 8 * kg + 4);
    }
    uint4 h, l;
    ktc_split(a.x, a.y, h.x, l.x);
    ktc_split(a.z, a.w, h.y, l.y);
    ktc_split(b.x, b.y, h.z, l.z);
    ktc_split(b.z, b.w, h.w, l.w);
    *reinterpret_cast<uint4*>(hi + k5_off(c, 8 * kg)) = h;
    *reinterpret_cast<uint4*>(lo + k5_off(c, 8 * kg)) = l;
  }
}

__global__ void __launch_bounds__(256, 1) km_assign_tc5_kernel(const SegDesc* __restrict__ segs,
                                                                const float* __restrict__ P_all,
                                                                const float* __restrict__ C_all,
                                                                int32_t* __restrict__ A_all,
                                                                const __nv_bfloat16* __restrict__ pk) {
  constexpr int d = K5_D;
  const SegDesc sg = segs[blockIdx.y];
  if (sg.k <= 1) return;
  if ((long long)sg.L * sg.k <= 1200) return;  // OpenBLAS small-kernel shapes: km_assign_small_kernel
  const int p0 = blockIdx.x * K5_M;
  if (p0 >= sg.L) return;
  extern __shared__ __align__(1024) unsigned char k5s[];
  unsigned char* Ah = k5s;
  unsigned char* Al = Ah + K5_A_BYTES;
  unsigned char* Bh = Al + K5_A_BYTES;
  unsigned char* Bl = Bh + K5_B_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bl + K5_B_BYTES);  // [0] MMA commits, [1] B bulk copies
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const float* P = P_all + (size_t)sg.p_off * d;
  const float* C = C_all + (size_t)sg.c_off * d;
  const int t = threadIdx.x, warp = t >> 5;
  const int nchunk = (sg.k + K5_N - 1) / K5_N;  // <= 2 (k <= 512)
  const uint32_t ncols = nchunk > 1 ? 512u : 256u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  // points -> A (hi / lo): row t % 128, dims of half t / 128
  {
    const int row = t & (K5_M - 1), kh = t >> 7;
    const float* pr = P + (size_t)min(p0 + row, sg.L - 1) * d;
#pragma unroll 4
    for (int kg = kh * (d / 16); kg < (kh + 1) * (d / 16); kg++) {
      const float4 a = *reinterpret_cast<const float4*>(pr + 8 * kg), b = *reinterpret_cast<const float4*>(pr + 8 * kg + 4);
      uint4 h, l;
      ktc_split(a.x, a.y, h.x, l.x);
      ktc_split(a.z, a.w, h.y, l.y);
      ktc_split(b.x, b.y, h.z, l.z);
      ktc_split(b.z, b.w, h.w, l.w);
      *reinterpret_cast<uint4*>(Ah + k5_off(row, 8 * kg)) = h;
      *reinterpret_cast<uint4*>(Al + k5_off(row, 8 * kg)) = l;
    }
  }
  fence_proxy_async();  // A (generic-proxy smem writes) -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  if (t == 0) {
    // B chunks: one bulk copy each of the pre-split hi / lo rows, MMAs once they land
    const int k8 = (sg.k + 7) & ~7;
    const unsigned char* hi = reinterpret_cast<const unsigned char*>(pk + ((size_t)sg.c_off + 8 * (size_t)blockIdx.y) * 2 * d);
    const unsigned char* lo = hi + (size_t)k8 * d * 2;
    const uint32_t ah = smem_u32(Ah), al = smem_u32(Al), bh = smem_u32(Bh), bl = smem_u32(Bl);
    for (int j = 0; j < nchunk; j++) {
      if (j > 0) mbar_wait(bar, (uint32_t)((j - 1) & 1));  // the previous chunk's MMAs have read B
      const int rows = min(K5_N, k8 - j * K5_N);
      const uint32_t bytes = (uint32_t)rows * d * 2;
      mbar_arrive_expect_tx(bar + 1, 2 * bytes);
      bulk_g2s(Bh, hi + (size_t)j * K5_N * d * 2, bytes, bar + 1);
      bulk_g2s(Bl, lo + (size_t)j * K5_N * d * 2, bytes, bar + 1);
      mbar_wait(bar + 1, (uint32_t)(j & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tc = tmem + (uint32_t)(j * K5_N);
      uint32_t acc = 0;
#pragma unroll
      for (int kk = 0; kk < d / 16; kk++) {  // K step: 2 core matrices along K = 256 B
        const uint32_t ko = (uint32_t)kk * 256u;
        k5_mma(tc, k5_desc(ah + ko), k5_desc(bh + ko), acc); acc = 1;
        k5_mma(tc, k5_desc(ah + ko), k5_desc(bl + ko), 1);
        k5_mma(tc, k5_desc(al + ko), k5_desc(bh + ko), 1);
      }
      k5_commit(bar);
    }
  }
  if (t != 0)  // thread 0 passed these phases in its chunk loop
    for (int j = 0; j + 1 < nchunk; j++) mbar_wait(bar, (uint32_t)(j & 1));  // phases in order
  mbar_wait(bar, (uint32_t)((nchunk - 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // epilogue: warps w and w + 4 read TMEM lanes 32 (w % 4) .. + 31 (their points),
  // columns [0, 256) and [256, 512) respectively, 32 at a time; the two top-4
  // lists of a point meet in smem (aliasing the consumed B buffer)
  float tv[4];
  int ti[4];
#pragma unroll
  for (int i = 0; i < 4; i++) { tv[i] = -INFINITY; ti[i] = 0x7fffffff; }
  const int half = warp >> 2, row = t & (K5_M - 1);
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int cend = min(sg.k, (half + 1) * K5_N);
  for (int c0 = half * K5_N; c0 < cend; c0 += 32) {
    float v[32];
    k5_ld32(lane_base + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 32; i++)
      if (c0 + i < sg.k) ktc_ins(tv, ti, v[i], c0 + i);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  float* xv = reinterpret_cast<float*>(Bh);          // [128][4] values of the upper half
  int* xi = reinterpret_cast<int*>(Bh + 128 * 16);   // [128][4] indices
  if (half == 1)
#pragma unroll
    for (int i = 0; i < 4; i++) { xv[row * 4 + i] = tv[i]; xi[row * 4 + i] = ti[i]; }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
  if (half == 1) return;
#pragma unroll
  for (int i = 0; i < 4; i++) ktc_ins(tv, ti, xv[row * 4 + i], xi[row * 4 + i]);
  const int r = p0 + row;
  if (r >= sg.L) return;
  const float* pr = P + (size_t)r * d;
  const float lim = tv[0] - 2.f * KTC_B;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  if (tv[3] >= lim) {
    // more than four candidates within the margin: every centroid, four at a time
    for (int c = 0; c < sg.k; c += 4) {
      float v4[4];
      const float* cb = C + (size_t)c * d;
      ktc_exact4(pr, cb, c + 1 < sg.k ? cb + d : cb, c + 2 < sg.k ? cb + 2 * d : cb, c + 3 < sg.k ? cb + 3 * d : cb,
                 d, v4);
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (c + i < sg.k && v4[i] > best) { best = v4[i]; bi = c + i; }
    }
  } else {
    // the (<= 4) candidates' chains side by side (slots past the last
    // candidate repeat the first and are ignored)
    float v4[4];
    const float* cc[4];
#pragma unroll
    for (int i = 0; i < 4; i++) cc[i] = C + (size_t)((tv[i] >= lim) ? ti[i] : ti[0]) * d;
    ktc_exact4(pr, cc[0], cc[1], cc[2], cc[3], d, v4);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      if (!(tv[i] >= lim)) break;
      if (v4[i] > best || (v4[i] == best && ti[i] < bi)) { best = v4[i]; bi = ti[i]; }
    }
    if (bi == 0x7fffffff) bi = ti[0];
  }
  A_all[sg.p_off + r] = bi;
}

// ---------------------------------------------------------------------------
// phase 3: assignment = argmax(points @ centroids.T) (clustering.py:85,96).
// Every score is the reference's sequential fp32 FMA chain over t; register
// tiled 64 points x 64 centroids per CTA iteration, transposed smem tiles.
// grid = (ceil(Lmax/64), n_segments), block = 256, dyn smem = 2*d*65 floats
// ---------------------------------------------------------------------------
constexpr int AT = 64;  // tile edge
__global__ void __launch_bounds__(256) km_assign_kernel(const SegDesc* __restrict__ segs,
                                                         const float* __restrict__ P_all,
                                                         const float* __restrict__ C_all,
                                                         int32_t* __restrict__ A_all, int d) {
  const SegDesc sg = segs[blockIdx.y];
  if (sg.k <= 1) return;
  if ((long long)sg.L * sg.k <= 1200 && d >= 32) return;  // small-kernel path elsewhere
  const int p0 = blockIdx.x * AT;
  if (p0 >= sg.L) return;
  extern __shared__ float sm[];
  float* PT = sm;                  // [d][AT+1]
  float* CT = sm + d * (AT + 1);   // [d][AT+1]
  const float* P = P_all + (size_t)sg.p_off * d;
  const float* C = C_all + (size_t)sg.c_off * d;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int np = min(AT, sg.L - p0);
  for (int idx = threadIdx.x; idx < AT * d; idx += 256) {
    int p = idx / d, t = idx % d;
    PT[t * (AT + 1) + p] = p < np ? P[(size_t)(p0 + p) * d + t] : 0.f;
  }
  float best[4];
  int bidx[4];
#pragma unroll
  for (int i = 0; i < 4; i++) { best[i] = -INFINITY; bidx[i] = 0x7fffffff; }
  for (int c0 = 0; c0 < sg.k; c0 += AT) {
    const int nc = min(AT, sg.k - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < AT * d; idx += 256) {
      int c = idx / d, t = idx % d;
      CT[t * (AT + 1) + c] = c < nc ? C[(size_t)(c0 + c) * d + t] : 0.f;
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
    for (int t = 0; t < d; t++) {
      float pv[4], cv[4];
#pragma unroll
      for (int i = 0; i < 4; i++) pv[i] = PT[t * (AT + 1) + ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; j++) cv[j] = CT[t * (AT + 1) + tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = __fmaf_rn(pv[i], cv[j], acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int c = c0 + tx * 4 + j;
      if (tx * 4 + j < nc) {
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (acc[i][j] > best[i]) { best[i] = acc[i][j]; bidx[i] = c; }
      }
    }
  }
  // reduce across the 16 tx threads of each point group (ties -> smaller id)
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float b = best[i];
    int bi = bidx[i];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, b, o, 16);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o, 16);
      if (ob > b || (ob == b && oi < bi)) { b = ob; bi = oi; }
    }
    int p = ty * 4 + i;
    if (tx == 0 && p < np) A_all[sg.p_off + p0 + p] = bi;
  }
}

// OpenBLAS SkylakeX small-matrix TN kernel model (n*k <= 1200, d >= 32):
// 16-lane FMA accumulator, adjacent-pair lane tree except the corner block.
__device__ float small_tn_score(const float* p, const float* c, int d, bool corner) {
  float a[16];
#pragma unroll
  for (int l = 0; l < 16; l++) a[l] = 0.f;
  for (int t = 0; t < d; t++) a[t & 15] = __fmaf_rn(p[t], c[t], a[t & 15]);
  const int adj[4] = {0, 1, 2, 3}, red[4] = {3, 2, 1, 0};
  for (int lev = 0; lev < 4; lev++) {
    int b = 1 << (corner ? red[lev] : adj[lev]);
    for (int l = 0; l < 16; l++)
      if (!(l & b)) a[l] = __fadd_rn(a[l], a[l | b]);
  }
  return a[0];
}

__global__ void km_assign_small_kernel(const SegDesc* __restrict__ segs, const float* __restrict__ P_all,
                                       const float* __restrict__ C_all, int32_t* __restrict__ A_all, int d) {
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  if (!((long long)sg.L * sg.k <= 1200 && d >= 32)) return;
  const float* P = P_all + (size_t)sg.p_off * d;
  const float* C = C_all + (size_t)sg.c_off * d;
  const int n4 = sg.L & ~3, k4 = sg.k & ~3;
  for (int i = threadIdx.x; i < sg.L; i += blockDim.x) {
    float best = -INFINITY;
    int bi = 0;
    for (int c = 0; c < sg.k; c++) {
      float s = small_tn_score(P + (size_t)i * d, C + (size_t)c * d, d, i >= n4 && c >= k4);
      if (c == 0 || s > best) { best = s; bi = c; }
    }
    A_all[sg.p_off + i] = bi;
  }
}

// ---------------------------------------------------------------------------
// helpers shared by update/finalize: counts + stable counting sort of the
// points by cluster (ascending point index within a cluster).
// smem layout: cnt[k+1] (int), cursor[k] (int)
// ---------------------------------------------------------------------------
__device__ void stable_bucket(const int32_t* A, int L, int k, int* cnt, int* cursor, int32_t* perm) {
  for (int c = threadIdx.x; c <= k; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += blockDim.x) atomicAdd(&cnt[A[i] + 1], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < k; c++) cnt[c + 1] += cnt[c];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) cursor[c] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int base = 0; base < L; base += 32) {
      int i = base + lane;
      bool act = i < L;
      unsigned am = __ballot_sync(0xffffffffu, act);
      if (act) {
        int a = A[i];
        unsigned peers = __match_any_sync(am, a);
        int rank = __popc(peers & ((1u << lane) - 1u));
        int pos = cnt[a] + cursor[a] + rank;
        __syncwarp(am);
        perm[pos] = i;
        if ((31 - __clz(peers)) == lane) cursor[a] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// _repair_empty (clustering.py:46-63); serial over empties, parallel argmin.
__device__ void repair_empty(const float* P, int L, int d, int32_t* A, float* C, int k, int* counts,
                             float* sims, int* s_flag) {
  __shared__ int s_any;
  __shared__ float s_bv[32];
  __shared__ int s_bi[32];
  if (threadIdx.x == 0) {
    s_any = 0;
    for (int c = 0; c < k; c++) if (counts[c] == 0) { s_any = 1; break; }
  }
  __syncthreads();
  if (!s_any) return;
  for (int i = threadIdx.x; i < L; i += blockDim.x)
    sims[i] = einsum_row(P + (size_t)i * d, C + (size_t)A[i] * d, d);
  __syncthreads();
  for (int c = 0; c < k; c++) {
    if (counts[c] != 0) continue;  // list of empties is fixed up front; repair never empties
    float bv = INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      float cand = counts[A[i]] > 1 ? sims[i] : INFINITY;
      if (cand < bv || (cand == bv && i < bi)) { bv = cand; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { s_bv[threadIdx.x >> 5] = bv; s_bi[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      int nw = (blockDim.x + 31) >> 5;
      for (int w = 1; w < nw; w++)
        if (s_bv[w] < bv || (s_bv[w] == bv && s_bi[w] < bi)) { bv = s_bv[w]; bi = s_bi[w]; }
      int victim = bi;
      counts[A[victim]] -= 1;
      A[victim] = c;
      counts[c] = 1;
      sims[victim] = 1.0f;
      s_bi[0] = victim;
    }
    __syncthreads();
    int victim = s_bi[0];
    for (int t = threadIdx.x; t < d; t += blockDim.x) C[(size_t)c * d + t] = P[(size_t)victim * d + t];
    __syncthreads();
  }
  if (s_flag) { /* reserved */ }
}

// ---------------------------------------------------------------------------
// phase 4: Lloyd update (clustering.py:86-95): counts, fp64 per-cluster sums
// in ascending point order (np.bincount(weights=...)), divide -> fp32,
// normalize, repair.  final=1: only counts + repair (clustering.py:99-100).
// grid = n_segments, block = 512, dyn smem = (2k+1) ints
// ---------------------------------------------------------------------------
__global__ void km_update_kernel(const SegDesc* __restrict__ segs, const float* __restrict__ P_all,
                                 float* __restrict__ C_all, int32_t* __restrict__ A_all,
                                 int32_t* __restrict__ perm_all, float* __restrict__ sims_all,
                                 int d, int final_pass) {
  const SegDesc sg = segs[blockIdx.x];
  if (sg.k <= 1) return;
  extern __shared__ int smi[];
  int* cnt = smi;            // k+1
  int* cursor = smi + sg.k + 1;  // k
  const float* P = P_all + (size_t)sg.p_off * d;
  float* C = C_all + (size_t)sg.c_off * d;
  int32_t* A = A_all + sg.p_off;
  int32_t* perm = perm_all + sg.p_off;
  float* sims = sims_all + sg.p_off;
  stable_bucket(A, sg.L, sg.k, cnt, cursor, perm);
  // counts[c] = cnt[c+1]-cnt[c]; keep in cursor[] (reused) for repair
  for (int c = threadIdx.x; c < sg.k; c += blockDim.x) cursor[c] = cnt[c + 1] - cnt[c];
  __syncthreads();
  if (!final_pass) {
    for (int idx = threadIdx.x; idx < sg.k * d; idx += blockDim.x) {
      int c = idx / d, t = idx % d;
      int b = cnt[c], e = cnt[c + 1];
      if (e > b) {
        // sequential fp64 sum in member order (bincount, clustering.py:87-91);
        // eight members' loads issued ahead of their adds
        double s = 0.0;
        int j = b;
        for (; j + 8 <= e; j += 8) {
          float pv[8];
#pragma unroll
          for (int q = 0; q < 8; q++) pv[q] = P[(size_t)perm[j + q] * d + t];
#pragma unroll
          for (int q = 0; q < 8; q++) s = __dadd_rn(s, (double)pv[q]);
        }
        for (; j < e; j++) s = __dadd_rn(s, (double)P[(size_t)perm[j] * d + t]);
        C[(size_t)c * d + t] = __double2float_rn(__ddiv_rn(s, (double)(e - b)));
      }
    }
    __syncthreads();
    if (d == 32 || d == 64 || d == 128) {
      // warp per centroid row, coalesced; the 8 pairwise-norm chains on lanes 0-7
      // (same bits as row_norm_f32, see km_prep_v2_kernel)
      float* sq = reinterpret_cast<float*>(cursor + sg.k) + (threadIdx.x >> 5) * d;
      const int lane = threadIdx.x & 31, epl = d >> 5;
      for (int c = threadIdx.x >> 5; c < sg.k; c += blockDim.x >> 5) {
        float* row = C + (size_t)c * d;
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (e < epl) { x[e] = row[lane * epl + e]; sq[lane * epl + e] = __fmul_rn(x[e], x[e]); }
        __syncwarp();
        float r = 0.f;
        if (lane < 8) {
          r = sq[lane];
          for (int j = 8; j < d; j += 8) r = __fadd_rn(r, sq[j + lane]);
        }
        r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));
        r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 2));
        r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 4));
        const float nr = __fsqrt_rn(__shfl_sync(0xffffffffu, r, 0));
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (e < epl) row[lane * epl + e] = nr != 0.f ? __fdiv_rn(x[e], nr) : (lane * epl + e == 0 ? 1.f : 0.f);
      }
    } else {
      for (int c = threadIdx.x; c < sg.k; c += blockDim.x) {
        float* row = C + (size_t)c * d;
        float nr = row_norm_f32(row, d);
        if (nr != 0.0f) {
          for (int t = 0; t < d; t++) row[t] = __fdiv_rn(row[t], nr);
        } else {
          for (int t = 0; t < d; t++) row[t] = 0.f;
          row[0] = 1.0f;
        }
      }
    }
    __syncthreads();
  }
  repair_empty(P, sg.L, d, A, C, sg.k, cursor, sims, nullptr);
}

// ---------------------------------------------------------------------------
// phase 5: finalize_cluster (index.py:43-58) + pack the cluster-private store
// (store.py:69-90).  fp64 mean of the raw member keys and fp64 value sums in
// ascending token order; members written cluster-contiguously to the store.
// grid = n_segments, block = 256, dyn smem = (2k+1) ints
// ---------------------------------------------------------------------------
template <typename T>
__global__ void km_finalize_kernel(const SegDesc* __restrict__ segs, const int32_t* __restrict__ A_all,
                                   int32_t* __restrict__ perm_all, IndexView ix, int d,
                                   int* __restrict__ status, int fin_smem_perm) {
  const SegDesc sg = segs[blockIdx.x];
  extern __shared__ int smi[];
  int* cnt = smi;
  int* cursor = smi + sg.k + 1;
  int32_t* perm = perm_all + sg.p_off;
  if (sg.k <= 1) {
    // k == 1 shortcut (clustering.py:79-80): everything in cluster 0
    if (threadIdx.x == 0) { cnt[0] = 0; cnt[1] = sg.L; }
    for (int i = threadIdx.x; i < sg.L; i += blockDim.x) perm[i] = i;
    __syncthreads();
  } else {
    stable_bucket(A_all + sg.p_off, sg.L, sg.k, cnt, cursor, perm);
  }
  const size_t u = sg.unit;
  T* sk = (T*)ix.store_k + u * ix.s_cap * d;
  T* sv = (T*)ix.store_v + u * ix.s_cap * d;
  int32_t* stok = ix.store_tok + u * ix.s_cap;
  for (int c = threadIdx.x; c < sg.k; c += blockDim.x) {
    int s = cnt[c + 1] - cnt[c];
    if (s == 0) set_status(status, kErrEmptyCluster);
    size_t cid = (size_t)sg.cid_base + c;
    ix.cl_off[u * ix.m_cap + cid] = sg.row_base + cnt[c];
    ix.cl_size[u * ix.m_cap + cid] = s;
  }
  for (int j = threadIdx.x; j < sg.L; j += blockDim.x) stok[sg.row_base + j] = sg.tok_base + perm[j];
  const bool swz = kv_swizzled<T>(d);
  for (size_t idx = threadIdx.x; idx < (size_t)sg.L * d; idx += blockDim.x) {
    size_t j = idx / d, t = idx % d;
    size_t src = (size_t)perm[j] * sg.key_stride + t;
    const size_t row = (size_t)sg.row_base + j;
    const size_t col = swz ? (size_t)swz_col((int)t, (long long)row) : t;
    sk[row * d + col] = KV<T>::from_f(sg.keys[src]);
    sv[row * d + col] = KV<T>::from_f(sg.values[src]);
  }
  // member lists in shared memory when they fit (dynamic smem past cnt / cursor)
  const int32_t* mem = perm;
  if (fin_smem_perm) {
    int* sp = smi + 2 * sg.k + 1;
    __syncthreads();  // perm complete (stable_bucket)
    for (int j = threadIdx.x; j < sg.L; j += blockDim.x) sp[j] = perm[j];
    __syncthreads();
    mem = sp;
  }
  for (int idx = threadIdx.x; idx < sg.k * d; idx += blockDim.x) {
    int c = idx / d, t = idx % d;
    int b = cnt[c], e = cnt[c + 1];
    double ks = 0.0, vs = 0.0;
    // the reference's sequential fp64 sums in member order; eight members'
    // loads issued ahead of their adds (the loop is otherwise latency-bound)
    int j = b;
    for (; j + 8 <= e; j += 8) {
      float kv[8], vv[8];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const size_t src = (size_t)mem[j + q] * sg.key_stride + t;
        kv[q] = sg.keys[src];
        vv[q] = sg.values[src];
      }
#pragma unroll
      for (int q = 0; q < 8; q++) {
        ks = __dadd_rn(ks, (double)kv[q]);
        vs = __dadd_rn(vs, (double)vv[q]);
      }
    }
    for (; j < e; j++) {
      size_t src = (size_t)mem[j] * sg.key_stride + t;
      ks = __dadd_rn(ks, (double)sg.keys[src]);
      vs = __dadd_rn(vs, (double)sg.values[src]);
    }
    double mean = e > b ? __ddiv_rn(ks, (double)(e - b)) : 0.0;
    size_t row = u * ix.m_cap + (size_t)sg.cid_base + c;
    ix.C64[row * d + t] = mean;
    ix.C32[row * d + t] = __double2float_rn(mean);
    ix.VS32[row * d + t] = __double2float_rn(vs);
    if (ix.VS64) ix.VS64[row * d + t] = vs;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < sg.k; c += blockDim.x) {
    size_t row = u * ix.m_cap + (size_t)sg.cid_base + c;
    const float* cr = ix.C32 + row * d;
    float s = 0.f;
    for (int t = 0; t < d; t++) s = fmaf(cr[t], cr[t], s);
    ix.Cnorm[row] = sqrtf(s);
    // the unit's max centroid norm: the scan's error bound (score_error_bound_v2)
    if (ix.Cmax) atomicMax(reinterpret_cast<int*>(ix.Cmax + u), __float_as_int(sqrtf(s)));  // >= 0
  }
}

template __global__ void km_finalize_kernel<float>(const SegDesc*, const int32_t*, int32_t*, IndexView, int, int*, int);
template __global__ void km_finalize_kernel<__nv_bfloat16>(const SegDesc*, const int32_t*, int32_t*, IndexView, int, int*, int);

}  // namespace wk
