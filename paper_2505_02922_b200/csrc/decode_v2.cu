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
