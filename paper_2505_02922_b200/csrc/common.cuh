// common.cuh -- shared device helpers for the wave-index kernels (sm_100a).
//
// Exactness-critical arithmetic uses explicit round-to-nearest intrinsics
// (__fmaf_rn/__fadd_rn/__fmul_rn/__fdiv_rn, __fma_rn/...) so nvcc can neither
// contract nor reorder it; these restate the numpy/OpenBLAS evaluation orders
// the reference (tierkv) runs with -- see DESIGN.md "Numerics recipes".
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define WK_DEVINL __device__ __forceinline__

namespace wk {

// status word codes written by kernels (mapped to IntegrityError by the host)
enum : int {
  kOk = 0,
  kErrBandOverflow = 1,   // exact-rescoring band exceeded its scratch capacity
  kErrEmptyCluster = 2,   // finalize saw an empty cluster
  kErrCapacity = 3,       // device block cache over capacity
  kErrUnion = 4,          // union list overflow
  kErrUnknownCluster = 5, // cache access to an unregistered cluster
  kErrEmptyMerge = 6,     // all partials empty (attention.py:117-119)
  kErrSteadyFull = 7,     // decode append beyond the steady buffer capacity
};

WK_DEVINL void set_status(int* status, int code) {
  if (status) atomicCAS(status, 0, code);
}

// ---- storage type helpers ---------------------------------------------------
template <typename T> struct KV;
template <> struct KV<float> {
  static WK_DEVINL float to_f(float x) { return x; }
  static WK_DEVINL float from_f(float x) { return x; }
};
template <> struct KV<__nv_bfloat16> {
  static WK_DEVINL float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static WK_DEVINL __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// bf16 K/V rows of the fast path (d in {64, 128}) are stored swizzled: the
// 16-byte piece c of row r (8 elements) sits at piece c ^ (r & 7) of the row,
// r = the row's index in its array (cluster store, steady buffer, slot arena).
// A contiguous run of rows copied as one block then reads conflict-free with
// ldmatrix (attend_v5).  swz_col maps a logical element index to its slot.
__host__ __device__ __forceinline__ int swz_col(int t, long long row) {
  return ((((t >> 3) ^ (int)(row & 7)) << 3) | (t & 7));
}
template <typename T>
__host__ __device__ __forceinline__ bool kv_swizzled(int d) {
  return sizeof(T) == 2 && (d == 64 || d == 128);
}

// order-preserving float <-> uint32 (ascending)
WK_DEVINL uint32_t f2u_ord(float f) {
  uint32_t u = __float_as_uint(f);
  if (f == 0.0f) u = 0u;  // -0.0 == +0.0 (lexsort semantics, test_index.py:63-70)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
WK_DEVINL float u2f_ord(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// ---- numpy PCG64 (XSL-RR 128/64) + Generator draws --------------------------
struct Pcg64 {
  uint64_t hi, lo, ihi, ilo;
  int has32;
  uint32_t u32;
};
WK_DEVINL uint64_t pcg_next64(Pcg64& g) {
  // state = state * MULT + inc  (128-bit)
  const uint64_t MH = 2549297995355413924ULL, ML = 4865540595714422341ULL;
  uint64_t lo = g.lo * ML;
  uint64_t hi = __umul64hi(g.lo, ML) + g.lo * MH + g.hi * ML;
  uint64_t nlo = lo + g.ilo;
  uint64_t carry = nlo < lo ? 1ULL : 0ULL;
  g.lo = nlo;
  g.hi = hi + g.ihi + carry;
  uint64_t v = g.hi ^ g.lo;
  unsigned rot = (unsigned)(g.hi >> 58);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}
WK_DEVINL uint32_t pcg_next32(Pcg64& g) {
  if (g.has32) { g.has32 = 0; return g.u32; }
  uint64_t nx = pcg_next64(g);
  g.has32 = 1;
  g.u32 = (uint32_t)(nx >> 32);
  return (uint32_t)nx;
}
WK_DEVINL double pcg_next_double(Pcg64& g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}
// Generator.integers(n) for n <= 2^32 (buffered_bounded_lemire_uint32)
WK_DEVINL int64_t pcg_integers(Pcg64& g, int64_t n) {
  uint64_t rng = (uint64_t)(n - 1);
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return (int64_t)pcg_next32(g);
  uint32_t r32 = (uint32_t)rng, rng_excl = r32 + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * rng_excl;
  uint32_t left = (uint32_t)m;
  if (left < rng_excl) {
    uint32_t thr = (uint32_t)((0xFFFFFFFFu - r32) % rng_excl);
    while (left < thr) {
      m = (uint64_t)pcg_next32(g) * rng_excl;
      left = (uint32_t)m;
    }
  }
  return (int64_t)(m >> 32);
}

// ---- OpenBLAS sgemv_t recipe (clustering.py:33,42) -------------------------
// Row class of row i in an n-row sgemv/dgemv with `threads` chunks:
// 0 = main (group of 4), 1 = trailing pair, 2 = odd trailing row.
WK_DEVINL int gemv_row_class(int i, int n, int d, int threads) {
  int r0 = 0, r1 = n;
  if ((long long)n * d >= 460800LL && threads > 1) {
    int s = 0, rem = n, t = threads;
    while (rem > 0) {
      int w = (rem + t - 1) / t;
      if (w < 4) w = 4;
      if (rem < w) w = rem;
      if (i < s + w) { r0 = s; r1 = s + w; break; }
      s += w; rem -= w; t--;
      if (t < 1) t = 1;
    }
  }
  int len = r1 - r0, off = i - r0;
  int main_end = (len >> 2) << 2;
  if (off < main_end) return 0;
  if ((len & 2) && off < main_end + 2) return 1;
  return 2;
}

template <typename RowT>
WK_DEVINL float sgemv_row(const RowT* a, const float* x, int d, int cls) {
  if (cls == 0) {
    float c[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < d; t++) c[t & 7] = __fmaf_rn((float)a[t], x[t], c[t & 7]);
    float s0 = __fadd_rn(c[0], c[4]), s1 = __fadd_rn(c[1], c[5]);
    float s2 = __fadd_rn(c[2], c[6]), s3 = __fadd_rn(c[3], c[7]);
    return __fadd_rn(0.f, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
  } else if (cls == 1) {
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < d; t++) c[t & 3] = __fadd_rn(c[t & 3], __fmul_rn((float)a[t], x[t]));
    return __fadd_rn(0.f, __fadd_rn(__fadd_rn(c[0], c[1]), __fadd_rn(c[2], c[3])));
  } else {
    float c[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < d; t++) c[t & 7] = __fadd_rn(c[t & 7], __fmul_rn((float)a[t], x[t]));
    float s0 = __fadd_rn(c[0], c[4]), s1 = __fadd_rn(c[1], c[5]);
    float s2 = __fadd_rn(c[2], c[6]), s3 = __fadd_rn(c[3], c[7]);
    return __fadd_rn(0.f, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
  }
}

// ---- OpenBLAS dgemv_t recipe (index.py:74, metrics.py:14) ------------------
WK_DEVINL double dgemv_row(const double* a, const double* x, int d, int cls) {
  if (cls == 0) {
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int t = 0; t < d; t += 4) {
      c0 = __fma_rn(a[t], x[t], c0);
      if (t + 1 < d) c1 = __fma_rn(a[t + 1], x[t + 1], c1);
      if (t + 2 < d) c2 = __fma_rn(a[t + 2], x[t + 2], c2);
      if (t + 3 < d) c3 = __fma_rn(a[t + 3], x[t + 3], c3);
    }
    return __dadd_rn(0.0, __dadd_rn(__dadd_rn(c0, c2), __dadd_rn(c1, c3)));
  } else if (cls == 1) {
    double c0 = 0, c1 = 0;
    for (int t = 0; t < d; t++) {
      double p = __dmul_rn(a[t], x[t]);
      if (t & 1) c1 = __dadd_rn(c1, p); else c0 = __dadd_rn(c0, p);
    }
    return __dadd_rn(0.0, __dadd_rn(c0, c1));
  } else {
    double c[4] = {0, 0, 0, 0};
    for (int t = 0; t < d; t++) c[t & 3] = __dadd_rn(c[t & 3], __dmul_rn(a[t], x[t]));
    return __dadd_rn(0.0, __dadd_rn(__dadd_rn(c[0], c[2]), __dadd_rn(c[1], c[3])));
  }
}

// ---- numpy pairwise sum of squares + sqrt: np.linalg.norm(axis=1) ----------
// (clustering.py:18; numpy loops_utils.h.src FLOAT_pairwise_sum)
template <typename Get>
WK_DEVINL float pairwise_sum_f32(Get get, long long off, long long n) {
  // iterative form of the recursion for n <= 1024 (d <= 1024)
  if (n < 8) {
    float r = 0.f;
    for (long long i = 0; i < n; i++) r = __fadd_rn(r, get(off + i));
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; j++) r[j] = get(off + j);
    long long i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], get(off + i + j));
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __fadd_rn(res, get(off + i));
    return res;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  // one level of recursion handles d <= 256 (both halves <= 128)
  float a, b;
  {
    long long nn = n2;
    float r[8];
    for (int j = 0; j < 8; j++) r[j] = get(off + j);
    long long i;
    for (i = 8; i < nn - (nn % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], get(off + i + j));
    a = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                  __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < nn; i++) a = __fadd_rn(a, get(off + i));
  }
  {
    long long o2 = off + n2, nn = n - n2;
    float r[8];
    for (int j = 0; j < 8; j++) r[j] = get(o2 + j);
    long long i;
    for (i = 8; i < nn - (nn % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], get(o2 + i + j));
    b = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                  __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < nn; i++) b = __fadd_rn(b, get(o2 + i));
  }
  return __fadd_rn(a, b);
}

WK_DEVINL float row_norm_f32(const float* x, int d) {
  auto get = [x](long long i) { return __fmul_rn(x[i], x[i]); };
  return __fsqrt_rn(pairwise_sum_f32(get, 0, d));
}

// np.einsum("ij,ij->i") fp32 (clustering.py:55)
WK_DEVINL float einsum_row(const float* x, const float* y, int d) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int c = d, t = 0;
  for (; c >= 16; c -= 16, t += 16)
    for (int q = 3; q >= 0; q--)
      for (int l = 0; l < 4; l++)
        acc[l] = __fadd_rn(acc[l], __fmul_rn(x[t + 4 * q + l], y[t + 4 * q + l]));
  for (; c > 0; c -= 4, t += 4)
    for (int l = 0; l < 4; l++) {
      float xv = (l < c) ? x[t + l] : 0.f, yv = (l < c) ? y[t + l] : 0.f;
      acc[l] = __fadd_rn(acc[l], __fmul_rn(xv, yv));
    }
  return __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
}

// Rigorous bound on |s' - s| for every centroid row: s' = the scoring kernel's
// score, s = the reference's fp64 dgemv.  fp64-accumulated scores (score_v3):
// C32 rounding + fp32 store = 2^-23 |q||C|; fp32-accumulated scores (v1):
// additionally gamma_d = d 2^-24 / (1 - d 2^-24).  1.25x margin covers the fp32
// evaluation of |q| and max|C|.
WK_DEVINL double score_error_bound(double qnorm2, double cmax, int d, bool fp64_scores) {
  const double uu = 5.9604644775390625e-08;  // 2^-24
  const double gam = fp64_scores ? 0.0 : (double)d * uu / (1.0 - (double)d * uu);
  return 1.25 * (gam + 2.0 * uu + 1e-13) * sqrt(qnorm2) * cmax;
}

// Bound for the scoring modes of wk_zone_params.score_mode:
//  0: fp32 FMA scan of C32           gamma_d + C32 rounding + store
//  1: fp64-accumulated scan of C32   C32 rounding + fp32 store (2^-23)
WK_DEVINL double score_error_bound_v2(double qnorm2, double cmax, int d, int mode) {
  return score_error_bound(qnorm2, cmax, d, mode == 1);
}

// Zone bitmaps (per-head R / E sets, select_v6 -> unions -> cache_v2) use a
// permuted layout so one warp ballot over 32 lanes x float4 covers a word:
// cluster c <-> word ((c >> 7) << 2) | (c & 3), bit (c >> 2) & 31.
// Words per unit: 4 * ceil(m / 128).
// programmatic dependent launch: the decode kernels are launched with the
// programmatic-serialization attribute and wait here for the preceding grid
// (completion and memory visibility; a no-op without the attribute).  They
// never trigger early (griddepcontrol.launch_dependents): measured, early
// triggers let waiting dependents take SM slots from the primary's tail
// (-5%), while the implicit trigger at exit hides the launch latency (+4%).
WK_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef WK_TRIG_MASK
#define WK_TRIG_MASK 0  // tuning experiments: bit k = early trigger in kernel k (score, select, attend, merge)
#endif
template <int BIT>
WK_DEVINL void pdl_trigger() {
  if (WK_TRIG_MASK & BIT) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// distributed shared memory (thread-block clusters): 32-bit shared::cluster
// address of `p` (a shared-memory object of this CTA) in CTA `rank` of the
// cluster -- all CTAs of a kernel share the layout -- and a 32-bit load.
WK_DEVINL uint32_t dsmem_addr(const void* p, int rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
WK_DEVINL uint32_t dsmem_ld_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

__host__ __device__ __forceinline__ int zb_word(int c) { return ((c >> 7) << 2) | (c & 3); }
__host__ __device__ __forceinline__ int zb_bit(int c) { return (c >> 2) & 31; }
__host__ __device__ __forceinline__ int zb_cluster(int w, int b) { return ((w >> 2) << 7) | (b << 2) | (w & 3); }
__host__ __device__ __forceinline__ int zb_words(int m) { return ((m + 127) >> 7) << 2; }

WK_DEVINL float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
WK_DEVINL float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace wk

// ---- TMA bulk copies (cp.async.bulk, global -> shared) + mbarriers ---------
namespace wk {
WK_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
WK_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
WK_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
WK_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
WK_DEVINL void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D bulk copy of `bytes` (multiple of 16, 16B-aligned) completing on `bar`
WK_DEVINL void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
WK_DEVINL void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
WK_DEVINL void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
}  // namespace wk
