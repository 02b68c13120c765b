/* wk_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see wk_oracle.h).
 *
 * Plain-C restatement of tierkv (reference pkg/src/tierkv).  Each function
 * cites the reference file:line it restates.  Compile with
 *   -O3 -ffp-contract=off -mavx2 -mfma   (no -ffast-math: order matters)
 */
#include "wk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ========================================================================
 * numpy PCG64 (numpy/random/src/pcg64/pcg64.h: pcg64_random_r, XSL-RR) and
 * Generator draws (distributions.c: buffered_bounded_lemire_uint32,
 * next_double).  Used by clustering.py:81 (default_rng(SeedSequence)).
 * ======================================================================*/
static const u128 PCG_MULT = (((u128)2549297995355413924ULL) << 64) | 4865540595714422341ULL;

void wko_rng_init(wko_rng* g, const uint64_t w[4]) {
  g->st_hi = w[0]; g->st_lo = w[1]; g->inc_hi = w[2]; g->inc_lo = w[3];
  g->has32 = 0; g->u32 = 0;
}

uint64_t wko_next64(wko_rng* g) {
  u128 s = (((u128)g->st_hi) << 64) | g->st_lo;
  u128 inc = (((u128)g->inc_hi) << 64) | g->inc_lo;
  s = s * PCG_MULT + inc;
  g->st_hi = (uint64_t)(s >> 64); g->st_lo = (uint64_t)s;
  uint64_t v = g->st_hi ^ g->st_lo;
  unsigned rot = (unsigned)(s >> 122);
  return (v >> rot) | (v << ((-rot) & 63));
}

uint32_t wko_next32(wko_rng* g) {
  if (g->has32) { g->has32 = 0; return g->u32; }
  uint64_t nx = wko_next64(g);
  g->has32 = 1; g->u32 = (uint32_t)(nx >> 32);
  return (uint32_t)(nx & 0xffffffffULL);
}

double wko_next_double(wko_rng* g) {
  return (double)(wko_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

int64_t wko_integers(wko_rng* g, int64_t n) {
  uint64_t rng = (uint64_t)(n - 1);
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return (int64_t)wko_next32(g);
  uint32_t r32 = (uint32_t)rng, rng_excl = r32 + 1;
  uint64_t m = (uint64_t)wko_next32(g) * rng_excl;
  uint32_t leftover = (uint32_t)(m & 0xFFFFFFFFULL);
  if (leftover < rng_excl) {
    uint32_t threshold = (uint32_t)((UINT32_MAX - r32) % rng_excl);
    while (leftover < threshold) {
      m = (uint64_t)wko_next32(g) * rng_excl;
      leftover = (uint32_t)(m & 0xFFFFFFFFULL);
    }
  }
  return (int64_t)(m >> 32);
}

/* ========================================================================
 * sgemm, points @ centroids.T (clustering.py:85,96).  OpenBLAS 0.3.30 on
 * SkylakeX: small-matrix TN kernel when n*k <= 1200 and d >= 32 (16-lane
 * FMA accumulator; adjacent-pair lane tree, except the (n&~3, k&~3) corner
 * block which uses _mm512_reduce_add_ps order); otherwise every output is a
 * sequential fp32 FMA chain over t.
 * ======================================================================*/
static float lane_tree(float* a, int corner) {
  /* 16 lanes; combine lanes differing in bit b, bits in the given order */
  static const int order_adj[4] = {0, 1, 2, 3}, order_red[4] = {3, 2, 1, 0};
  const int* ord = corner ? order_red : order_adj;
  for (int lev = 0; lev < 4; lev++) {
    int b = 1 << ord[lev];
    for (int l = 0; l < 16; l++)
      if (!(l & b)) a[l] = a[l] + a[l | b];
  }
  return a[0];
}

void wko_sgemm_nt(const float* P, const float* C, int n, int k, int d, float* out) {
  if ((long)n * k <= 1200 && d >= 32 && k > 1) {
    int n4 = n & ~3, k4 = k & ~3;
    for (int i = 0; i < n; i++)
      for (int c = 0; c < k; c++) {
        float a[16] = {0};
        for (int t = 0; t < d; t++) a[t & 15] = fmaf(P[(long)i * d + t], C[(long)c * d + t], a[t & 15]);
        out[(long)i * k + c] = lane_tree(a, i >= n4 && c >= k4);
      }
    return;
  }
  /* sequential chain; vectorised across centroids (each lane its own chain) */
  float* CT = (float*)malloc(sizeof(float) * (size_t)d * k);
  for (int c = 0; c < k; c++)
    for (int t = 0; t < d; t++) CT[(long)t * k + c] = C[(long)c * d + t];
  float* acc = (float*)malloc(sizeof(float) * (size_t)k);
  for (int i = 0; i < n; i++) {
    const float* p = P + (long)i * d;
    for (int c = 0; c < k; c++) acc[c] = 0.f;
    for (int t = 0; t < d; t++) {
      const float pt = p[t];
      const float* ct = CT + (long)t * k;
      for (int c = 0; c < k; c++) acc[c] = fmaf(pt, ct[c], acc[c]);
    }
    memcpy(out + (long)i * k, acc, sizeof(float) * (size_t)k);
  }
  free(acc);
  free(CT);
}

/* ========================================================================
 * sgemv_t (clustering.py:33,42): per thread chunk, rows in groups of 4 use
 * 8 FMA accumulators a[t%8] then (a0+a4,a1+a5,a2+a6,a3+a7) -> (s0+s1)+(s2+s3);
 * a trailing pair uses 4 unfused accumulators -> (a0+a1)+(a2+a3); an odd
 * trailing row 8 unfused accumulators reduced like the main rows.  Chunks:
 * one if n*d < 460800 else `threads` chunks of ceil(rem/threads_left).
 * Modelled domain: d % 8 == 0, d >= 16, n >= 2 (d<16 uses other kernels).
 * ======================================================================*/
static float sv_main(const float* a, const float* x, int d) {
  float c[8] = {0};
  for (int t = 0; t < d; t++) c[t & 7] = fmaf(a[t], x[t], c[t & 7]);
  float s0 = c[0] + c[4], s1 = c[1] + c[5], s2 = c[2] + c[6], s3 = c[3] + c[7];
  return (s0 + s1) + (s2 + s3);
}
static float sv_r2(const float* a, const float* x, int d) {
  float c[4] = {0};
  for (int t = 0; t < d; t++) { float p = a[t] * x[t]; c[t & 3] = c[t & 3] + p; }
  return (c[0] + c[1]) + (c[2] + c[3]);
}
static float sv_r1(const float* a, const float* x, int d) {
  float c[8] = {0};
  for (int t = 0; t < d; t++) { float p = a[t] * x[t]; c[t & 7] = c[t & 7] + p; }
  float s0 = c[0] + c[4], s1 = c[1] + c[5], s2 = c[2] + c[6], s3 = c[3] + c[7];
  return (s0 + s1) + (s2 + s3);
}
static void sv_chunk(const float* A, const float* x, int r0, int r1, int d, float* y) {
  int n = r1 - r0, i = r0;
  for (int g = 0; g < (n >> 2); g++)
    for (int j = 0; j < 4; j++, i++) y[i] = 0.f + sv_main(A + (long)i * d, x, d);
  if (n & 2)
    for (int j = 0; j < 2; j++, i++) y[i] = 0.f + sv_r2(A + (long)i * d, x, d);
  if (n & 1) { y[i] = 0.f + sv_r1(A + (long)i * d, x, d); i++; }
}
void wko_sgemv(const float* A, const float* x, int n, int d, int threads, float* y) {
  if ((long)n * d < 460800L || threads <= 1) { sv_chunk(A, x, 0, n, d, y); return; }
  int s = 0, rem = n, t = threads;
  while (rem > 0) {
    int w = (rem + t - 1) / t;
    if (w < 4) w = 4;
    if (rem < w) w = rem;
    sv_chunk(A, x, s, s + w, d, y);
    s += w; rem -= w; t--;
    if (t < 1) t = 1;
  }
}

/* ========================================================================
 * dgemv_t (index.py:74, metrics.py:14): rows in groups of 4 use 4 FMA
 * accumulators a[t%4] -> (a0+a2)+(a1+a3); a trailing pair 2 unfused
 * accumulators -> a0+a1; an odd trailing row 4 unfused -> (a0+a2)+(a1+a3).
 * Same chunking rule.  Modelled domain: d % 4 == 0, n >= 2.
 * ======================================================================*/
static double dv_main(const double* a, const double* x, int d) {
  double c[4] = {0};
  for (int t = 0; t < d; t++) c[t & 3] = fma(a[t], x[t], c[t & 3]);
  return (c[0] + c[2]) + (c[1] + c[3]);
}
static double dv_r2(const double* a, const double* x, int d) {
  double c[2] = {0};
  for (int t = 0; t < d; t++) { double p = a[t] * x[t]; c[t & 1] = c[t & 1] + p; }
  return c[0] + c[1];
}
static double dv_r1(const double* a, const double* x, int d) {
  double c[4] = {0};
  for (int t = 0; t < d; t++) { double p = a[t] * x[t]; c[t & 3] = c[t & 3] + p; }
  return (c[0] + c[2]) + (c[1] + c[3]);
}
static void dv_chunk(const double* A, const double* x, int r0, int r1, int d, double* y) {
  int n = r1 - r0, i = r0;
  for (int g = 0; g < (n >> 2); g++)
    for (int j = 0; j < 4; j++, i++) y[i] = 0.0 + dv_main(A + (long)i * d, x, d);
  if (n & 2)
    for (int j = 0; j < 2; j++, i++) y[i] = 0.0 + dv_r2(A + (long)i * d, x, d);
  if (n & 1) { y[i] = 0.0 + dv_r1(A + (long)i * d, x, d); i++; }
}
void wko_dgemv(const double* A, const double* x, int n, int d, int threads, double* y) {
  if ((long)n * d < 460800L || threads <= 1) { dv_chunk(A, x, 0, n, d, y); return; }
  int s = 0, rem = n, t = threads;
  while (rem > 0) {
    int w = (rem + t - 1) / t;
    if (w < 4) w = 4;
    if (rem < w) w = rem;
    dv_chunk(A, x, s, s + w, d, y);
    s += w; rem -= w; t--;
    if (t < 1) t = 1;
  }
}

/* ========================================================================
 * numpy pairwise summation (loops_utils.h.src FLOAT_pairwise_sum), used by
 * np.linalg.norm(axis=1) (clustering.py:18) on x*x.
 * ======================================================================*/
static float pairwise_f32(const float* a, long n) {
  if (n < 8) {
    float r = 0.f;
    for (long i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    long i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  long n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_f32(a, n2) + pairwise_f32(a + n2, n - n2);
}

void wko_row_norms(const float* x, int n, int d, float* out) {
  float* sq = (float*)malloc(sizeof(float) * (size_t)d);
  for (int i = 0; i < n; i++) {
    for (int t = 0; t < d; t++) { float v = x[(long)i * d + t]; sq[t] = v * v; }
    out[i] = sqrtf(pairwise_f32(sq, d));
  }
  free(sq);
}

/* np.einsum("ij,ij->i") fp32 (clustering.py:55): SSE baseline sum-of-products,
 * 4 lanes, 4-vector unroll accumulated last vector first, unfused mul+add,
 * reduce (l0+l1)+(l2+l3). */
float wko_einsum_row(const float* x, const float* y, int d) {
  float acc[4] = {0, 0, 0, 0};
  int c = d, t = 0;
  for (; c >= 16; c -= 16, t += 16)
    for (int q = 3; q >= 0; q--)
      for (int l = 0; l < 4; l++) { float p = x[t + 4 * q + l] * y[t + 4 * q + l]; acc[l] = acc[l] + p; }
  for (; c > 0; c -= 4, t += 4)
    for (int l = 0; l < 4; l++) {
      float xv = (l < c) ? x[t + l] : 0.f, yv = (l < c) ? y[t + l] : 0.f;
      float p = xv * yv;
      acc[l] = acc[l] + p;
    }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

/* ========================================================================
 * clustering.py
 * ======================================================================*/
/* _normalize_rows, clustering.py:16-23 */
static void normalize_rows(float* x, int n, int d) {
  float* nr = (float*)malloc(sizeof(float) * (size_t)n);
  wko_row_norms(x, n, d, nr);
  for (int i = 0; i < n; i++) {
    float* r = x + (long)i * d;
    if (nr[i] != 0.0f) {
      for (int t = 0; t < d; t++) r[t] = r[t] / nr[i];
    } else {
      for (int t = 0; t < d; t++) r[t] = 0.f;
      r[0] = 1.0f;
    }
  }
  free(nr);
}

/* _seed_centroids, clustering.py:26-43 */
static void seed_centroids(const float* P, int n, int d, int k, wko_rng* g, int threads, float* C) {
  float* md = (float*)malloc(sizeof(float) * (size_t)n);
  float* dots = (float*)malloc(sizeof(float) * (size_t)n);
  float* cdf = (float*)malloc(sizeof(float) * (size_t)n);
  int64_t first = wko_integers(g, n);
  memcpy(C, P + first * d, sizeof(float) * (size_t)d);
  wko_sgemv(P, C, n, d, threads, dots);
  for (int i = 0; i < n; i++) { float v = 1.0f - dots[i]; md[i] = v < 0.f ? 0.f : v; }
  for (int c = 1; c < k; c++) {
    float s = 0.f;
    for (int i = 0; i < n; i++) { s = (i == 0) ? md[0] : s + md[i]; cdf[i] = s; }
    int64_t idx;
    float last = cdf[n - 1];
    if (last <= 0.0f) {
      idx = wko_integers(g, n);
    } else {
      float u = (float)wko_next_double(g);
      float thr = u * last;
      /* searchsorted side='right': number of entries <= thr */
      int lo = 0, hi = n;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (cdf[mid] <= thr) lo = mid + 1; else hi = mid; }
      idx = lo;
      if (idx > n - 1) idx = n - 1;
    }
    memcpy(C + (long)c * d, P + idx * d, sizeof(float) * (size_t)d);
    wko_sgemv(P, C + (long)c * d, n, d, threads, dots);
    for (int i = 0; i < n; i++) {
      float v = 1.0f - dots[i];
      v = v < 0.f ? 0.f : v;
      if (!(md[i] <= v)) md[i] = v;
    }
  }
  free(md); free(dots); free(cdf);
}

/* argmax(points @ centroids.T, axis=1), first index on ties */
static void assign_argmax(const float* P, int n, const float* C, int k, int d, int64_t* a) {
  /* row-blocked to bound the score buffer */
  const int RB = 256;
  float* S = (float*)malloc(sizeof(float) * (size_t)RB * k);
  for (int i0 = 0; i0 < n; i0 += RB) {
    int nb = n - i0 < RB ? n - i0 : RB;
    if ((long)n * k <= 1200 && d >= 32 && k > 1) {
      /* small kernel depends on the full (n,k) shape: evaluate whole */
      float* Sf = (float*)malloc(sizeof(float) * (size_t)n * k);
      wko_sgemm_nt(P, C, n, k, d, Sf);
      for (int i = 0; i < n; i++) {
        int best = 0;
        for (int c = 1; c < k; c++) if (Sf[(long)i * k + c] > Sf[(long)i * k + best]) best = c;
        a[i] = best;
      }
      free(Sf);
      break;
    }
    wko_sgemm_nt(P + (long)i0 * d, C, nb, k, d, S);
    for (int i = 0; i < nb; i++) {
      const float* s = S + (long)i * k;
      int best = 0;
      for (int c = 1; c < k; c++) if (s[c] > s[best]) best = c;
      a[i0 + i] = best;
    }
  }
  free(S);
}

/* _repair_empty, clustering.py:46-63 */
static void repair_empty(const float* P, int n, int d, int64_t* a, float* C, int k, int64_t* counts) {
  float* sims = NULL;
  int* empties = (int*)malloc(sizeof(int) * (size_t)k);
  int ne = 0;
  for (int c = 0; c < k; c++) if (counts[c] == 0) empties[ne++] = c;
  for (int q = 0; q < ne; q++) {
    int c = empties[q];
    if (!sims) {
      sims = (float*)malloc(sizeof(float) * (size_t)n);
      for (int i = 0; i < n; i++) sims[i] = wko_einsum_row(P + (long)i * d, C + a[i] * d, d);
    }
    int victim = -1;
    float best = INFINITY;
    for (int i = 0; i < n; i++) {
      float cand = counts[a[i]] > 1 ? sims[i] : INFINITY;
      if (victim < 0 || cand < best) { best = cand; victim = i; }
    }
    counts[a[victim]] -= 1;
    a[victim] = c;
    counts[c] = 1;
    memcpy(C + (long)c * d, P + (long)victim * d, sizeof(float) * (size_t)d);
    sims[victim] = 1.0f;
  }
  free(sims);
  free(empties);
}

/* spherical_kmeans, clustering.py:66-101 */
int wko_spherical_kmeans(const float* keys, int n, int d, int k, int iters,
                         const uint64_t rng_words[4], int threads, int64_t* a) {
  if (k < 1 || k > n) return -1;
  if (k == 1) { for (int i = 0; i < n; i++) a[i] = 0; return 0; }
  wko_rng g;
  wko_rng_init(&g, rng_words);
  float* P = (float*)malloc(sizeof(float) * (size_t)n * d);
  float* mean = (float*)malloc(sizeof(float) * (size_t)d);
  for (int t = 0; t < d; t++) {
    float s = 0.f;
    for (int i = 0; i < n; i++) s += keys[(long)i * d + t];
    mean[t] = s / (float)n;
  }
  for (long i = 0; i < (long)n * d; i++) P[i] = keys[i] - mean[i % d];
  normalize_rows(P, n, d);
  float* C = (float*)malloc(sizeof(float) * (size_t)k * d);
  seed_centroids(P, n, d, k, &g, threads, C);
  assign_argmax(P, n, C, k, d, a);
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  double* sums = (double*)malloc(sizeof(double) * (size_t)k * d);
  for (int it = 0; it < iters; it++) {
    memset(counts, 0, sizeof(int64_t) * (size_t)k);
    memset(sums, 0, sizeof(double) * (size_t)k * d);
    for (int i = 0; i < n; i++) {
      counts[a[i]]++;
      double* s = sums + a[i] * d;
      const float* p = P + (long)i * d;
      for (int t = 0; t < d; t++) s[t] += (double)p[t];
    }
    for (int c = 0; c < k; c++)
      if (counts[c] > 0)
        for (int t = 0; t < d; t++) C[(long)c * d + t] = (float)(sums[(long)c * d + t] / (double)counts[c]);
    normalize_rows(C, k, d);
    repair_empty(P, n, d, a, C, k, counts);
    assign_argmax(P, n, C, k, d, a);
  }
  memset(counts, 0, sizeof(int64_t) * (size_t)k);
  for (int i = 0; i < n; i++) counts[a[i]]++;
  repair_empty(P, n, d, a, C, k, counts);
  free(P); free(mean); free(C); free(counts); free(sums);
  return 0;
}

/* ========================================================================
 * index.py ranking / zones
 * ======================================================================*/
int wko_round_half_up(double x) { return (int)floor(x + 0.5); }

static const double* g_sort_scores;
static int cmp_rank(const void* A, const void* B) {
  int64_t a = *(const int64_t*)A, b = *(const int64_t*)B;
  double sa = g_sort_scores[a], sb = g_sort_scores[b];
  if (sa > sb) return -1;
  if (sa < sb) return 1;
  return a < b ? -1 : (a > b);
}

/* rank_clusters, index.py:61-76: dgemv then lexsort((arange, -scores)) */
void wko_rank_clusters(const double* C, int m, int d, const double* q, int threads,
                       int64_t* order, double* scores) {
  if (m == 0) return;
  wko_dgemv(C, q, m, d, threads, scores);
  for (int i = 0; i < m; i++) order[i] = i;
  g_sort_scores = scores;
  qsort(order, (size_t)m, sizeof(int64_t), cmp_rank);
}

/* ========================================================================
 * Block cache (block_cache.py:52-225) and slow-tier block accounting
 * (store.py:38-105).  Cluster-granular LRU, all-or-nothing admission.
 * ======================================================================*/
typedef struct { int32_t type, cluster, aux; int64_t step; } ev_t;

struct wko_cache {
  int64_t capacity, occupied, bsz, token_bytes;
  int64_t hits, misses, bytes_s2f, bytes_fi, bytes_read;
  int32_t ncl, cap_cl;
  int32_t* nblocks;   /* per cluster */
  int32_t* cached;
  int64_t* slot_off;  /* per cluster offset into slot_ids (allocated on register) */
  int32_t* slot_ids;
  int64_t slot_ids_len, slot_ids_cap;
  int64_t* last_access;
  int32_t *prev, *next; /* LRU list, head = oldest */
  int32_t head, tail;
  /* free slots: min-heap */
  int32_t* heap; int64_t heap_n, heap_cap;
  int32_t next_slot;
  ev_t* ev; int64_t nev, ev_cap;
  uint8_t* touched;
};

static void ev_push(wko_cache* c, int32_t type, int64_t step, int32_t cl, int32_t aux) {
  if (c->nev == c->ev_cap) {
    c->ev_cap = c->ev_cap ? 2 * c->ev_cap : 1024;
    c->ev = (ev_t*)realloc(c->ev, sizeof(ev_t) * (size_t)c->ev_cap);
  }
  c->ev[c->nev].type = type; c->ev[c->nev].step = step; c->ev[c->nev].cluster = cl; c->ev[c->nev].aux = aux;
  c->nev++;
}

wko_cache* wko_cache_new(int64_t capacity_blocks, int block_size_bytes, int d) {
  wko_cache* c = (wko_cache*)calloc(1, sizeof(wko_cache));
  c->capacity = capacity_blocks;
  c->bsz = block_size_bytes;
  c->token_bytes = 2L * d * 4;
  c->head = c->tail = -1;
  return c;
}

void wko_cache_free(wko_cache* c) {
  if (!c) return;
  free(c->nblocks); free(c->cached); free(c->slot_off); free(c->slot_ids); free(c->last_access);
  free(c->prev); free(c->next); free(c->heap); free(c->ev); free(c->touched);
  free(c);
}

int wko_cache_register(wko_cache* c, int32_t cid, int32_t nb) {
  if (cid != c->ncl) return -2; /* ids are dense in the engine */
  if (c->ncl == c->cap_cl) {
    c->cap_cl = c->cap_cl ? 2 * c->cap_cl : 1024;
    size_t n = (size_t)c->cap_cl;
    c->nblocks = (int32_t*)realloc(c->nblocks, 4 * n);
    c->cached = (int32_t*)realloc(c->cached, 4 * n);
    c->slot_off = (int64_t*)realloc(c->slot_off, 8 * n);
    c->last_access = (int64_t*)realloc(c->last_access, 8 * n);
    c->prev = (int32_t*)realloc(c->prev, 4 * n);
    c->next = (int32_t*)realloc(c->next, 4 * n);
    c->touched = (uint8_t*)realloc(c->touched, n);
  }
  c->nblocks[cid] = nb; c->cached[cid] = 0; c->last_access[cid] = -1;
  c->prev[cid] = c->next[cid] = -1; c->touched[cid] = 0;
  if (c->slot_ids_len + nb > c->slot_ids_cap) {
    while (c->slot_ids_len + nb > c->slot_ids_cap) c->slot_ids_cap = c->slot_ids_cap ? 2 * c->slot_ids_cap : 4096;
    c->slot_ids = (int32_t*)realloc(c->slot_ids, 4 * (size_t)c->slot_ids_cap);
  }
  c->slot_off[cid] = c->slot_ids_len;
  c->slot_ids_len += nb;
  c->ncl++;
  return 0;
}

void wko_cache_set_capacity(wko_cache* c, int64_t cap) { c->capacity = cap; }

static void lru_unlink(wko_cache* c, int32_t x) {
  if (c->prev[x] >= 0) c->next[c->prev[x]] = c->next[x]; else c->head = c->next[x];
  if (c->next[x] >= 0) c->prev[c->next[x]] = c->prev[x]; else c->tail = c->prev[x];
  c->prev[x] = c->next[x] = -1;
}
static void lru_append(wko_cache* c, int32_t x) {
  c->prev[x] = c->tail; c->next[x] = -1;
  if (c->tail >= 0) c->next[c->tail] = x; else c->head = x;
  c->tail = x;
}
static void heap_push(wko_cache* c, int32_t v) {
  if (c->heap_n == c->heap_cap) {
    c->heap_cap = c->heap_cap ? 2 * c->heap_cap : 1024;
    c->heap = (int32_t*)realloc(c->heap, 4 * (size_t)c->heap_cap);
  }
  int64_t i = c->heap_n++;
  c->heap[i] = v;
  while (i > 0) { int64_t p = (i - 1) / 2; if (c->heap[p] <= c->heap[i]) break; int32_t t = c->heap[p]; c->heap[p] = c->heap[i]; c->heap[i] = t; i = p; }
}
static int32_t heap_pop(wko_cache* c) {
  int32_t top = c->heap[0];
  c->heap[0] = c->heap[--c->heap_n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < c->heap_n && c->heap[l] < c->heap[s]) s = l;
    if (r < c->heap_n && c->heap[r] < c->heap[s]) s = r;
    if (s == i) break;
    int32_t t = c->heap[s]; c->heap[s] = c->heap[i]; c->heap[i] = t; i = s;
  }
  return top;
}
/* _alloc_slot, block_cache.py:147-153: smallest free id, else next new id */
static int32_t alloc_slot(wko_cache* c) { return c->heap_n ? heap_pop(c) : c->next_slot++; }
/* _evict, block_cache.py:155-161 */
static void evict(wko_cache* c, int32_t x) {
  int32_t* s = c->slot_ids + c->slot_off[x];
  for (int j = 0; j < c->nblocks[x]; j++) heap_push(c, s[j]);
  c->occupied -= c->nblocks[x];
  c->cached[x] = 0;
  lru_unlink(c, x);
}

/* lookup (:79-96) + assemble accounting (:98-143) + commit_update (:163-213) */
int wko_cache_step(wko_cache* c, const int32_t* ids, int n, int64_t step, int n_steady, uint8_t* snap) {
  for (int i = 0; i < n; i++) if (ids[i] < 0 || ids[i] >= c->ncl) return -3; /* IntegrityError */
  int64_t h = 0;
  for (int i = 0; i < n; i++) { snap[i] = (uint8_t)c->cached[ids[i]]; h += snap[i]; }
  c->hits += h; c->misses += n - h;
  ev_push(c, 0, step, n, (int32_t)h); /* access event: aux = hits, cluster = count */
  c->bytes_fi += (int64_t)n_steady * c->token_bytes;
  for (int i = 0; i < n; i++) {
    int64_t nb = c->nblocks[ids[i]];
    if (snap[i]) c->bytes_fi += nb * c->bsz;
    else { c->bytes_s2f += nb * c->bsz; c->bytes_read += nb * c->bsz; }
  }
  /* commit */
  for (int i = 0; i < n; i++) c->touched[ids[i]] = 1;
  for (int i = 0; i < n; i++) {
    c->last_access[ids[i]] = step;
    if (snap[i]) { lru_unlink(c, ids[i]); lru_append(c, ids[i]); }
  }
  for (int i = 0; i < n; i++) {
    if (snap[i]) continue;
    int32_t cid = ids[i];
    int64_t need = c->nblocks[cid];
    if (need > c->capacity) { ev_push(c, 3, step, cid, 0); continue; }
    /* evictable = LRU order minus touched; touched clusters sit at the MRU end */
    while (c->capacity - c->occupied < need) {
      int32_t v = c->head;
      if (v < 0 || c->touched[v]) break;
      evict(c, v);
      ev_push(c, 1, step, v, 0);
    }
    if (c->capacity - c->occupied < need) { ev_push(c, 3, step, cid, 0); continue; }
    int32_t* s = c->slot_ids + c->slot_off[cid];
    for (int j = 0; j < need; j++) s[j] = alloc_slot(c);
    c->occupied += need;
    c->cached[cid] = 1;
    lru_append(c, cid);
    c->bytes_fi += need * c->bsz;
    ev_push(c, 2, step, cid, (int32_t)need);
  }
  for (int i = 0; i < n; i++) c->touched[ids[i]] = 0;
  if (c->occupied > c->capacity) return -4; /* IntegrityError */
  return 0;
}

void wko_cache_counters(const wko_cache* c, int64_t out[8]) {
  out[0] = c->hits; out[1] = c->misses; out[2] = c->bytes_s2f; out[3] = c->bytes_fi;
  out[4] = c->capacity; out[5] = c->occupied; out[6] = c->bytes_read; out[7] = c->ncl;
}
int64_t wko_cache_events(const wko_cache* c, int64_t max, int32_t* type, int64_t* step, int32_t* cl, int32_t* aux) {
  int64_t n = c->nev < max ? c->nev : max;
  for (int64_t i = 0; i < n; i++) { type[i] = c->ev[i].type; step[i] = c->ev[i].step; cl[i] = c->ev[i].cluster; aux[i] = c->ev[i].aux; }
  return c->nev;
}
int wko_cache_is_cached(const wko_cache* c, int32_t cid) { return c->cached[cid]; }
int64_t wko_cache_lru(const wko_cache* c, int32_t* out, int64_t max) {
  int64_t n = 0;
  for (int32_t x = c->head; x >= 0; x = c->next[x]) { if (n < max) out[n] = x; n++; }
  return n;
}
void wko_cache_slots(const wko_cache* c, int32_t cid, int32_t* out) {
  memcpy(out, c->slot_ids + c->slot_off[cid], 4 * (size_t)c->nblocks[cid]);
}

/* ========================================================================
 * Head engine (engine.py:40-237)
 * ======================================================================*/
typedef struct { double rmax; double* num; double den; int64_t count; } partial_t;

struct wko_engine {
  wko_config cfg;
  wko_seed_fn seed_fn;
  int d, prefilled;
  int64_t step, total, n_sink, buffer_start, cap_tokens;
  float *keys, *values; /* all tokens, token order */
  /* index */
  int m, m_cap;
  double *C, *VS;
  int64_t* sizes;
  int64_t* mem_off; /* member list offsets, m+1 */
  int32_t* members; int64_t mem_len, mem_cap;
  int64_t update_round;
  /* store */
  int64_t n_blocks, bytes_written, block_cap;
  wko_cache* cache;
  /* scratch */
  int32_t *last_r, *last_e; int n_last_r, n_last_e;
};

static void grow_tokens(wko_engine* e, int64_t need) {
  if (need <= e->cap_tokens) return;
  int64_t cap = e->cap_tokens ? e->cap_tokens : 1024;
  while (cap < need) cap *= 2;
  e->keys = (float*)realloc(e->keys, sizeof(float) * (size_t)cap * e->d);
  e->values = (float*)realloc(e->values, sizeof(float) * (size_t)cap * e->d);
  e->cap_tokens = cap;
}

wko_engine* wko_engine_new(const wko_config* cfg, wko_seed_fn seed_fn) {
  wko_engine* e = (wko_engine*)calloc(1, sizeof(wko_engine));
  e->cfg = *cfg;
  e->seed_fn = seed_fn;
  return e;
}

void wko_engine_free(wko_engine* e) {
  if (!e) return;
  free(e->keys); free(e->values); free(e->C); free(e->VS); free(e->sizes); free(e->mem_off);
  free(e->members); free(e->last_r); free(e->last_e);
  wko_cache_free(e->cache);
  free(e);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* store.pack_cluster (store.py:69-90): fresh cluster-private blocks */
static int64_t pack_blocks(wko_engine* e, int64_t n_tokens) {
  int64_t nb = ceil_div(n_tokens, e->block_cap);
  e->n_blocks += nb;
  e->bytes_written += nb * e->cfg.block_size_bytes;
  return nb;
}

static void ensure_clusters(wko_engine* e, int need) {
  if (need <= e->m_cap) return;
  int cap = e->m_cap ? e->m_cap : 256;
  while (cap < need) cap *= 2;
  e->C = (double*)realloc(e->C, sizeof(double) * (size_t)cap * e->d);
  e->VS = (double*)realloc(e->VS, sizeof(double) * (size_t)cap * e->d);
  e->sizes = (int64_t*)realloc(e->sizes, sizeof(int64_t) * (size_t)cap);
  e->mem_off = (int64_t*)realloc(e->mem_off, sizeof(int64_t) * (size_t)(cap + 1));
  e->m_cap = cap;
}

/* finalize_cluster for every cluster of one clustered batch (index.py:43-58,
 * 143-151): tokens are the contiguous token-id range [t0, t0+L), `a` their
 * assignment (freed here) */
static int finalize_batch(wko_engine* e, int64_t t0, int L, int k, int64_t* a) {
  int d = e->d;
  ensure_clusters(e, e->m + k);
  if (e->mem_len + L > e->mem_cap) {
    while (e->mem_len + L > e->mem_cap) e->mem_cap = e->mem_cap ? 2 * e->mem_cap : 65536;
    e->members = (int32_t*)realloc(e->members, sizeof(int32_t) * (size_t)e->mem_cap);
  }
  /* stable counting sort of members by cluster (ascending token order) */
  int64_t* cnt = (int64_t*)calloc((size_t)k + 1, sizeof(int64_t));
  for (int i = 0; i < L; i++) cnt[a[i] + 1]++;
  for (int c = 0; c < k; c++) cnt[c + 1] += cnt[c];
  int64_t base = e->mem_len;
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int c = 0; c < k; c++) pos[c] = cnt[c];
  for (int i = 0; i < L; i++) e->members[base + pos[a[i]]++] = (int32_t)(t0 + i);
  for (int c = 0; c < k; c++) {
    int cid = e->m + c;
    int64_t s = cnt[c + 1] - cnt[c];
    if (s == 0) { free(cnt); free(pos); free(a); return -5; } /* IntegrityError */
    e->mem_off[cid] = base + cnt[c];
    e->mem_off[cid + 1] = base + cnt[c + 1];
    double* cc = e->C + (long)cid * d;
    double* vv = e->VS + (long)cid * d;
    for (int t = 0; t < d; t++) { cc[t] = 0.0; vv[t] = 0.0; }
    for (int64_t j = cnt[c]; j < cnt[c + 1]; j++) {
      int64_t tok = e->members[base + j];
      for (int t = 0; t < d; t++) {
        cc[t] += (double)e->keys[tok * d + t];
        vv[t] += (double)e->values[tok * d + t];
      }
    }
    for (int t = 0; t < d; t++) cc[t] = cc[t] / (double)s;
    e->sizes[cid] = s;
    int64_t nb = pack_blocks(e, s);
    if (e->cache) wko_cache_register(e->cache, cid, (int32_t)nb);
  }
  e->mem_len += L;
  e->m += k;
  free(cnt); free(pos); free(a);
  return 0;
}

/* _cluster_batch (index.py:143-151): spherical k-means, then finalize */
static int cluster_batch(wko_engine* e, int64_t t0, int L, int k, int kind, int64_t idx) {
  uint64_t words[4];
  e->seed_fn(e->cfg.rng_seed, kind, idx, words);
  int64_t* a = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
  int rc = wko_spherical_kmeans(e->keys + t0 * e->d, L, e->d, k, e->cfg.kmeans_iters, words,
                                e->cfg.blas_threads, a);
  if (rc) { free(a); return rc; }
  return finalize_batch(e, t0, L, k, a);
}

/* engine._update_capacity (engine.py:98-101) */
static void update_capacity(wko_engine* e) {
  int64_t want = (int64_t)ceil(e->cfg.cache_fraction * (double)e->n_blocks);
  if (want > e->cache->capacity) e->cache->capacity = want;
}

/* segment k-means workers of the segmented build (one segment per pull) */
typedef struct {
  wko_engine* e;
  int64_t L;
  int nseg;
  const uint64_t* words;
  int64_t** asg;
  int next, rc;
  pthread_mutex_t mu;
} seg_job;

static void* seg_worker(void* arg) {
  seg_job* j = (seg_job*)arg;
  wko_engine* e = j->e;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int seg = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (seg >= j->nseg) return NULL;
    int64_t s0 = (int64_t)seg * e->cfg.segment_size;
    int64_t len = j->L - s0 < e->cfg.segment_size ? j->L - s0 : e->cfg.segment_size;
    int k = (int)ceil_div(len, e->cfg.centroid_ratio);
    j->asg[seg] = (int64_t*)malloc(sizeof(int64_t) * (size_t)len);
    int rc = wko_spherical_kmeans(e->keys + (e->n_sink + s0) * e->d, (int)len, e->d, k, e->cfg.kmeans_iters,
                                  j->words + 4 * seg, e->cfg.blas_threads, j->asg[seg]);
    if (rc) {
      pthread_mutex_lock(&j->mu);
      j->rc = rc;
      pthread_mutex_unlock(&j->mu);
    }
  }
}

/* HeadEngine.prefill (engine.py:110-138) */
int wko_engine_prefill(wko_engine* e, const float* keys, const float* values, int n, int d) {
  if (e->prefilled) return -1;
  if (n < 1 || d < 1) return -1;
  e->d = d;
  int64_t bc = e->cfg.block_size_bytes / (2L * d * 4);
  if (bc < 1) return -1;
  e->block_cap = bc;
  e->cache = wko_cache_new(0, e->cfg.block_size_bytes, d);
  grow_tokens(e, n);
  memcpy(e->keys, keys, sizeof(float) * (size_t)n * d);
  memcpy(e->values, values, sizeof(float) * (size_t)n * d);
  e->total = n;
  e->n_sink = n < e->cfg.sink_tokens ? n : e->cfg.sink_tokens;
  int64_t index_end = n - e->cfg.local_window;
  if (index_end < e->n_sink) index_end = e->n_sink;
  e->buffer_start = index_end;
  if (e->n_sink) pack_blocks(e, e->n_sink);
  ensure_clusters(e, 1);
  e->mem_off[0] = 0;
  /* segmented_build (index.py:153-166): segments are independent (seed
   * [rng_seed, 1, seg]), so their k-means runs on all host cores; finalize
   * and packing stay sequential in segment order (dense ids). */
  int64_t L = index_end - e->n_sink;
  int nseg = (int)ceil_div(L, e->cfg.segment_size);
  uint64_t* words = (uint64_t*)malloc(sizeof(uint64_t) * 4 * (size_t)(nseg > 0 ? nseg : 1));
  int64_t** asg = (int64_t**)calloc((size_t)(nseg > 0 ? nseg : 1), sizeof(int64_t*));
  for (int seg = 0; seg < nseg; seg++) e->seed_fn(e->cfg.rng_seed, 1, seg, words + 4 * seg);
  seg_job job = {e, L, nseg, words, asg, 0, 0};
  pthread_mutex_init(&job.mu, NULL);
  long ncpu = sysconf(_SC_NPROCESSORS_ONLN);
  int nth = (int)(ncpu < 1 ? 1 : ncpu);
  if (nth > nseg) nth = nseg;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)(nth > 0 ? nth : 1));
  int started = 0;
  for (int i = 1; i < nth; i++)
    if (pthread_create(&th[started], NULL, seg_worker, &job) == 0) started++;
  seg_worker(&job);
  for (int i = 0; i < started; i++) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&job.mu);
  int rc = job.rc ? -1 : 0;
  for (int seg = 0; seg < nseg; seg++) {
    int64_t s0 = (int64_t)seg * e->cfg.segment_size;
    int64_t len = L - s0 < e->cfg.segment_size ? L - s0 : e->cfg.segment_size;
    int k = (int)ceil_div(len, e->cfg.centroid_ratio);
    if (!rc) rc = finalize_batch(e, e->n_sink + s0, (int)len, k, asg[seg]);
    else free(asg[seg]);
    asg[seg] = NULL;
  }
  free(asg);
  free(words);
  if (rc) return rc;
  update_capacity(e);
  e->prefilled = 1;
  return 0;
}

static void exact_partial(const double* q, const float* K, const float* V, int64_t T, int d,
                          partial_t* p, double* scratch) {
  p->count = T;
  p->den = 0.0;
  for (int t = 0; t < d; t++) p->num[t] = 0.0;
  if (T == 0) { p->rmax = -INFINITY; return; }
  double sq = sqrt((double)d);
  double mx = -INFINITY;
  for (int64_t j = 0; j < T; j++) {
    double s = 0.0;
    for (int t = 0; t < d; t++) s = fma((double)K[j * d + t], q[t], s);
    s = s / sq;
    scratch[j] = s;
    if (s > mx) mx = s;
  }
  for (int64_t j = 0; j < T; j++) {
    double w = exp(scratch[j] - mx);
    p->den += w;
    for (int t = 0; t < d; t++) p->num[t] += w * (double)V[j * d + t];
  }
  p->rmax = mx;
}

/* estimate_partial (attention.py:81-104) with precomputed scores; zero_num
 * gives tail_denominator_partial (:107-112) */
static void estimate_partial(const wko_engine* e, const int32_t* ids, int n, const double* scores,
                             int zero_num, partial_t* p) {
  int d = e->d;
  p->count = n; p->den = 0.0;
  for (int t = 0; t < d; t++) p->num[t] = 0.0;
  if (n == 0) { p->rmax = -INFINITY; return; }
  double sq = sqrt((double)d), mx = -INFINITY;
  for (int i = 0; i < n; i++) { double s = scores[ids[i]] / sq; if (s > mx) mx = s; }
  for (int i = 0; i < n; i++) {
    double w = exp(scores[ids[i]] / sq - mx);
    p->den += (double)e->sizes[ids[i]] * w;
    if (!zero_num) {
      const double* vs = e->VS + (long)ids[i] * d;
      for (int t = 0; t < d; t++) p->num[t] += w * vs[t];
    }
  }
  p->rmax = mx;
}

/* merged_sums (attention.py:115-130) */
static int merged_sums(partial_t** ps, int np_, int d, double* gmax, double* num, double* den) {
  double g = -INFINITY;
  int live = 0;
  for (int i = 0; i < np_; i++) if (ps[i]->count > 0) { live++; if (ps[i]->rmax > g) g = ps[i]->rmax; }
  if (!live) return -1;
  for (int t = 0; t < d; t++) num[t] = 0.0;
  *den = 0.0;
  for (int i = 0; i < np_; i++) {
    if (ps[i]->count <= 0) continue;
    double sc = exp(ps[i]->rmax - g);
    for (int t = 0; t < d; t++) num[t] += ps[i]->num[t] * sc;
    *den += ps[i]->den * sc;
  }
  *gmax = g;
  return 0;
}

typedef struct { const double* s; } tk_ctx;
static const double* g_tk;
static int cmp_tk(const void* A, const void* B) {
  int64_t a = *(const int64_t*)A, b = *(const int64_t*)B;
  if (g_tk[a] > g_tk[b]) return -1;
  if (g_tk[a] < g_tk[b]) return 1;
  return a < b ? -1 : (a > b);
}

/* HeadEngine.decode_step (engine.py:174-232) */
int wko_engine_decode(wko_engine* e, const double* q, const float* knew, const float* vnew,
                      int with_oracle, int with_recall, double* out, wko_metrics* met) {
  if (!e->prefilled) return -1;
  int d = e->d;
  const wko_config* cfg = &e->cfg;
  grow_tokens(e, e->total + 1);
  memcpy(e->keys + e->total * d, knew, sizeof(float) * (size_t)d);
  memcpy(e->values + e->total * d, vnew, sizeof(float) * (size_t)d);
  e->total++;
  int m = e->m;
  /* rank + plan_zones (index.py:61-93) */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  double* scores = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  wko_rank_clusters(e->C, m, d, q, cfg->blas_threads, order, scores);
  int r = 0, ne = 0;
  if (m > 0) {
    r = wko_round_half_up(cfg->retrieval_fraction * m);
    if (r < 1) r = 1;
    if (r > m) r = m;
    ne = wko_round_half_up(cfg->estimation_fraction * m);
    if (ne > m - r) ne = m - r;
  }
  e->last_r = (int32_t*)realloc(e->last_r, sizeof(int32_t) * (size_t)(r + 1));
  e->last_e = (int32_t*)realloc(e->last_e, sizeof(int32_t) * (size_t)(ne + 1));
  for (int i = 0; i < r; i++) e->last_r[i] = (int32_t)order[i];
  for (int i = 0; i < ne; i++) e->last_e[i] = (int32_t)order[r + i];
  e->n_last_r = r; e->n_last_e = ne;

  double* nbuf = (double*)calloc((size_t)6 * d, sizeof(double));
  partial_t est = {0, nbuf, 0, 0}, ex = {0, nbuf + d, 0, 0}, tail = {0, nbuf + 2 * d, 0, 0};
  estimate_partial(e, e->last_e, ne, scores, 0, &est);

  int64_t h0 = e->cache->hits, m0 = e->cache->misses, s0 = e->cache->bytes_s2f, f0 = e->cache->bytes_fi;
  /* steady zone (engine.py:87-96) + retrieval clusters in rank order */
  int64_t n_steady = e->n_sink + (e->total - e->buffer_start);
  int64_t T = n_steady;
  for (int i = 0; i < r; i++) T += e->sizes[e->last_r[i]];
  float* K = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1) * d);
  float* V = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1) * d);
  uint8_t* retrieved = (uint8_t*)calloc((size_t)e->total, 1);
  int64_t pos = 0;
  for (int64_t t = 0; t < e->n_sink; t++, pos++) {
    memcpy(K + pos * d, e->keys + t * d, 4 * (size_t)d); memcpy(V + pos * d, e->values + t * d, 4 * (size_t)d);
    retrieved[t] = 1;
  }
  for (int64_t t = e->buffer_start; t < e->total; t++, pos++) {
    memcpy(K + pos * d, e->keys + t * d, 4 * (size_t)d); memcpy(V + pos * d, e->values + t * d, 4 * (size_t)d);
    retrieved[t] = 1;
  }
  for (int i = 0; i < r; i++) {
    int c = e->last_r[i];
    for (int64_t j = e->mem_off[c]; j < e->mem_off[c + 1]; j++, pos++) {
      int64_t tok = e->members[j];
      memcpy(K + pos * d, e->keys + tok * d, 4 * (size_t)d); memcpy(V + pos * d, e->values + tok * d, 4 * (size_t)d);
      retrieved[tok] = 1;
    }
  }
  /* lookup/assemble/commit accounting happen in wko_cache_step below; the
   * attention result does not depend on residency (payload equivalence,
   * block_cache.py:98-143) */
  double* scratch = (double*)malloc(sizeof(double) * (size_t)((T > e->total ? T : e->total) + 1));
  exact_partial(q, K, V, T, d, &ex, scratch);

  /* _final_output (engine.py:150-172) */
  double gmax, den, cov, logden;
  double* num = nbuf + 3 * d;
  partial_t* parts[3] = {&ex, &est, &tail};
  int np_ = 2;
  int32_t* dropped = NULL;
  int nd = m - r - ne;
  if (cfg->tail_denominator_only && nd > 0) {
    dropped = (int32_t*)malloc(sizeof(int32_t) * (size_t)nd);
    for (int i = 0; i < nd; i++) dropped[i] = (int32_t)order[r + ne + i];
    estimate_partial(e, dropped, nd, scores, 1, &tail);
    np_ = 3;
  }
  int rc = 0;
  if (!cfg->denominator_eq2) {
    if (merged_sums(parts, np_, d, &gmax, num, &den)) { rc = -1; goto done; }
    double exd = ex.count > 0 ? ex.den * exp(ex.rmax - gmax) : 0.0;
    cov = den > 0 ? exd / den : 0.0;
    for (int t = 0; t < d; t++) out[t] = num[t] / den;
    logden = gmax + log(den);
  } else {
    double gn, dn_unused;
    if (merged_sums(parts, np_, d, &gn, num, &dn_unused)) { rc = -1; goto done; }
    partial_t st = {0, nbuf + 4 * d, 0, 0}, ct = {0, nbuf + 5 * d, 0, 0};
    exact_partial(q, K, V, n_steady, d, &st, scratch);
    int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    for (int i = 0; i < m; i++) all[i] = i;
    estimate_partial(e, all, m, scores, 1, &ct);
    free(all);
    partial_t* p2[2] = {&st, &ct};
    double gd, dd;
    double* tmp = (double*)calloc((size_t)d, sizeof(double));
    if (merged_sums(p2, 2, d, &gd, tmp, &dd)) { free(tmp); rc = -1; goto done; }
    free(tmp);
    for (int t = 0; t < d; t++) out[t] = num[t] * exp(gn - gd) / dd;
    double sd = st.count > 0 ? st.den * exp(st.rmax - gd) : 0.0;
    cov = dd > 0 ? sd / dd : 0.0;
    logden = gd + log(dd);
  }

  /* metrics: recall_at_k (metrics.py:19-26), oracle rel error */
  met->recall = NAN;
  if (with_recall) {
    int64_t n = e->total, kk = cfg->metrics_k < n ? cfg->metrics_k : n;
    double* Kd = (double*)malloc(sizeof(double) * (size_t)n * d);
    for (int64_t i = 0; i < n * d; i++) Kd[i] = (double)e->keys[i];
    double* sc = (double*)malloc(sizeof(double) * (size_t)n);
    wko_dgemv(Kd, q, (int)n, d, cfg->blas_threads, sc);
    int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) ord[i] = i;
    g_tk = sc;
    qsort(ord, (size_t)n, sizeof(int64_t), cmp_tk);
    int64_t hit = 0;
    for (int64_t i = 0; i < kk; i++) hit += retrieved[ord[i]];
    met->recall = kk == 0 ? 1.0 : (double)hit / (double)kk;
    free(Kd); free(sc); free(ord);
  }
  met->rel_error = NAN;
  if (with_oracle) {
    partial_t o = {0, nbuf + 4 * d, 0, 0};
    exact_partial(q, e->keys, e->values, e->total, d, &o, scratch);
    double nrm = 0, diff = 0;
    for (int t = 0; t < d; t++) {
      double ov = o.num[t] / o.den;
      nrm += ov * ov;
      diff += (out[t] - ov) * (out[t] - ov);
    }
    met->rel_error = nrm == 0 ? sqrt(diff) : sqrt(diff) / sqrt(nrm);
  }

  {
    uint8_t* snap = (uint8_t*)malloc((size_t)(r > 0 ? r : 1));
    int crc = wko_cache_step(e->cache, e->last_r, r, e->step, (int)n_steady, snap);
    free(snap);
    if (crc) { rc = crc; goto done; }
  }
  /* index.update (index.py:168-186) */
  while (e->total - e->buffer_start >= cfg->update_segment + cfg->local_window) {
    int k = (int)ceil_div(cfg->update_segment, cfg->centroid_ratio);
    int crc = cluster_batch(e, e->buffer_start, cfg->update_segment, k, 2, e->update_round);
    e->update_round++;
    if (crc) { rc = crc; goto done; }
    e->buffer_start += cfg->update_segment;
    update_capacity(e);
  }
  met->step = e->step;
  met->hits = e->cache->hits - h0;
  met->misses = e->cache->misses - m0;
  met->bytes_slow_to_fast = e->cache->bytes_s2f - s0;
  met->bytes_fast_internal = e->cache->bytes_fi - f0;
  met->denominator_coverage = cov;
  met->log_denominator = logden;
  met->m = e->m;
  met->r = r;
  met->e = ne;
  e->step++;
done:
  free(order); free(scores); free(nbuf); free(K); free(V); free(retrieved); free(scratch); free(dropped);
  return rc;
}

static void* dup_mem(const void* src, size_t bytes) {
  if (!src || !bytes) return NULL;
  void* d = malloc(bytes);
  memcpy(d, src, bytes);
  return d;
}

static wko_cache* cache_clone(const wko_cache* c) {
  if (!c) return NULL;
  wko_cache* x = (wko_cache*)malloc(sizeof(wko_cache));
  *x = *c;
  size_t n = (size_t)c->cap_cl;
  x->nblocks = (int32_t*)dup_mem(c->nblocks, 4 * n);
  x->cached = (int32_t*)dup_mem(c->cached, 4 * n);
  x->slot_off = (int64_t*)dup_mem(c->slot_off, 8 * n);
  x->last_access = (int64_t*)dup_mem(c->last_access, 8 * n);
  x->prev = (int32_t*)dup_mem(c->prev, 4 * n);
  x->next = (int32_t*)dup_mem(c->next, 4 * n);
  x->touched = (uint8_t*)dup_mem(c->touched, n);
  x->slot_ids = (int32_t*)dup_mem(c->slot_ids, 4 * (size_t)c->slot_ids_cap);
  x->heap = (int32_t*)dup_mem(c->heap, 4 * (size_t)c->heap_cap);
  x->ev = (ev_t*)dup_mem(c->ev, sizeof(ev_t) * (size_t)c->ev_cap);
  return x;
}

/* Deep copy of an engine: the G heads of a GQA group build the identical
 * index (the seeds do not depend on the head, index.py:162), so tests prefill
 * once and clone per head (test infrastructure). */
wko_engine* wko_engine_clone(const wko_engine* e) {
  wko_engine* x = (wko_engine*)malloc(sizeof(wko_engine));
  *x = *e;
  size_t d = (size_t)(e->d > 0 ? e->d : 0), mc = (size_t)e->m_cap;
  x->keys = (float*)dup_mem(e->keys, sizeof(float) * (size_t)e->cap_tokens * d);
  x->values = (float*)dup_mem(e->values, sizeof(float) * (size_t)e->cap_tokens * d);
  x->C = (double*)dup_mem(e->C, sizeof(double) * mc * d);
  x->VS = (double*)dup_mem(e->VS, sizeof(double) * mc * d);
  x->sizes = (int64_t*)dup_mem(e->sizes, sizeof(int64_t) * mc);
  x->mem_off = (int64_t*)dup_mem(e->mem_off, sizeof(int64_t) * (mc + 1));
  x->members = (int32_t*)dup_mem(e->members, sizeof(int32_t) * (size_t)e->mem_cap);
  x->last_r = x->last_e = NULL;
  x->n_last_r = x->n_last_e = 0;
  x->cache = cache_clone(e->cache);
  return x;
}

int wko_engine_m(const wko_engine* e) { return e->m; }
const double* wko_engine_centroids(const wko_engine* e) { return e->C; }
const double* wko_engine_value_sums(const wko_engine* e) { return e->VS; }
const int64_t* wko_engine_sizes(const wko_engine* e) { return e->sizes; }
const int32_t* wko_engine_members(const wko_engine* e, int c, int* count) {
  *count = (int)(e->mem_off[c + 1] - e->mem_off[c]);
  return e->members + e->mem_off[c];
}
void wko_engine_counters(const wko_engine* e, int64_t out[12]) {
  int64_t cc[8];
  wko_cache_counters(e->cache, cc);
  for (int i = 0; i < 8; i++) out[i] = cc[i];
  out[8] = e->n_blocks; out[9] = e->bytes_written; out[10] = e->total; out[11] = e->buffer_start;
}
const int32_t* wko_engine_last_retrieval(const wko_engine* e, int* count) { *count = e->n_last_r; return e->last_r; }
const int32_t* wko_engine_last_estimation(const wko_engine* e, int* count) { *count = e->n_last_e; return e->last_e; }
int64_t wko_engine_events(const wko_engine* e, int64_t max, int32_t* type, int64_t* step, int32_t* cl, int32_t* aux) {
  return wko_cache_events(e->cache, max, type, step, cl, aux);
}
