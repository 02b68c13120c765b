/* wk_oracle.h -- CPU oracle for the wave-index decode-attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * package `tierkv` (/root/reference/pkg/src/tierkv), used solely as the
 * checker in tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  Nothing in the product (paper_2505_02922_b200/)
 * links, imports or executes it.
 *
 * Every floating-point primitive reproduces the exact evaluation order that
 * numpy 2.3 + OpenBLAS 0.3.30 (SkylakeX kernels) use for the corresponding
 * reference call site, so outputs are bit-identical to tierkv where the
 * recipe is modelled (see DESIGN.md "Numerics recipes" for the domain).
 * Parity pinned against tierkv by oracle/make_golden.py -> tests/golden/.
 */
#ifndef WK_ORACLE_H
#define WK_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- numpy PCG64 / Generator draws (numpy/random/src/pcg64, distributions.c) */
typedef struct {
  uint64_t st_hi, st_lo, inc_hi, inc_lo; /* 128-bit LCG state and increment */
  int has32;
  uint32_t u32;
} wko_rng;
void wko_rng_init(wko_rng* g, const uint64_t words[4]); /* state_hi, state_lo, inc_hi, inc_lo */
uint64_t wko_next64(wko_rng* g);
uint32_t wko_next32(wko_rng* g);
double wko_next_double(wko_rng* g);
int64_t wko_integers(wko_rng* g, int64_t n); /* Generator.integers(n), n <= 2^32 */

/* ---- BLAS / numpy evaluation-order recipes --------------------------------*/
/* points[n,d] @ cents[k,d].T  (clustering.py:85,96 sgemm) */
void wko_sgemm_nt(const float* P, const float* C, int n, int k, int d, float* out);
/* A[n,d] @ x[d]  fp32 (clustering.py:33,42 sgemv), OpenBLAS thread chunking */
void wko_sgemv(const float* A, const float* x, int n, int d, int threads, float* y);
/* A[n,d] @ x[d]  fp64 (index.py:74 dgemv, metrics.py:14) */
void wko_dgemv(const double* A, const double* x, int n, int d, int threads, double* y);
/* np.linalg.norm(x, axis=1) fp32 (clustering.py:18) */
void wko_row_norms(const float* x, int n, int d, float* out);
/* np.einsum("ij,ij->i") fp32 (clustering.py:55) */
float wko_einsum_row(const float* a, const float* b, int d);

/* ---- clustering.py -------------------------------------------------------*/
/* returns 0 ok, -1 ConfigError (k<1 or k>n) */
int wko_spherical_kmeans(const float* keys, int n, int d, int k, int iters,
                         const uint64_t rng_words[4], int threads, int64_t* assignment);

/* ---- index.py ------------------------------------------------------------*/
void wko_rank_clusters(const double* C, int m, int d, const double* q, int threads,
                       int64_t* order, double* scores);
int wko_round_half_up(double x);

/* ---- head engine (engine.py + index.py + block_cache.py + store.py) ------*/
typedef struct wko_engine wko_engine;
typedef struct {
  int centroid_ratio, segment_size, kmeans_iters, update_segment, sink_tokens, local_window;
  double retrieval_fraction, estimation_fraction;
  int tail_denominator_only; /* tail_mode */
  int64_t rng_seed;
  double cache_fraction;
  int block_size_bytes;
  int denominator_eq2; /* denominator_mode */
  int metrics_k;
  int blas_threads; /* OPENBLAS_NUM_THREADS of the modelled reference run */
} wko_config;

typedef struct {
  int64_t step;
  double recall;
  double rel_error; /* NaN when not requested */
  int64_t hits, misses, bytes_slow_to_fast, bytes_fast_internal;
  double denominator_coverage, log_denominator;
  int64_t m, r, e;
} wko_metrics;

/* seed_words_fn: callback returning the 4 PCG64 state words for
 * SeedSequence([rng_seed, kind, idx]) (computed by numpy on the host). */
typedef void (*wko_seed_fn)(int64_t rng_seed, int kind, int64_t idx, uint64_t out[4]);

wko_engine* wko_engine_new(const wko_config* cfg, wko_seed_fn seed_fn);
wko_engine* wko_engine_clone(const wko_engine* e);
void wko_engine_free(wko_engine* e);
int wko_engine_prefill(wko_engine* e, const float* keys, const float* values, int n, int d);
int wko_engine_decode(wko_engine* e, const double* q, const float* k, const float* v,
                      int with_oracle, int with_recall, double* out, wko_metrics* met);
/* state accessors (views valid until the next call) */
int wko_engine_m(const wko_engine* e);
const double* wko_engine_centroids(const wko_engine* e);
const double* wko_engine_value_sums(const wko_engine* e);
const int64_t* wko_engine_sizes(const wko_engine* e);
/* member token ids of cluster c: pointer + count */
const int32_t* wko_engine_members(const wko_engine* e, int c, int* count);
void wko_engine_counters(const wko_engine* e, int64_t out[12]);
/* last step's plan: retrieval ids (rank order), estimation ids */
const int32_t* wko_engine_last_retrieval(const wko_engine* e, int* count);
const int32_t* wko_engine_last_estimation(const wko_engine* e, int* count);
/* event log: type (0 access,1 evict,2 admit,3 reject), step, cluster, blocks/cached */
int64_t wko_engine_events(const wko_engine* e, int64_t max, int32_t* type, int64_t* step,
                          int32_t* cluster, int32_t* aux);

/* ---- standalone block cache (block_cache.py), fed an arbitrary stream ---*/
typedef struct wko_cache wko_cache;
wko_cache* wko_cache_new(int64_t capacity_blocks, int block_size_bytes, int d);
void wko_cache_free(wko_cache* c);
int wko_cache_register(wko_cache* c, int32_t cluster_id, int32_t n_blocks);
void wko_cache_set_capacity(wko_cache* c, int64_t capacity_blocks);
/* one step: lookup + assemble accounting + commit. ids in rank order (unique).
 * cached_out[i] = residency snapshot.  n_steady tokens charged as fast-internal. */
int wko_cache_step(wko_cache* c, const int32_t* ids, int n, int64_t step, int n_steady,
                   uint8_t* cached_out);
void wko_cache_counters(const wko_cache* c, int64_t out[8]);
int64_t wko_cache_events(const wko_cache* c, int64_t max, int32_t* type, int64_t* step,
                         int32_t* cluster, int32_t* aux);
int wko_cache_is_cached(const wko_cache* c, int32_t cluster_id);
int64_t wko_cache_lru(const wko_cache* c, int32_t* out, int64_t max);
void wko_cache_slots(const wko_cache* c, int32_t cluster_id, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
