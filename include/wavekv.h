/* wavekv.h -- C ABI of the B200 wave-index decode-attention path.
 *
 * Drop-in boundary for the reference package tierkv (/root/reference/pkg/src/
 * tierkv).  The reference exposes a Python API, not an FFI; every entry point
 * below replaces the compute behind one reference call site (cited), and the
 * Python host layer paper_2505_02922_b200 binds them with ctypes exactly as a
 * tierkv maintainer would.
 *
 * Conventions
 *  - All data pointers are device pointers to caller-allocated memory (the
 *    library allocates nothing); `stream` is a cudaStream_t passed as void*.
 *    Calls are stream-ordered and asynchronous.
 *  - Return value: 0 ok; WK_ECONFIG (<0) for caller/config errors (maps to
 *    tierkv.ConfigError).  Device-detected invariant violations are reported
 *    through the int status word in the step/build views (non-zero ->
 *    tierkv.IntegrityError, errors.py:4-23).
 *  - d % 4 == 0, d <= 256; G (query heads per kv head) <= 8.
 */
#ifndef WAVEKV_H
#define WAVEKV_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WK_ECONFIG (-1)
#define WK_ECUDA (-2)

/* Per-layer index arrays of U (request, kv-head) units (index.py:96-189,
 * store.py:48-105).  Shapes in elements. */
typedef struct wk_index_view {
  void* store_k;      /* [U, s_cap, d] bf16|fp32 keys, cluster-contiguous     */
  void* store_v;      /* [U, s_cap, d] values                                  */
  int32_t* store_tok; /* [U, s_cap] token id per store row                     */
  int32_t* cl_off;    /* [U, m_cap] first store row of each cluster            */
  int32_t* cl_size;   /* [U, m_cap] cluster sizes (MetaIndexEntry.size)        */
  double* C64;        /* [U, m_cap, d] fp64 centroids (MetaIndexEntry.centroid)*/
  float* C32;         /* [U, m_cap, d] fp32 copy for the scoring scan          */
  float* Cnorm;       /* [U, m_cap] ||C32||                                    */
  float* VS32;        /* [U, m_cap, d] fp32 value sums                         */
  double* VS64;       /* [U, m_cap, d] fp64 value sums (optional, may be NULL) */
  int64_t s_cap, m_cap;
  float* Cmax;        /* [U] max_c ||C32_c|| (score error bound), set at build */
} wk_index_view;

/* One clustering segment: a contiguous token range of one unit
 * (index.py:153-166 segments; index.py:168-186 decode-time updates). */
typedef struct wk_segment {
  const float* keys;  /* device fp32 keys of the segment, row stride key_stride */
  const float* values;
  int64_t key_stride;
  int32_t L, k;       /* points, clusters (k = ceil(L / centroid_ratio))       */
  int32_t unit, cid_base, row_base, tok_base;
  int64_t p_off, c_off; /* offsets (rows) into the build scratch                */
  uint64_t rng[4];    /* numpy PCG64 state of SeedSequence([seed, kind, idx])  */
} wk_segment;

/* Build scratch, sized by the caller: P/A/perm/sims/md rows = sum L,
 * C rows = sum k (see paper_2505_02922_b200/wave.py:_build_scratch). */
typedef struct wk_build_scratch {
  float* P;           /* [sum L, d] normalized points                          */
  float* C;           /* [sum k, d] spherical centroids                        */
  int32_t* A;         /* [sum L] assignment                                    */
  int32_t* perm;      /* [sum L] members sorted by cluster                     */
  float* sims;        /* [sum L] repair similarities                           */
  float* md;          /* [2 * sum L] min-dist + cdf (k-means++ seeding)        */
  wk_segment* segs_dev; /* [n_segments] device copy of the descriptors         */
  int* status;        /* device status word                                    */
  void* P16;          /* [sum L, d] fp16 copy of P: k-means++ first pass (may be NULL) */
} wk_build_scratch;

/* Steady zone: sinks + decode buffer per unit (engine.py:87-96). */
typedef struct wk_steady_view {
  void* k;            /* [U, t_cap, d]                                          */
  void* v;
  int32_t* tok;       /* [U, t_cap]                                             */
  int32_t* n;         /* [U] live rows                                          */
  int32_t* next_tok;  /* [U] token id of the next appended token                */
  int64_t t_cap;
} wk_steady_view;

/* Per-step buffers (decode_step, engine.py:174-232). */
typedef struct wk_step_view {
  const float* q;     /* [U, G, d] queries                                      */
  int32_t* m;         /* [U] cluster count                                      */
  float* scores;      /* [U, G, m_cap] approximate q.C (ZonePlan.scores)        */
  int32_t* rlist;     /* [U, G, r_cap] retrieval ids in rank order              */
  int32_t* elist;     /* [U, G, e_cap] estimation ids (optional)                */
  int32_t* nr;        /* [U] r                                                  */
  int32_t* ne;        /* [U] e                                                  */
  uint32_t* zmask;    /* [U, m_cap] zone bits (zeroed by wk_score_topk)         */
  int32_t* ru_ids;    /* [U, ru_cap] union of retrieval clusters                */
  uint8_t* ru_mask;
  int32_t* ru_pre;    /* [U, ru_cap + 1]                                        */
  int32_t* eu_ids;    /* [U, eu_cap] union of estimation clusters               */
  uint8_t* eu_mask;
  int32_t* cnt;       /* [U, 4]                                                 */
  float* tail;        /* [U, G, 4]                                              */
  float* part;        /* partial records: wk_tripartite_attn [12 (S + U), 3, G,
                         4 + d] (attend_v6 keys consumer x (CTA + unit),
                         attend_v4 CTA warp + unit); reference kernels
                         [U, S, G, 3, 2 + d]                                     */
  float* out;         /* [U, G, d] attention output (AttentionOutput.output)    */
  float* logden;      /* [U, G] StepMetrics.log_denominator                     */
  float* cov;         /* [U, G] StepMetrics.denominator_coverage                */
  int* status;        /* device status word                                     */
  int32_t r_cap, e_cap, ru_cap, eu_cap;
  int32_t* rtok_row;  /* [U, rt_cap] every retrieved token of the unit's union:
                         store row | head mask << 24 (fast path, bf16 store:
                         written by the zone planning instead of `pieces` and
                         read by the attention; NULL: pieces)                 */
  uint8_t* rtok_mask; /* unused (NULL)                                           */
  int32_t* sel_done;  /* [U] zero-initialised counter (last-CTA handoff)        */
  int32_t rt_cap, pad_;
  float* eu_x;        /* [U, eu_cap, G] estimation-row scores (-inf: head not in zone) */
  float* eu_sz;       /* [U, eu_cap] estimation-row cluster sizes                */
  uint32_t* rbits;    /* [U, G, w_cap] retrieval set of each head (bitmap)      */
  uint32_t* ebits;    /* [U, G, w_cap] estimation set of each head (bitmap)     */
  int32_t* pieces;    /* [U, pc_cap, 2] retrieval runs: (store row, n | mask<<8) */
  int32_t* woff;      /* [U + 1] attention chunk prefix (scratch)               */
  int32_t w_cap, pc_cap;
  /* offload path (host store + HBM slot arena); pstride 2 = in-HBM store */
  void* arena_k;      /* [U, arena_rows, d] cached blocks (block_tokens rows/slot) */
  void* arena_v;
  const int32_t* slot_ids; /* [U, slot_cap] physical slot of each cluster block  */
  const int32_t* slot_off; /* [U, m_cap] first block of each cluster            */
  int64_t arena_rows, slot_cap;
  int32_t block_tokens, pstride; /* pieces: 2 ints (in HBM) or 4 (offload)      */
  /* exact selection (index.py:74-75): fp64 queries for the exact re-scoring
   * (optional; NULL = the fp32 q, exact when q is fp32-representable) and the
   * scratch of the tie-safe fallback (exact scores of every row + radix select,
   * csrc/exact_select.cuh) taken when the error band overflows */
  const double* q64;  /* [U, G, d] or NULL                                      */
  double* xscr;       /* [U, G, m_cap] (NULL: overflow -> status, no fallback)  */
  int32_t* xcount;    /* [1] number of (unit, head) fallbacks, or NULL          */
} wk_step_view;

typedef struct wk_zone_params {
  int32_t G, d, blas_threads;
  double retrieval_fraction;  /* IndexConfig.retrieval_fraction  (config.py:26) */
  double estimation_fraction; /* IndexConfig.estimation_fraction (config.py:27) */
  int32_t tail_denominator_only; /* IndexConfig.tail_mode                      */
  int32_t denominator_eq2;       /* EngineConfig.denominator_mode              */
  int32_t score_mode;            /* 1: the C32 scan accumulated in fp64 (the
                                    error bound select_v6 uses)                */
  int32_t piece_rows;            /* rows per retrieval piece, <= the attention
                                    chunk rows (16 for bf16 stores; 0: 16 for
                                    G <= 4, 8 for G <= 8, valid for both)      */
} wk_zone_params;

/* Device block cache (the wave buffer), one state machine per cache unit
 * (block_cache.py:52-225).  Cache unit = (unit, head) reproduces the
 * reference's per-head HeadEngine exactly; cache unit = kv-head unit serves
 * the union access stream of its GQA group.  Arrays sized by the caller. */
typedef struct wk_cache_view {
  int32_t* nblk;      /* [C, m_cap] slow-tier blocks per cluster (store.py:38-45) */
  int32_t* slot_off;  /* [C, m_cap] offset of the cluster's slot list           */
  int32_t* slot_ids;  /* [C, slot_cap] fast-tier slot ids (ClusterDescriptor)   */
  uint8_t* cached;    /* [C, m_cap]                                             */
  int32_t* prev;      /* [C, m_cap] LRU list (oldest first)                     */
  int32_t* next;
  int32_t* touched;   /* [C, m_cap] step stamp of the last access               */
  int64_t* last_access; /* [C, m_cap] ClusterDescriptor.last_access_step        */
  int32_t* lru_ht;    /* [C, 2] head, tail                                      */
  int32_t* heap;      /* [C, heap_cap] free slot ids (min-heap)                 */
  int32_t* heap_n;    /* [C]                                                    */
  int32_t* next_slot; /* [C]                                                    */
  int64_t* capacity;  /* [C] capacity_blocks                                    */
  int64_t* occupied;  /* [C]                                                    */
  int64_t* counters;  /* [C, 8] hits, misses, bytes_slow_to_fast,
                         bytes_fast_internal, store bytes_read_total, evictions,
                         admissions, rejections                                 */
  int32_t* ids;       /* [C, ids_cap] this step's access stream (rank order)    */
  int32_t* n_ids;     /* [C]                                                    */
  uint8_t* snapshot;  /* [C, ids_cap] residency before the commit               */
  int32_t* events;    /* [C, ev_cap, 4] (type, step, cluster, aux) or NULL      */
  int64_t* ev_n;      /* [C]                                                    */
  const int32_t* m_live; /* [U] registered clusters per unit                    */
  int64_t m_cap, slot_cap, heap_cap, ids_cap, ev_cap;
  int32_t block_bytes, token_bytes;
} wk_cache_view;

/* Offload block cache (cache_v2.cu): per kv-head unit, the union access
 * stream of the GQA group, tierkv BlockCache lookup/assemble/commit
 * (block_cache.py:79-213) in parallel, then the attention pieces (hits from
 * the slot arena, misses from the pinned host store, admitted misses written
 * through by the attention kernel). */
typedef struct wk_cache2_view {
  int32_t* nblk; int32_t* slot_off; int32_t* slot_ids; uint8_t* cached;
  int32_t* touched; int32_t* first; int32_t* lru; int32_t* lru_tmp; int32_t* lru_n;
  int32_t* freel; int32_t* free_n; int32_t* next_slot; int64_t* capacity; int64_t* occupied;
  int64_t* counters;  /* [U, 8] hits, misses, bytes_slow_to_fast, bytes_fast_internal,
                         store bytes_read_total, evictions, admissions, rejections */
  int32_t* ids; int32_t* n_ids; uint8_t* snapshot; int32_t* scratch;
  const int32_t* m_live;
  int64_t m_cap, slot_cap, lru_cap, ids_cap;
  int32_t block_bytes, token_bytes, block_tokens;
  int32_t piece_rows; /* rows per attention piece (wk_zone_params.piece_rows)  */
} wk_cache2_view;

int wk_version(void);

/* Segmented spherical k-means + finalize + store packing for a batch of
 * segments.  Replaces ClusterIndex.segmented_build / update -> _cluster_batch
 * -> spherical_kmeans + finalize_cluster + SlowTierStore.pack_cluster
 * (index.py:143-186, clustering.py:66-101, index.py:43-58, store.py:69-90).
 * `segs` is a HOST array; copied to scratch->segs_dev. */
int wk_kmeans_segments(const wk_index_view* ix, const wk_segment* segs, int n_segs,
                       const wk_build_scratch* scratch, int d, int store_bf16,
                       int kmeans_iters, int blas_threads, int max_L, int max_k,
                       void* stream);

/* Append one decode token per unit to the steady buffer
 * (HeadEngine._append_tokens + buffer.append, engine.py:178-182).  A full
 * steady buffer writes nothing and sets *status (may be NULL) to 7. */
int wk_append_tokens(const wk_steady_view* st, const float* k_new, const float* v_new, int U,
                     int d, int store_bf16, int* status, void* stream);

/* Centroid scoring over GQA groups + exact zone planning + per-unit unions.
 * Replaces ClusterIndex.rank -> rank_clusters and plan_zones
 * (index.py:61-93, 188-189). */
int wk_score_topk(const wk_index_view* ix, const wk_step_view* sv, const wk_zone_params* zp,
                  int U, int m_max, void* stream);

/* Fused tripartite attention: steady + retrieved clusters (exact) +
 * estimation zone (centroids) + LSE merge.  Replaces exact_partial,
 * estimate_partial, tail_denominator_partial, merge and
 * HeadEngine._final_output (attention.py:67-148, engine.py:150-172).
 * S = CTAs per unit. */
int wk_tripartite_attn(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                       const wk_zone_params* zp, int U, int S, int store_bf16, void* stream);

/* Full-attention decode over every stored token of each unit (the comparator
 * and HeadEngine.oracle_step_output / oracle_attention, attention.py:55-64).
 * Uses sv->q, sv->part, sv->out, sv->logden, sv->cov; n_store[u] = live
 * store rows of unit u. */
int wk_full_attn(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                 const int32_t* n_store, int U, int G, int d, int S, int store_bf16, void* stream);

/* One lookup + assemble accounting + commit_update for every cache unit
 * (BlockCache.lookup / assemble / commit_update, block_cache.py:79-213).
 * rlist/nr come from wk_score_topk; n_steady = steady tokens per unit.
 * union_mode=0: C = U*G cache units (per head); 1: C = U (GQA union). */
int wk_cache_step(const wk_cache_view* cv, const int32_t* rlist, const int32_t* nr,
                  const int32_t* n_steady, int r_cap, int G, int union_mode, int64_t step,
                  int C, int* status, void* stream);

/* recall@k of each (unit, head) (metrics.py:8-26 as used by
 * engine.py:200-203): exact top-k tokens by fp64 q.K (dgemv recipe, ties to
 * the lower token id) intersected with the retrieved set (steady tokens +
 * this step's retrieval clusters).  Scratch: s [U*G, n_cap] f32,
 * rflag [U*G, s_cap] u8.  recall_out [U*G] f32. */
int wk_recall_at_k(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                   const int32_t* n_store, int U, int G, int d, int metrics_k, int blas_threads,
                   float* s_scratch, uint8_t* rflag, int64_t n_cap, int store_bf16,
                   float* recall_out, void* stream);

/* One decode step of the in-HBM path in one call: append (fused into the
 * zone-planning kernel), centroid scan, exact zone planning + unions,
 * tripartite attention and merge (HeadEngine.decode_step minus the metrics,
 * engine.py:174-210). */
int wk_decode_step(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                   const wk_zone_params* zp, const float* k_new, const float* v_new, int U, int m_max, int S,
                   int store_bf16, void* stream);

/* The two halves of wk_score_topk, for pipelining unit groups on streams:
 * the centroid scan (HBM-bound) and the exact zone planning + unions
 * (latency-bound; optionally with the fused token append). */
int wk_centroid_scan(const wk_index_view* ix, const wk_step_view* sv, const wk_zone_params* zp, int U, int m_max,
                     void* stream);
int wk_plan_zones(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                  const wk_zone_params* zp, const float* k_new, const float* v_new, int U, int m_max,
                  int store_bf16, void* stream);

/* The BlockCache phases as separate calls on cache unit 0 of `cv` (the
 * function-level API: BlockCache.lookup / assemble / commit_update,
 * block_cache.py:79-96, 98-143, 163-213).  phase bits: 1 lookup (ids
 * de-duplicated in place, snapshot -> snap_out, *n_out distinct ids, hit /
 * miss counters, access event), 2 assemble byte accounting (n_steady steady
 * tokens, then ids in the given order with snap_in), 4 commit_update(ids,
 * snap_in, step).  Unknown ids set *status (IntegrityError). */
int wk_cache_phase(const wk_cache_view* cv, int32_t* ids, const uint8_t* snap_in, int n, int64_t n_steady,
                   int64_t step, int phase, uint8_t* snap_out, int32_t* n_out, int* status, void* stream);

/* Function-level attention / ranking in fp64 on the device (tierkv
 * attention.py:55-148, index.py:43-76, metrics.py:8-16).  One partial:
 * mode 0 exact_partial over rows = K, vals = V; 1 estimate_partial over
 * rows = C (or given scores), vals = value sums, sizes; 2
 * tail_denominator_partial.  out [3 + d] = running_max, denominator, count,
 * numerator[d]; scratch: n doubles. */
int wk_attn_partial_f64(const double* q, const double* rows, const double* vals, const double* sizes,
                        const double* scores, int n, int d, int mode, int blas_threads, double* scratch,
                        double* out, void* stream);
/* merge (attention.py:115-148) of P partials [P, 3 + d]: out [2d + 3] =
 * output[d], exact-denominator coverage (1 if exact_mask NULL),
 * log-denominator, merged denominator, merged numerator[d] (merged_sums).
 * All partials empty sets *status (ConfigError). */
int wk_merge_f64(const double* parts, int P, int d, const uint8_t* exact_mask, double* out, int* status,
                 void* stream);
/* rank_clusters / top_k_token_ids: exact dgemv-recipe scores of m rows
 * (scores [m]) and, if order != NULL, the full lexsort((arange, -scores))
 * order [m]. */
int wk_rank_f64(const double* q, const double* rows, int m, int d, int blas_threads, double* scores,
                int64_t* order, void* stream);
/* finalize_cluster sums: for k clusters with members[offsets[c]..offsets[c+1])
 * (row indices into keys / values [., d] fp32), fp64 centroid = mean and
 * value_sum = sum, in member order (index.py:43-58). */
int wk_cluster_sums_f64(const float* keys, const float* values, const int32_t* members, const int32_t* offsets,
                        int k, int d, double* centroids, double* value_sums, void* stream);

/* Offload cache step + attention pieces for U kv-head units (one CTA each). */
int wk_cache_offload_step(const wk_cache2_view* cv, const wk_index_view* ix, const wk_steady_view* st,
                          const wk_step_view* sv, int G, int64_t step, int U, void* stream);

/* Pinned, device-mapped host memory for the offloaded store (cudaHostAlloc
 * mapped|portable); the returned pointer is valid on host and device. */
int wk_host_alloc(size_t bytes, void** ptr);
int wk_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif
