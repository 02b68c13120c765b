// cache.cu -- the wave buffer's block cache on the device.
//
// Restates tierkv BlockCache (block_cache.py:52-225) per cache unit:
// residency snapshot as of the last commit (lookup, :79-96), assemble byte
// accounting (:98-143), then commit_update (:163-213): touched hits move to
// MRU in rank order, missed clusters are admitted all-or-nothing in rank order
// evicting least-recently-used untouched clusters, oversize/unfittable ones
// are rejected, slots are allocated smallest-free-id first (:147-161).
// One thread runs one cache unit's sequential state machine; cache units are
// independent and run in parallel (per (unit, head) = reference semantics, or
// per kv-head unit over the union access stream of its GQA group).
#include "common.cuh"
#include "cache_internal.h"

namespace wk {

struct CacheCtx {
  const CacheView& cv;
  int64_t c;  // cache unit
  __device__ int32_t* nb() const { return cv.nblk + c * cv.m_cap; }
  __device__ int32_t* so() const { return cv.slot_off + c * cv.m_cap; }
  __device__ int32_t* sl() const { return cv.slot_ids + c * cv.slot_cap; }
  __device__ uint8_t* ca() const { return cv.cached + c * cv.m_cap; }
  __device__ int32_t* pv() const { return cv.prev + c * cv.m_cap; }
  __device__ int32_t* nx() const { return cv.next + c * cv.m_cap; }
  __device__ int32_t* tc() const { return cv.touched + c * cv.m_cap; }
  __device__ int32_t* hp() const { return cv.heap + c * cv.heap_cap; }
  __device__ int64_t* la() const { return cv.last_access + c * cv.m_cap; }
};

__device__ __forceinline__ void lru_unlink(const CacheCtx& x, int32_t* st, int32_t v) {
  int32_t* p = x.pv();
  int32_t* n = x.nx();
  if (p[v] >= 0) n[p[v]] = n[v]; else st[0] = n[v];
  if (n[v] >= 0) p[n[v]] = p[v]; else st[1] = p[v];
  p[v] = n[v] = -1;
}
__device__ __forceinline__ void lru_append(const CacheCtx& x, int32_t* st, int32_t v) {
  int32_t* p = x.pv();
  int32_t* n = x.nx();
  p[v] = st[1];
  n[v] = -1;
  if (st[1] >= 0) n[st[1]] = v; else st[0] = v;
  st[1] = v;
}
__device__ __forceinline__ void heap_push(const CacheCtx& x, int32_t* st, int32_t v) {
  int32_t* h = x.hp();
  int i = st[2]++;
  h[i] = v;
  while (i > 0) {
    int pa = (i - 1) >> 1;
    if (h[pa] <= h[i]) break;
    int32_t t = h[pa]; h[pa] = h[i]; h[i] = t;
    i = pa;
  }
}
__device__ __forceinline__ int32_t heap_pop(const CacheCtx& x, int32_t* st) {
  int32_t* h = x.hp();
  int32_t top = h[0];
  int n = --st[2];
  h[0] = h[n];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, s = i;
    if (l < n && h[l] < h[s]) s = l;
    if (r < n && h[r] < h[s]) s = r;
    if (s == i) break;
    int32_t t = h[s]; h[s] = h[i]; h[i] = t;
    i = s;
  }
  return top;
}

__device__ __forceinline__ void push_event(const CacheView& cv, int64_t c, int32_t type, int64_t step,
                                           int32_t cl, int32_t aux) {
  if (!cv.events) return;
  int64_t i = cv.ev_n[c]++;
  if (i < cv.ev_cap) {
    int32_t* e = cv.events + (c * cv.ev_cap + i) * 4;
    e[0] = type; e[1] = (int32_t)step; e[2] = cl; e[3] = aux;
  }
}

// commit_update (block_cache.py:163-213) of one cache unit over its access
// stream ids[0..n) with the lookup snapshot snap[]; every id is stamped
// `stamp` in tc[] (the touched set).  st = (lru head, lru tail, heap size).
__device__ void commit_phase(const CacheCtx& x, const int32_t* ids, const uint8_t* snap, int n, int64_t step,
                             int32_t stamp, int32_t* st, int64_t* cnt, int* status) {
  const CacheView& cv = x.cv;
  const int64_t c = x.c;
  const int32_t* nb = x.nb();
  uint8_t* ca = x.ca();
  int32_t* tc = x.tc();
  const int64_t bsz = cv.block_bytes;
  int64_t* la = x.la();
  for (int i = 0; i < n; i++) {
    la[ids[i]] = step;
    if (snap[i]) { lru_unlink(x, st, ids[i]); lru_append(x, st, ids[i]); }
  }
  const int64_t cap = cv.capacity[c];
  int64_t occ = cv.occupied[c];
  int32_t nxt = cv.next_slot[c];
  for (int i = 0; i < n; i++) {
    if (snap[i]) continue;
    const int32_t cl = ids[i];
    if (ca[cl]) continue;  // admitted earlier in this commit (repeated id)
    const int64_t need = nb[cl];
    if (need > cap) { push_event(cv, c, 3, step, cl, 0); cnt[7]++; continue; }
    while (cap - occ < need) {
      int32_t v = st[0];
      if (v < 0 || tc[v] == stamp) break;  // untouched clusters precede touched ones
      int32_t* s = x.sl() + x.so()[v];
      for (int j = 0; j < nb[v]; j++) heap_push(x, st, s[j]);
      occ -= nb[v];
      ca[v] = 0;
      lru_unlink(x, st, v);
      push_event(cv, c, 1, step, v, 0);
      cnt[5]++;
    }
    if (cap - occ < need) { push_event(cv, c, 3, step, cl, 0); cnt[7]++; continue; }
    int32_t* s = x.sl() + x.so()[cl];
    for (int j = 0; j < need; j++) s[j] = st[2] ? heap_pop(x, st) : nxt++;
    occ += need;
    ca[cl] = 1;
    lru_append(x, st, cl);
    cnt[3] += need * bsz;
    cnt[6]++;
    push_event(cv, c, 2, step, cl, (int32_t)need);
  }
  if (occ > cap) set_status(status, kErrCapacity);
  cv.occupied[c] = occ;
  cv.next_slot[c] = nxt;
}

// grid = ceil(C / 64), block = 64; one thread per cache unit.
// ids for cache unit c: if union_heads > 1, the union (round-robin over rank
// positions of the G heads, first occurrence kept) of rlist[u, 0..G); else
// rlist[c] directly (c = u*G + g).
__global__ void cache_step_kernel(CacheView cv, const int32_t* __restrict__ rlist, const int32_t* __restrict__ nr,
                                  const int32_t* __restrict__ n_steady, int r_cap, int G, int union_mode,
                                  int64_t step, int C, int* status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  CacheCtx x{cv, c};
  const int u = union_mode ? (int)c : (int)(c / G);
  const int r = nr[u];
  const int32_t stamp = (int32_t)(step + 1);
  int32_t* ids = cv.ids + c * cv.ids_cap;
  uint8_t* snap = cv.snapshot + c * cv.ids_cap;
  int n = 0;
  int32_t* tc = x.tc();
  // ---- access stream (deduplicated, rank order) ----
  if (union_mode) {
    for (int pos = 0; pos < r; pos++)
      for (int g = 0; g < G; g++) {
        int32_t cl = rlist[((int64_t)u * G + g) * r_cap + pos];
        if (tc[cl] != stamp) { tc[cl] = stamp; ids[n++] = cl; }
      }
  } else {
    const int32_t* rl = rlist + (int64_t)c * r_cap;
    for (int i = 0; i < r; i++) {
      int32_t cl = rl[i];
      if (tc[cl] != stamp) { tc[cl] = stamp; ids[n++] = cl; }
    }
  }
  cv.n_ids[c] = n;
  int32_t st[3];  // head, tail, heap_n
  st[0] = cv.lru_ht[c * 2]; st[1] = cv.lru_ht[c * 2 + 1]; st[2] = cv.heap_n[c];
  int64_t* cnt = cv.counters + c * 8;
  const int32_t* nb = x.nb();
  uint8_t* ca = x.ca();
  const int64_t bsz = cv.block_bytes;
  // ---- lookup (snapshot as of the last commit) ----
  int64_t hits = 0;
  for (int i = 0; i < n; i++) {
    if (ids[i] < 0 || ids[i] >= cv.m_live[u]) { set_status(status, kErrUnknownCluster); return; }
    snap[i] = ca[ids[i]];
    hits += snap[i];
  }
  cnt[0] += hits;
  cnt[1] += n - hits;
  push_event(cv, c, 0, step, n, (int32_t)hits);
  // ---- assemble accounting ----
  cnt[3] += (int64_t)n_steady[u] * cv.token_bytes;
  for (int i = 0; i < n; i++) {
    int64_t b = nb[ids[i]];
    if (snap[i]) cnt[3] += b * bsz;
    else { cnt[2] += b * bsz; cnt[4] += b * bsz; }
  }
  // ---- commit_update ----
  commit_phase(x, ids, snap, n, step, stamp, st, cnt, status);
  cv.lru_ht[c * 2] = st[0];
  cv.lru_ht[c * 2 + 1] = st[1];
  cv.heap_n[c] = st[2];
}

// The BlockCache phases as separate calls on cache unit 0 (the function-level
// API, block_cache.py:79-213); one thread.  ids[0..n) as the caller passes them.
//   phase 1 lookup(ids, step): de-duplicate (first occurrence), validate,
//     snapshot -> snap_out[0..n_out), hit / miss counters, access event;
//     *n_out = distinct ids (written back over ids[]).
//   phase 2 assemble accounting: steady bytes + per id (rank order, as given)
//     hit -> fast internal, miss -> slow-to-fast + store read bytes.
//   phase 4 commit_update(ids, snapshot, step).
__global__ void cache_phase_kernel(CacheView cv, int32_t* ids, const uint8_t* snap_in, int n, int64_t n_steady,
                                   int64_t step, int phase, uint8_t* snap_out, int32_t* n_out, int* status) {
  if (threadIdx.x || blockIdx.x) return;
  CacheCtx x{cv, 0};
  int64_t* cnt = cv.counters;
  const int32_t* nb = x.nb();
  uint8_t* ca = x.ca();
  const int64_t bsz = cv.block_bytes;
  if (phase & 1) {
    int k = 0;
    for (int i = 0; i < n; i++) {
      const int32_t cl = ids[i];
      if (cl < 0 || cl >= cv.m_live[0]) { set_status(status, kErrUnknownCluster); return; }
      bool dup = false;
      for (int j = 0; j < k; j++) dup |= ids[j] == cl;
      if (!dup) ids[k++] = cl;
    }
    int64_t hits = 0;
    for (int i = 0; i < k; i++) {
      snap_out[i] = ca[ids[i]];
      hits += snap_out[i];
    }
    cnt[0] += hits;
    cnt[1] += k - hits;
    push_event(cv, 0, 0, step, k, (int32_t)hits);
    *n_out = k;
  }
  if (phase & 2) {
    cnt[3] += n_steady * cv.token_bytes;
    for (int i = 0; i < n; i++) {
      const int64_t b = nb[ids[i]];
      if (snap_in[i]) cnt[3] += b * bsz;
      else { cnt[2] += b * bsz; cnt[4] += b * bsz; }
    }
  }
  if (phase & 4) {
    const int32_t stamp = (int32_t)(step + 1) ^ 0x40000000;  // distinct from the fused kernel's stamps
    int32_t* tc = x.tc();
    for (int i = 0; i < n; i++) tc[ids[i]] = stamp;
    int32_t st[3] = {cv.lru_ht[0], cv.lru_ht[1], cv.heap_n[0]};
    commit_phase(x, ids, snap_in, n, step, stamp, st, cnt, status);
    for (int i = 0; i < n; i++) tc[ids[i]] = 0;  // the touched set lives for one commit
    cv.lru_ht[0] = st[0];
    cv.lru_ht[1] = st[1];
    cv.heap_n[0] = st[2];
  }
}

}  // namespace wk
