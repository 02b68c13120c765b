// cache_v2.cu -- the wave buffer (block cache over pinned host KV) for the
// offload path.  One CTA per kv-head unit runs tierkv BlockCache's lookup +
// assemble accounting + commit_update (block_cache.py:79-213) on the union
// access stream of its GQA group, in parallel, and then emits the unit's
// attention pieces: hits read their blocks from the HBM slot arena, misses
// read the cluster-contiguous host store (zero-copy TMA over the host link)
// and, when admitted, are written through into their new slots by attend_v4.
//
// Equivalence with the sequential state machine (cache.cu, bit-exact vs the
// reference event stream): the LRU list is an array in LRU order.  Touched
// hits move to the MRU end in rank order, then misses are admitted in rank
// order.  Evictions take the oldest untouched clusters: with E the untouched
// cached clusters in LRU order and SE their block prefix sums, the k-th
// admitted miss needs the shortest prefix p with SE[p] >= N_k + need_k - free
// (N_k = blocks admitted before it) -- a lower_bound, parallel over misses.
// Misses larger than the capacity are rejected (block_cache.py:181).  From
// the first miss that cannot fit even with E exhausted, one thread finishes
// the step sequentially exactly like the reference.  Hits, misses, bytes,
// evictions, admissions, rejections, LRU order and residency are therefore
// the reference's; physical slot ids are internal (any free slot may serve).
#include "common.cuh"
#include "decode_internal.h"

namespace wk {

using Cache2View = ::wk_cache2_view;

constexpr int C2_T = 512;

// block exclusive scan over C2_T threads; ws: >= 17 entries of shared memory
template <typename V>
WK_DEVINL V c2_scan(V v, V* tot, V* ws) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = C2_T / 32;
  V x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    const V s = lane < nw ? ws[lane] : (V)0;
    V iv = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const V y = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += y;
    }
    if (lane < nw) ws[lane] = iv - s;
    if (lane == nw - 1) ws[16] = iv;
  }
  __syncthreads();
  const V ex = ws[w] + x - v;
  *tot = ws[16];
  __syncthreads();
  return ex;
}

// [lo, hi) of thread t when n items are split into contiguous ranges
WK_DEVINL void c2_range(int n, int& lo, int& hi) {
  lo = (int)((long long)n * threadIdx.x / C2_T);
  hi = (int)((long long)n * (threadIdx.x + 1) / C2_T);
}

// grid = U, block = C2_T
__global__ void __launch_bounds__(C2_T) cache2_step_kernel(Cache2View cv, IndexView ix, SteadyView st, StepView sv,
                                                           int G, int64_t step) {
  const int u = blockIdx.x, t = threadIdx.x;
  __shared__ int64_t ws64[17];
  __shared__ int ws32[17];
  __shared__ int s_kx;
  __shared__ long long s_req;
  const int r = sv.nr[u];
  const int32_t stamp = (int32_t)(step + 1);
  int32_t* first = cv.first + (size_t)u * cv.m_cap;
  int32_t* touched = cv.touched + (size_t)u * cv.m_cap;
  uint8_t* cached = cv.cached + (size_t)u * cv.m_cap;
  const int32_t* nb = cv.nblk + (size_t)u * cv.m_cap;
  int32_t* ids = cv.ids + (size_t)u * cv.ids_cap;
  uint8_t* snap = cv.snapshot + (size_t)u * cv.ids_cap;
  int64_t* cnt = cv.counters + (size_t)u * 8;
  int32_t* scr = cv.scratch + (size_t)u * (cv.lru_cap + 1 + 2 * cv.ids_cap);
  int32_t* SE = scr;                            // [nE + 1]
  int32_t* Mids = scr + cv.lru_cap + 1;         // misses (positions into ids), rank order
  int32_t* MN = Mids + cv.ids_cap;              // admissible blocks before miss k
  const int64_t bsz = cv.block_bytes;
  auto rl = [&](int i) { return sv.rlist[((size_t)u * G + (i % G)) * sv.r_cap + i / G]; };

  // ---- 1. union access stream: rank positions round-robin over the G
  //         heads, first occurrence kept (cache.cu union_mode) ----
  const int K = r * G;
  for (int i = t; i < K; i += C2_T) atomicMin(first + rl(i), i);
  __syncthreads();
  int k0, k1;
  c2_range(K, k0, k1);
  int mine = 0;
  for (int i = k0; i < k1; i++) mine += first[rl(i)] == i;
  int n;
  int pos = c2_scan<int>(mine, &n, ws32);
  if (n > cv.ids_cap) {
    if (t == 0) set_status(sv.status, kErrUnion);
    for (int i = t; i < K; i += C2_T) first[rl(i)] = 0x7fffffff;
    return;
  }
  for (int i = k0; i < k1; i++)
    if (first[rl(i)] == i) ids[pos++] = rl(i);
  __syncthreads();
  // ---- 2. lookup (snapshot before the commit) + assemble accounting ----
  int64_t hit = 0, fast = 0, slow = 0;
  for (int i = t; i < n; i += C2_T) {
    const int cl = ids[i];
    first[cl] = 0x7fffffff;
    if (cl < 0 || cl >= cv.m_live[u]) { set_status(sv.status, kErrUnknownCluster); snap[i] = 1; continue; }
    const uint8_t s = cached[cl];
    snap[i] = s;
    touched[cl] = stamp;
    hit += s;
    if (s) fast += (int64_t)nb[cl] * bsz; else slow += (int64_t)nb[cl] * bsz;
  }
  int64_t H, F, S;
  c2_scan<int64_t>(hit, &H, ws64);
  c2_scan<int64_t>(fast, &F, ws64);
  c2_scan<int64_t>(slow, &S, ws64);
  // ---- 3. evictable set E: untouched cached clusters, LRU order ----
  int32_t* lru = cv.lru + (size_t)u * cv.lru_cap;
  int32_t* E = cv.lru_tmp + (size_t)u * cv.lru_cap;
  const int nl = cv.lru_n[u];
  int l0, l1;
  c2_range(nl, l0, l1);
  int ke = 0;
  for (int j = l0; j < l1; j++) ke += touched[lru[j]] != stamp;
  int nE;
  int pe = c2_scan<int>(ke, &nE, ws32);
  int sb = 0;
  for (int j = l0; j < l1; j++) {
    const int v = lru[j];
    if (touched[v] != stamp) { E[pe++] = v; sb += nb[v]; }
  }
  {
    int tot;
    int base = c2_scan<int>(sb, &tot, ws32);
    pe -= ke;
    for (int j = l0; j < l1; j++) {
      const int v = lru[j];
      if (touched[v] != stamp) { SE[pe++] = base; base += nb[v]; }
    }
    if (t == 0) SE[nE] = tot;
  }
  // ---- 4. misses in rank order; admissible blocks before each ----
  const int64_t cap = cv.capacity[u];
  const int64_t occ0 = cv.occupied[u];
  const int64_t free0 = cap - occ0;
  int q0, q1;
  c2_range(n, q0, q1);
  int km = 0, kb = 0;
  for (int i = q0; i < q1; i++)
    if (!snap[i]) { km++; const int need = nb[ids[i]]; kb += need <= cap ? need : 0; }
  int nm, totb;
  int pm = c2_scan<int>(km, &nm, ws32);
  int pb = c2_scan<int>(kb, &totb, ws32);
  for (int i = q0; i < q1; i++)
    if (!snap[i]) {
      Mids[pm] = i;
      MN[pm] = pb;
      pm++;
      const int need = nb[ids[i]];
      pb += need <= cap ? need : 0;
    }
  if (t == 0) s_kx = nm;
  __syncthreads();
  // first miss that cannot fit even with E fully evicted
  for (int k = t; k < nm; k += C2_T) {
    const int need = nb[ids[Mids[k]]];
    if (need <= cap && (int64_t)MN[k] + need - free0 > (int64_t)SE[nE]) atomicMin(&s_kx, k);
  }
  __syncthreads();
  const int kx = s_kx;
  // evictions of the closed form: p of the last admissible miss before kx
  if (t == 0) s_req = 0;
  __syncthreads();
  for (int k = t; k < kx; k += C2_T) {
    const int need = nb[ids[Mids[k]]];
    if (need <= cap) atomicMax(&s_req, (long long)MN[k] + need - free0);
  }
  __syncthreads();
  const long long req = s_req;
  int P = 0;
  if (req > 0) {
    int lo = 0, hi = nE;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((long long)SE[mid] >= req) hi = mid; else lo = mid + 1;
    }
    P = lo;
  }
  const int freed = SE[P];
  const int adm_tot = kx > 0 ? MN[kx - 1] + (nb[ids[Mids[kx - 1]]] <= cap ? nb[ids[Mids[kx - 1]]] : 0) : 0;
  // ---- 5. slots: pool = free list ++ slots of evicted E[0, P) ++ fresh ----
  int32_t* freel = cv.freel + (size_t)u * cv.slot_cap;
  int32_t* slots = cv.slot_ids + (size_t)u * cv.slot_cap;
  const int32_t* soff = cv.slot_off + (size_t)u * cv.m_cap;
  const int nfree = cv.free_n[u];
  const int nxt0 = cv.next_slot[u];
  auto pool = [&](int k) -> int32_t {
    if (k < nfree) return freel[k];
    k -= nfree;
    if (k < freed) {
      int lo = 0, hi = P - 1;  // last p with SE[p] <= k
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (SE[mid] <= k) lo = mid; else hi = mid - 1;
      }
      return slots[soff[E[lo]] + (k - SE[lo])];
    }
    return nxt0 + (k - freed);
  };
  for (int k = t; k < kx; k += C2_T) {
    const int cl = ids[Mids[k]];
    const int need = nb[cl];
    if (need > cap) continue;
    for (int j = 0; j < need; j++) slots[soff[cl] + j] = pool(MN[k] + j);
  }
  const int pool_n = nfree + freed;
  const int used = min(adm_tot, pool_n);
  const int rem = pool_n - used;
  // unused pool tail -> free list (reads precede writes: read index >= write index + used)
  for (int base = 0; base < rem; base += C2_T) {
    const int j = base + t;
    const int32_t v = j < rem ? pool(used + j) : 0;
    __syncthreads();
    if (j < rem) freel[j] = v;
  }
  __syncthreads();
  // ---- 6. residency ----
  for (int j = t; j < P; j += C2_T) cached[E[j]] = 0;
  for (int k = t; k < kx; k += C2_T) {
    const int cl = ids[Mids[k]];
    if (nb[cl] <= cap) cached[cl] = 1;
  }
  // ---- 7. LRU: E[P..) ++ hits (rank order) ++ admitted misses (rank order) ----
  const int keep = nE - P;
  for (int j = t; j < keep; j += C2_T) lru[j] = E[P + j];
  int kh = 0;
  for (int i = q0; i < q1; i++) kh += snap[i];
  int nh;
  int ph = c2_scan<int>(kh, &nh, ws32);
  for (int i = q0; i < q1; i++)
    if (snap[i]) lru[keep + ph++] = ids[i];
  int a0, a1;
  c2_range(kx, a0, a1);
  int ka = 0;
  for (int k = a0; k < a1; k++) ka += nb[ids[Mids[k]]] <= cap;
  int na;
  int pa = c2_scan<int>(ka, &na, ws32);
  for (int k = a0; k < a1; k++)
    if (nb[ids[Mids[k]]] <= cap) lru[keep + nh + pa++] = ids[Mids[k]];
  __syncthreads();
  if (t == 0) {
    int rej = 0;
    for (int k = 0; k < kx; k++) rej += nb[ids[Mids[k]]] > cap;
    int64_t occ = occ0 - freed + adm_tot, adm_blocks = adm_tot;
    int evict = P, admit = na, ln = keep + nh + na, fl = rem, nx = nxt0 + max(0, adm_tot - pool_n);
    // ---- exhaustion tail (rare): the reference's loop, one thread ----
    int eh = P, drop = 0;  // E[eh..) still cached+untouched; they sit at lru[0..keep)
    for (int k = kx; k < nm; k++) {
      const int cl = ids[Mids[k]];
      const int need = nb[cl];
      if (need > cap) { rej++; continue; }
      while (cap - occ < need && eh < nE) {
        const int v = E[eh++];
        for (int j = 0; j < nb[v]; j++) freel[fl++] = slots[soff[v] + j];
        occ -= nb[v];
        cached[v] = 0;
        evict++;
        drop++;  // the oldest entry of lru
      }
      if (cap - occ < need) { rej++; continue; }
      for (int j = 0; j < need; j++) slots[soff[cl] + j] = fl ? freel[--fl] : nx++;
      occ += need;
      adm_blocks += need;
      cached[cl] = 1;
      lru[ln++] = cl;
      admit++;
    }
    if (drop)
      for (int j = 0; j + drop < ln; j++) lru[j] = lru[j + drop];
    cv.lru_n[u] = ln - drop;
    cv.free_n[u] = fl;
    cv.next_slot[u] = nx;
    if (occ > cap) set_status(sv.status, kErrCapacity);
    cv.occupied[u] = occ;
    cnt[0] += H;
    cnt[1] += n - H;
    cnt[2] += S;
    cnt[3] += F + adm_blocks * bsz + (int64_t)st.n[u] * cv.token_bytes;
    cnt[4] += S;
    cnt[5] += evict;
    cnt[6] += admit;
    cnt[7] += rej;
    cv.n_ids[u] = n;
  }
  __syncthreads();

  // ---- 8. attention pieces of the retrieval union (rank order) ----
  //   hit:  runs of consecutive arena slots, <= PR rows  (flag 1: arena)
  //   miss: host store rows, <= PR rows; admitted -> flag 2 (write-through)
  const int PR = cv.piece_rows > 0 ? cv.piece_rows : (G <= 4 ? 16 : 8);  // attention chunk rows
  const int bt = cv.block_tokens;
  const int* csize = ix.cl_size + (size_t)u * ix.m_cap;
  const int* coff = ix.cl_off + (size_t)u * ix.m_cap;
  const uint32_t* rb = sv.rbits + (size_t)u * G * sv.w_cap;
  auto count_pieces = [&](int i) {
    const int cl = ids[i], s = csize[cl];
    if (!snap[i]) return (s + PR - 1) / PR;
    int np = 0, b = 0;
    const int nbk = nb[cl];
    while (b < nbk) {
      int e = b + 1;
      while (e < nbk && slots[soff[cl] + e] == slots[soff[cl] + e - 1] + 1) e++;
      const int rows = min(s, e * bt) - b * bt;
      np += (rows + PR - 1) / PR;
      b = e;
    }
    return np;
  };
  int kp = 0;
  for (int i = q0; i < q1; i++) kp += count_pieces(i);
  int npc;
  int pp = c2_scan<int>(kp, &npc, ws32);
  if (npc > sv.pc_cap) {
    if (t == 0) { set_status(sv.status, kErrUnion); sv.cnt[u * 4 + 3] = 0; }
    return;
  }
  int4* pcs = reinterpret_cast<int4*>(sv.pieces) + (size_t)u * sv.pc_cap;
  for (int i = q0; i < q1; i++) {
    const int cl = ids[i], s = csize[cl];
    int mk = 0;
    for (int g = 0; g < G; g++) mk |= (int)((rb[(size_t)g * sv.w_cap + zb_word(cl)] >> zb_bit(cl)) & 1u) << g;
    if (!snap[i]) {
      const int fill = cached[cl] ? 2 : 0;
      for (int j = 0; j < s; j += PR)
        pcs[pp++] = make_int4(coff[cl] + j, min(PR, s - j) | (mk << 8) | (fill << 16), cl, j);
    } else {
      int b = 0;
      const int nbk = nb[cl];
      while (b < nbk) {
        int e = b + 1;
        while (e < nbk && slots[soff[cl] + e] == slots[soff[cl] + e - 1] + 1) e++;
        const int r0 = slots[soff[cl] + b] * bt, rows = min(s, e * bt) - b * bt;
        for (int j = 0; j < rows; j += PR)
          pcs[pp++] = make_int4(r0 + j, min(PR, rows - j) | (mk << 8) | (1 << 16), cl, b * bt + j);
        b = e;
      }
    }
  }
  if (t == 0) sv.cnt[u * 4 + 3] = npc;
}

}  // namespace wk
