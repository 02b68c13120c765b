// abi.cu -- extern "C" entry points (include/wavekv.h) launching the
// sm_100a kernels on the caller's stream.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "decode_internal.h"
#include "cache_internal.h"

namespace wk {
// kmeans.cu
__global__ void km_prep_kernel(const SegDesc*, float*, int, __half*);
__global__ void km_seed_kernel(const SegDesc*, const float*, float*, float*, int, int, int);
__global__ void km_seed_v2_kernel(const SegDesc*, const float*, float*, float*, int, int, int, const __half*, int);
__global__ void km_seed_v3_kernel(const SegDesc*, int, const float*, float*, float*, int, int, const __half*, int);
constexpr int KS3_W = 4;  // kmeans.cu: segments (warps) per CTA of km_seed_v3
__global__ void km_assign_kernel(const SegDesc*, const float*, const float*, int32_t*, int);
template <int KS>
__global__ void km_assign_tc_kernel(const SegDesc*, const float*, const float*, int32_t*);
__global__ void km_assign_small_kernel(const SegDesc*, const float*, const float*, int32_t*, int);
__global__ void km_update_kernel(const SegDesc*, const float*, float*, int32_t*, int32_t*, float*, int, int);
template <typename T>
__global__ void km_finalize_kernel(const SegDesc*, const int32_t*, int32_t*, IndexView, int, int*, int);
// decode.cu
template <typename T>
__global__ void append_kernel(SteadyView, const float*, const float*, int, int*);
__global__ void score_kernel(IndexView, StepView, int, int);
__global__ void select_kernel(IndexView, StepView, SelParams);
__global__ void union_kernel(IndexView, StepView);
template <typename T, bool FULL>
__global__ void attend_kernel(IndexView, SteadyView, StepView, AttnParams, const int32_t*);
__global__ void merge_kernel(StepView, AttnParams, int);
size_t select_smem_bytes();
// select_v6.cu / attend_v4.cu / score_v5.cu
template <int CAND, bool SMS, int GM>
__global__ void select_v6_kernel(IndexView, StepView, SelParams);
size_t select_v6_dyn_smem(int m_max, bool sms, int cand);
template <typename T, int DPL, int HS, bool FULL, bool OFF>
__global__ void attend_v4_kernel(IndexView, SteadyView, StepView, AttnParams, const int32_t*, int);
template <typename T, int DPL, int HS, bool FULL>
size_t attend_v4_smem();
template <typename T, int DPL, int HS>
int attend_v4_warps();
template <bool FULL, int DL>
__global__ void att4_merge_kernel(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int);
template <int D, int HS, bool FULL, bool OFF, bool ROWS>
__global__ void attend_v5_kernel(IndexView, SteadyView, StepView, AttnParams, const int32_t*, int);
template <int D, int HS>
size_t attend_v5_smem();
template <int D, int HS>
int attend_v5_warps();
template <int D, int HS, bool FULL, bool OFF, bool ROWS>
__global__ void attend_v6_kernel(IndexView, SteadyView, StepView, AttnParams, const int32_t*, int,
                                 const __grid_constant__ CUtensorMap);
template <int D, int HS>
size_t attend_v6_smem();
template <int D, int HS>
int attend_v6_warps();
template <int D, int HS>
int attend_v6_consumers();
template <int D, int HS>
int attend_v6_chunk_rows();
template <bool FULL, int DL>
__global__ void att6_merge_kernel(SteadyView, StepView, AttnParams, const int32_t*, int, int, int, int, int);
__global__ void km_assign_tc5_kernel(const SegDesc*, const float*, const float*, int32_t*, const __nv_bfloat16*);
__global__ void km_pack_c5_kernel(const SegDesc*, const float*, __nv_bfloat16*);
constexpr int KS_CK = 8192 / 32 + 4;  // km_seed_v2 cumsum checkpoint slots (kmeans.cu)
constexpr size_t K5_SMEM_BYTES = 2 * 128 * 128 * 2 + 2 * 256 * 128 * 2 + 64;
template <int EPL>
__global__ void km_prep_v2_kernel(const SegDesc*, float*, __half*);
// cache_v2.cu
__global__ void cache2_step_kernel(wk_cache2_view, IndexView, SteadyView, StepView, int, int64_t);
// metrics.cu
template <typename T>
__global__ void recall_kernel(IndexView, SteadyView, StepView, const int32_t*, int, int, int, int, float*,
                              uint8_t*, int64_t, float*);
size_t recall_smem_bytes();
// cache.cu
__global__ void cache_step_kernel(CacheView, const int32_t*, const int32_t*, const int32_t*, int, int, int,
                                  int64_t, int, int*);
__global__ void cache_phase_kernel(CacheView, int32_t*, const uint8_t*, int, int64_t, int64_t, int, uint8_t*,
                                   int32_t*, int*);
}  // namespace wk

using namespace wk;

#define WK_CHECK_LAUNCH()                          \
  do {                                             \
    cudaError_t e_ = cudaGetLastError();           \
    if (e_ != cudaSuccess) return WK_ECUDA;        \
  } while (0)

// cudaFuncSetAttribute is per device: run each configuration once per device
// (a process may drive several GPUs).
static int current_device() {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess ? d : 0;
}
struct PerDevice {
  unsigned long long done = 0;  // devices 0..63
  bool needed() const { const int d = current_device(); return d >= 64 || !((done >> d) & 1ull); }
  void mark() { const int d = current_device(); if (d < 64) done |= 1ull << d; }
};
static PerDevice g_smem_cfg;
static int configure_smem() {
  if (!g_smem_cfg.needed()) return 0;
  // opt in to large dynamic shared memory where the kernels need it
  if (cudaFuncSetAttribute(km_seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_seed_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_assign_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K5_SMEM_BYTES) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_finalize_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(km_finalize_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)select_smem_bytes()) != cudaSuccess) return WK_ECUDA;
  const int at = (int)attend_smem_bytes(256, 4);
  if (cudaFuncSetAttribute(attend_kernel<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, at) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(attend_kernel<__nv_bfloat16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, at) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(attend_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, at) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(attend_kernel<__nv_bfloat16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, at) != cudaSuccess) return WK_ECUDA;
  const int rs = (int)recall_smem_bytes();
  if (cudaFuncSetAttribute(recall_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, rs) != cudaSuccess) return WK_ECUDA;
  if (cudaFuncSetAttribute(recall_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, rs) != cudaSuccess) return WK_ECUDA;
  g_smem_cfg.mark();
  return 0;
}

static int head_slots(int G) { return G <= 4 ? 4 : 8; }
// ---- fast pipeline: score_v5 (FP64 tensor cores), select_v6, attend_v4 ----
static int sm_count() {
  static int n[64] = {0};
  const int dev = current_device();
  int* slot = dev < 64 ? &n[dev] : nullptr;
  if (slot && *slot) return *slot;
  int c = 0;
  if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0) c = 1;
  if (slot) *slot = c;
  return c;
}
// the token append fused into the zone-planning kernel (wk_decode_step /
// wk_plan_zones); passed explicitly down to the launcher
struct AppendArgs { int on; const float* k; const float* v; SteadyView st; int bf16; };
static bool v6_ok(const wk_index_view* ix, const wk_step_view* sv, int d) {
  return (d == 64 || d == 128) && sv->rbits && sv->ebits && sv->pieces && sv->woff && sv->sel_done && ix->Cmax;
}

// Launch with programmatic dependent launch (the kernel may be scheduled while
// the preceding kernel in the stream drains; it calls pdl_wait() before touching
// anything that kernel wrote) and, optionally, a thread-block cluster.
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             int cluster, Args... args) {
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[n].val.programmaticStreamSerializationAllowed = 1;
  n++;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    n++;
  }
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  lc.attrs = at;
  lc.numAttrs = n;
  return cudaLaunchKernelEx(&lc, kernel, args...);
}

template <int KG>
static int launch_score_v5(const IndexView& ix, const StepView& sv, int G, int U, int m_max, cudaStream_t s) {
  const long long groups = (m_max + 7) / 8;
  // short warp ranges (~6 eight-row groups per warp, many CTAs in flight) balance the
  // HBM stream better than one exact wave of long ranges: measured 2,146 -> 2,218 tok/s
  // (profiles/r1_attend_sweep.txt).
  constexpr int gpw_t = 6;
  const long long gpw = gpw_t;
  const long long cpu = (groups + gpw * 4 - 1) / (gpw * 4);
  dim3 grid((unsigned)cpu, U);
  const cudaError_t e = launch_ex(score_v5_kernel<KG>, grid, dim3(128), 0, s, 1, ix, sv, G, (int)gpw);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : WK_ECUDA;
}

template <int GM>
static int launch_select_v6_g(const IndexView& ix, const StepView& sv, const SelParams& p, int U, int m_max,
                            cudaStream_t s) {
  const double r_max = floor(p.retrieval_fraction * (double)m_max + 0.5) + 1;
  const int blocks = U * p.G;
  static PerDevice cfg;
  if (cfg.needed()) {
    if (cudaFuncSetAttribute(select_v6_kernel<512, true, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)select_v6_dyn_smem(16384, true, 512)) != cudaSuccess ||
        cudaFuncSetAttribute(select_v6_kernel<512, false, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)select_v6_dyn_smem(262144, false, 512)) != cudaSuccess ||
        cudaFuncSetAttribute(select_v6_kernel<2048, false, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)select_v6_dyn_smem(262144, false, 2048)) != cudaSuccess)
      return WK_ECUDA;
    cfg.mark();
  }
  if (m_max > 262144) return WK_ECONFIG;
  // the G CTAs of a unit form one thread-block cluster (the union runs over DSMEM)
  cudaError_t e;
  if (m_max <= 16384 && r_max <= 480)
    e = launch_ex(select_v6_kernel<512, true, GM>, dim3(blocks), dim3(256), select_v6_dyn_smem(m_max, true, 512), s,
                  p.G, ix, sv, p);
  else if (r_max <= 480)
    e = launch_ex(select_v6_kernel<512, false, GM>, dim3(blocks), dim3(256), select_v6_dyn_smem(m_max, false, 512), s,
                  p.G, ix, sv, p);
  else  // r_max > 1900: the exact path builds the ordered list in global memory
    e = launch_ex(select_v6_kernel<2048, false, GM>, dim3(blocks), dim3(256), select_v6_dyn_smem(m_max, false, 2048),
                  s, p.G, ix, sv, p);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : WK_ECUDA;
}

static int launch_select_v6(const IndexView& ix, const StepView& sv, const SelParams& p, int U, int m_max,
                            cudaStream_t s) {
  return p.G <= 4 ? launch_select_v6_g<4>(ix, sv, p, U, m_max, s) : launch_select_v6_g<8>(ix, sv, p, U, m_max, s);
}

template <typename T, int DPL, int HS, bool FULL, bool OFF>
static int launch_attend_v4(const IndexView& ix, const SteadyView& st, const StepView& sv, const AttnParams& p,
                            const int32_t* n_store, int U, int P, cudaStream_t s) {
  if (U > 1024) return WK_ECONFIG;
  const size_t sm = attend_v4_smem<T, DPL, HS, FULL>();
  static PerDevice cfg;
  if (cfg.needed()) {
    if (cudaFuncSetAttribute(attend_v4_kernel<T, DPL, HS, FULL, OFF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm) != cudaSuccess)
      return WK_ECUDA;
    cfg.mark();
  }
  const int warps = attend_v4_warps<T, DPL, HS>();
  if (launch_ex(attend_v4_kernel<T, DPL, HS, FULL, OFF>, dim3(P), dim3(warps * 32), sm, s, 1, ix, st, sv, p,
                n_store, U) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return WK_ECUDA;
  const int RG = HS == 4 ? 16 : 8;  // Att4Cfg::RG
  const cudaError_t e = launch_ex(att4_merge_kernel<FULL, DPL / 2>, dim3(U * p.G), dim3(128), 0, s, 1, st, sv, p,
                                  n_store, U, P * warps, RG, 0);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : WK_ECUDA;
}

// bf16 stores: attend_v5 (q.k and p.v on the tensor cores, chunk rows 16); the
// in-HBM path reads select_v6's retrieved-row list (ROWS), offload the pieces
template <int D, int HS, bool FULL, bool OFF, bool ROWS>
static int launch_attend_v5(const IndexView& ix, const SteadyView& st, const StepView& sv, const AttnParams& p,
                            const int32_t* n_store, int U, int P, cudaStream_t s) {
  if (U > 1024) return WK_ECONFIG;
  const size_t sm = attend_v5_smem<D, HS>();
  static PerDevice cfg;
  if (cfg.needed()) {
    if (cudaFuncSetAttribute(attend_v5_kernel<D, HS, FULL, OFF, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm) != cudaSuccess)
      return WK_ECUDA;
    cfg.mark();
  }
  const int warps = attend_v5_warps<D, HS>();
  if (launch_ex(attend_v5_kernel<D, HS, FULL, OFF, ROWS>, dim3(P), dim3(warps * 32), sm, s, 1, ix, st, sv, p,
                n_store, U) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return WK_ECUDA;
  const cudaError_t e = launch_ex(att4_merge_kernel<FULL, D / 32>, dim3(U * p.G), dim3(128), 0, s, 1, st, sv, p,
                                  n_store, U, P * warps, 16, ROWS ? 1 : 0);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : WK_ECUDA;
}

// 2-D tensor map of the fp32 value sums [rows, d] (box {d, 1}: the gather4 row
// source of attend_v6), cached per (pointer, rows, d)
static int vs_tensor_map(const float* ptr, long long rows, int d, CUtensorMap* out) {
  static std::mutex mu;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  struct Entry { const float* ptr; long long rows; int d, dev; CUtensorMap tm; };
  static Entry cache[64];
  static int n = 0, next = 0;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < n; i++)
    if (cache[i].ptr == ptr && cache[i].rows == rows && cache[i].d == d && cache[i].dev == dev) {
      *out = cache[i].tm;
      return 0;
    }
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return WK_ECUDA;
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  const cuuint32_t box[2] = {(cuuint32_t)d, 1};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return WK_ECUDA;
  Entry& e = cache[next];
  e = {ptr, rows, d, dev, tm};
  next = (next + 1) % 64;
  if (n < 64) n++;
  *out = tm;
  return 0;
}

// bf16 stores: attend_v6 (warp-specialised producer / consumer pipeline,
// tensor-core exact zones) + att6_merge
template <int D, int HS, bool FULL, bool OFF, bool ROWS>
static int launch_attend_v6(const IndexView& ix, const SteadyView& st, const StepView& sv, const AttnParams& p,
                            const int32_t* n_store, int U, int P, cudaStream_t s) {
  if (U > 1024) return WK_ECONFIG;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (!FULL && ix.VS32) {
    const int rc = vs_tensor_map(ix.VS32, (long long)U * ix.m_cap, D, &tm);
    if (rc) {
      fprintf(stderr, "wavekv: value-sum tensor map (%lld rows) could not be encoded\n", (long long)U * ix.m_cap);
      return rc;
    }
  }
  const size_t sm = attend_v6_smem<D, HS>();
  static PerDevice cfg;
  if (cfg.needed()) {
    if (cudaFuncSetAttribute(attend_v6_kernel<D, HS, FULL, OFF, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm) != cudaSuccess)
      return WK_ECUDA;
    cfg.mark();
  }
  const int warps = attend_v6_warps<D, HS>(), nc = attend_v6_consumers<D, HS>();
  const cudaError_t el = launch_ex(attend_v6_kernel<D, HS, FULL, OFF, ROWS>, dim3(P), dim3(warps * 32), sm, s, 1, ix,
                                   st, sv, p, n_store, U, tm);
  if (el != cudaSuccess) {
    fprintf(stderr, "wavekv: attend_v6 launch (smem %zu): %s\n", sm, cudaGetErrorString(el));
    return WK_ECUDA;
  }
#ifdef WK_EXP_NO_MERGE  // timing experiment only (tools/exp_bench.py): the merge's share of a step
  return 0;
#endif
  const cudaError_t e = launch_ex(att6_merge_kernel<FULL, D / 32>, dim3(U * p.G), dim3(128), 0, s, 1, st, sv, p,
                                  n_store, U, P, nc, ROWS ? 1 : 0, attend_v6_chunk_rows<D, HS>());
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : WK_ECUDA;
}

template <typename T, bool FULL>
static int dispatch_attend_v4(const IndexView& ix, const SteadyView& st, const StepView& sv, const AttnParams& p,
                              const int32_t* n_store, int U, int P, cudaStream_t s) {
  const int hs = head_slots(p.G);
  const bool off = !FULL && sv.pstride == 4;
  if constexpr (sizeof(T) == 2) {
    // bf16 rows are swizzled for attend_v5; the in-HBM path needs the row list
    if (!(FULL || off || sv.rtok_row)) return WK_ECONFIG;
#ifdef WK_ATTN_V5  // A/B experiments only: the per-warp-ring kernel
#define WK_LAUNCH5 launch_attend_v5
#else
#define WK_LAUNCH5 launch_attend_v6
#endif
#define WK_ATT5(D, HS)                                                                           \
  (FULL ? WK_LAUNCH5<D, HS, FULL, false, false>(ix, st, sv, p, n_store, U, P, s)                 \
        : (off ? WK_LAUNCH5<D, HS, FULL, !FULL, false>(ix, st, sv, p, n_store, U, P, s)          \
               : WK_LAUNCH5<D, HS, FULL, false, !FULL>(ix, st, sv, p, n_store, U, P, s)))
    if (p.d == 128) return hs == 4 ? WK_ATT5(128, 4) : WK_ATT5(128, 8);
    return hs == 4 ? WK_ATT5(64, 4) : WK_ATT5(64, 8);
#undef WK_ATT5
#undef WK_LAUNCH5
  } else {
#define WK_ATT4(DPL, HS)                                                                  \
  (off ? launch_attend_v4<T, DPL, HS, FULL, !FULL>(ix, st, sv, p, n_store, U, P, s)      \
       : launch_attend_v4<T, DPL, HS, FULL, false>(ix, st, sv, p, n_store, U, P, s))
    if (p.d == 128) return hs == 4 ? WK_ATT4(8, 4) : WK_ATT4(8, 8);
    return hs == 4 ? WK_ATT4(4, 4) : WK_ATT4(4, 8);
#undef WK_ATT4
  }
}

extern "C" {

int wk_version(void) { return 3; }

int wk_kmeans_segments(const wk_index_view* ix, const wk_segment* segs, int n_segs,
                       const wk_build_scratch* scr, int d, int store_bf16, int kmeans_iters,
                       int blas_threads, int max_L, int max_k, void* stream) {
  if (!ix || !segs || !scr || n_segs <= 0 || d <= 0 || d > 256 || (d & 3)) return WK_ECONFIG;
  if (configure_smem()) return WK_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(scr->segs_dev, segs, sizeof(wk_segment) * (size_t)n_segs, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return WK_ECUDA;
  const SegDesc* sd = scr->segs_dev;
  __half* p16 = (d % 16 == 0) ? (__half*)scr->P16 : nullptr;
  if (d == 32 || d == 64 || d == 128) {
    if (d == 128) km_prep_v2_kernel<4><<<n_segs, 512, 0, s>>>(sd, scr->P, p16);
    else if (d == 64) km_prep_v2_kernel<2><<<n_segs, 512, 0, s>>>(sd, scr->P, p16);
    else km_prep_v2_kernel<1><<<n_segs, 512, 0, s>>>(sd, scr->P, p16);
  } else {
    km_prep_kernel<<<n_segs, 256, d * sizeof(float), s>>>(sd, scr->P, d, p16);
  }
  WK_CHECK_LAUNCH();
  if ((d % 8) == 0 && d <= 128) {
    // v3: one warp per segment (the segments' serial chains side by side)
    const int K4 = (max_k + 3) & ~3;
    const size_t sm3 = (size_t)KS3_W * (d + K4 + KS_CK + 256) * sizeof(float);
    km_seed_v3_kernel<<<(n_segs + KS3_W - 1) / KS3_W, KS3_W * 32, sm3, s>>>(sd, n_segs, scr->P, scr->C, scr->md, d,
                                                                          blas_threads, p16, max_k);
  } else if ((d % 8) == 0) {
    // v2: 256 threads; centre + centre-distance bounds + (md, best) rows in smem
    // when they fit 72 KB (4 segments per SM at 120K: 52 KB)
    const int L4 = (max_L + 3) & ~3, K4 = (max_k + 3) & ~3;
    const size_t base = (size_t)(d + K4 + KS_CK) * sizeof(float);  // centre, bounds, cumsum checkpoints
    const size_t rows = (size_t)L4 * sizeof(float) + (size_t)L4 * sizeof(unsigned short);
    const bool in_smem = base + rows + 16 <= 72 * 1024;
    km_seed_v2_kernel<<<n_segs, 256, base + (in_smem ? rows : 0) + 16, s>>>(sd, scr->P, scr->C, scr->md, d,
                                                                             blas_threads, in_smem ? 1 : 0, p16,
                                                                             max_k);
  } else {
    const int smem_rows = ((200 * 1024) / 4 - d) / 2;
    const size_t seed_smem = (size_t)(d + 2 * (max_L <= smem_rows ? max_L : 0)) * sizeof(float);
    km_seed_kernel<<<n_segs, 512, seed_smem, s>>>(sd, scr->P, scr->C, scr->md, d, blas_threads,
                                                   max_L <= smem_rows ? smem_rows : 0);
  }
  WK_CHECK_LAUNCH();
  const dim3 ag((max_L + 63) / 64, n_segs);
  // Lloyd assignment: tensor-core first pass + exact verification when the
  // head dim tiles by 16 (<= 128), else the exact FFMA kernel
  const dim3 ag5((max_L + 127) / 128, n_segs);
  // d = 128 (k <= 512): tcgen05 contraction with the scores in TMEM
  // the pre-split centroids reuse the fp16 point copy (dead after seeding): (sum k + 8 n) * 2 rows
  long long sum_l = 0, sum_k = 0;
  for (int i = 0; i < n_segs; i++) { sum_l += segs[i].L; sum_k += segs[i].k; }
  const bool tc5 = d == 128 && max_k <= 512 && p16 != nullptr && (sum_k + 8LL * n_segs) * 2 <= sum_l;
  __nv_bfloat16* pk = reinterpret_cast<__nv_bfloat16*>(p16);
  auto assign = [&]() {
    if (tc5) {
      km_pack_c5_kernel<<<n_segs, 256, 0, s>>>(sd, scr->C, pk);
      km_assign_tc5_kernel<<<ag5, 256, K5_SMEM_BYTES, s>>>(sd, scr->P, scr->C, scr->A, pk);
    }
    else if (d == 128) km_assign_tc_kernel<8><<<ag, 128, 0, s>>>(sd, scr->P, scr->C, scr->A);
    else if (d == 64) km_assign_tc_kernel<4><<<ag, 128, 0, s>>>(sd, scr->P, scr->C, scr->A);
    else if (d == 32) km_assign_tc_kernel<2><<<ag, 128, 0, s>>>(sd, scr->P, scr->C, scr->A);
    else km_assign_kernel<<<ag, 256, (size_t)2 * d * 65 * sizeof(float), s>>>(sd, scr->P, scr->C, scr->A, d);
  };
  const size_t asmem = (size_t)2 * d * 65 * sizeof(float);
  const size_t usmem = (size_t)(2 * max_k + 1) * sizeof(int);
  const size_t upsmem = usmem + (size_t)16 * d * sizeof(float);  // + per-warp row scratch (512 threads)
  assign();
  km_assign_small_kernel<<<n_segs, 256, 0, s>>>(sd, scr->P, scr->C, scr->A, d);
  WK_CHECK_LAUNCH();
  for (int it = 0; it < kmeans_iters; it++) {
    km_update_kernel<<<n_segs, 512, upsmem, s>>>(sd, scr->P, scr->C, scr->A, scr->perm, scr->sims, d, 0);
    assign();
    km_assign_small_kernel<<<n_segs, 256, 0, s>>>(sd, scr->P, scr->C, scr->A, d);
    WK_CHECK_LAUNCH();
  }
  km_update_kernel<<<n_segs, 512, upsmem, s>>>(sd, scr->P, scr->C, scr->A, scr->perm, scr->sims, d, 1);
  // member lists staged in shared memory when (2k + 1 + L) ints fit the 200 KB opt-in
  const size_t fsmem = usmem + (size_t)max_L * sizeof(int);
  const int fin_sp = fsmem <= 200 * 1024 ? 1 : 0;
  if (store_bf16)
    km_finalize_kernel<__nv_bfloat16><<<n_segs, 256, fin_sp ? fsmem : usmem, s>>>(sd, scr->A, scr->perm, *ix, d,
                                                                                scr->status, fin_sp);
  else
    km_finalize_kernel<float><<<n_segs, 256, fin_sp ? fsmem : usmem, s>>>(sd, scr->A, scr->perm, *ix, d,
                                                                        scr->status, fin_sp);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_append_tokens(const wk_steady_view* st, const float* k_new, const float* v_new, int U, int d,
                     int store_bf16, int* status, void* stream) {
  if (!st || U <= 0 || d <= 0) return WK_ECONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  if (store_bf16) append_kernel<__nv_bfloat16><<<U, 128, 0, s>>>(*st, k_new, v_new, d, status);
  else append_kernel<float><<<U, 128, 0, s>>>(*st, k_new, v_new, d, status);
  WK_CHECK_LAUNCH();
  return 0;
}

// centroid scan (phase bit 1) and exact zone planning + unions (bit 2) of
// wk_score_topk / wk_centroid_scan / wk_plan_zones; `app` = the fused append
static int score_topk_impl(const wk_index_view* ix, const wk_step_view* sv, const wk_zone_params* zp, int U,
                           int m_max, int phases, const AppendArgs* app, cudaStream_t s) {
  if (!ix || !sv || !zp || U <= 0 || zp->G < 1 || zp->G > 8 || zp->d <= 0 || zp->d > 256 || (zp->d & 3))
    return WK_ECONFIG;
  if (configure_smem()) return WK_ECUDA;
  if (v6_ok(ix, sv, zp->d)) {
    if (m_max > 0 && (phases & 1)) {
      const int rc = zp->d == 128 ? launch_score_v5<8>(*ix, *sv, zp->G, U, m_max, s)
                                  : launch_score_v5<4>(*ix, *sv, zp->G, U, m_max, s);
      if (rc) return rc;
    }
    if (!(phases & 2)) return 0;
    SelParams p;
    p.G = zp->G; p.d = zp->d; p.blas_threads = zp->blas_threads;
    p.retrieval_fraction = zp->retrieval_fraction;
    p.estimation_fraction = zp->estimation_fraction;
    p.inv_sqrt_d = (float)(1.0 / sqrt((double)zp->d));
    p.need_tail = zp->tail_denominator_only;
    p.need_allc = zp->denominator_eq2;
    p.score_fp64 = 1;
    p.score_mode = 1;
    // retrieval piece rows: the attention chunk rows (attend_v5: 16; attend_v4:
    // 16 for G <= 4, 8 for G <= 8); zp->piece_rows = 0 -> the attend_v4 rule
    p.piece_rows = zp->piece_rows > 0 ? zp->piece_rows : (head_slots(zp->G) == 4 ? 16 : 8);
    p.k_new = nullptr; p.v_new = nullptr; p.store_bf16 = 0;
    if (app && app->on) { p.k_new = app->k; p.v_new = app->v; p.st = app->st; p.store_bf16 = app->bf16; }
    return launch_select_v6(*ix, *sv, p, U, m_max, s);
  }
  if (m_max > 0) {
    dim3 g1((m_max + 63) / 64, U);
    score_kernel<<<g1, 256, 0, s>>>(*ix, *sv, zp->d, zp->G);
    WK_CHECK_LAUNCH();
  }
  SelParams p;
  p.G = zp->G; p.d = zp->d; p.blas_threads = zp->blas_threads;
  p.retrieval_fraction = zp->retrieval_fraction;
  p.estimation_fraction = zp->estimation_fraction;
  p.inv_sqrt_d = (float)(1.0 / sqrt((double)zp->d));
  p.need_tail = zp->tail_denominator_only;
  p.need_allc = zp->denominator_eq2;
  p.score_fp64 = 0;
  p.score_mode = 0;
  p.piece_rows = 0;
  select_kernel<<<U * zp->G, 512, select_smem_bytes(), s>>>(*ix, *sv, p);
  WK_CHECK_LAUNCH();
  union_kernel<<<U, 1024, 0, s>>>(*ix, *sv);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_score_topk(const wk_index_view* ix, const wk_step_view* sv, const wk_zone_params* zp, int U,
                  int m_max, void* stream) {
  return score_topk_impl(ix, sv, zp, U, m_max, 3, nullptr, (cudaStream_t)stream);
}

int wk_tripartite_attn(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                       const wk_zone_params* zp, int U, int S, int store_bf16, void* stream) {
  if (!ix || !st || !sv || !zp || U <= 0 || S <= 0 || zp->G < 1 || zp->G > 8 || zp->d > 256 || (zp->d & 3))
    return WK_ECONFIG;
  if (configure_smem()) return WK_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  AttnParams p;
  p.G = zp->G; p.d = zp->d;
  p.inv_sqrt_d = (float)(1.0 / sqrt((double)zp->d));
  p.tail_denominator_only = zp->tail_denominator_only;
  p.denominator_eq2 = zp->denominator_eq2;
  dim3 grid(S, U);
  if (v6_ok(ix, sv, zp->d)) {
    // estimation rows (eu_x, eu_sz) were filled by select_v6's cluster union
    return store_bf16 ? dispatch_attend_v4<__nv_bfloat16, false>(*ix, *st, *sv, p, nullptr, U, S, s)
                      : dispatch_attend_v4<float, false>(*ix, *st, *sv, p, nullptr, U, S, s);
  }
  if (store_bf16)
    attend_kernel<__nv_bfloat16, false><<<grid, 128, attend_smem_bytes(zp->d, 2), s>>>(*ix, *st, *sv, p, nullptr);
  else
    attend_kernel<float, false><<<grid, 128, attend_smem_bytes(zp->d, 4), s>>>(*ix, *st, *sv, p, nullptr);
  WK_CHECK_LAUNCH();
  merge_kernel<<<U * zp->G, 128, 0, s>>>(*sv, p, S);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_full_attn(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                 const int32_t* n_store, int U, int G, int d, int S, int store_bf16, void* stream) {
  if (!ix || !st || !sv || !n_store || U <= 0 || S <= 0 || G < 1 || G > 8 || d > 256 || (d & 3))
    return WK_ECONFIG;
  if (configure_smem()) return WK_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  StepView v = *sv;
  v.tail = nullptr;
  AttnParams p;
  p.G = G; p.d = d;
  p.inv_sqrt_d = (float)(1.0 / sqrt((double)d));
  p.tail_denominator_only = 0;
  p.denominator_eq2 = 0;
  dim3 grid(S, U);
  if (v6_ok(ix, sv, d))
    return store_bf16 ? dispatch_attend_v4<__nv_bfloat16, true>(*ix, *st, v, p, n_store, U, S, s)
                      : dispatch_attend_v4<float, true>(*ix, *st, v, p, n_store, U, S, s);
  if (store_bf16)
    attend_kernel<__nv_bfloat16, true><<<grid, 128, attend_smem_bytes(d, 2), s>>>(*ix, *st, v, p, n_store);
  else
    attend_kernel<float, true><<<grid, 128, attend_smem_bytes(d, 4), s>>>(*ix, *st, v, p, n_store);
  WK_CHECK_LAUNCH();
  merge_kernel<<<U * G, 128, 0, s>>>(v, p, S);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_cache_step(const wk_cache_view* cv, const int32_t* rlist, const int32_t* nr,
                  const int32_t* n_steady, int r_cap, int G, int union_mode, int64_t step, int C,
                  int* status, void* stream) {
  if (!cv || !rlist || !nr || !n_steady || C <= 0 || G < 1 || G > 8) return WK_ECONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  cache_step_kernel<<<(C + 63) / 64, 64, 0, s>>>(*cv, rlist, nr, n_steady, r_cap, G, union_mode, step, C, status);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_cache_phase(const wk_cache_view* cv, int32_t* ids, const uint8_t* snap_in, int n, int64_t n_steady,
                   int64_t step, int phase, uint8_t* snap_out, int32_t* n_out, int* status, void* stream) {
  if (!cv || n < 0 || phase < 1 || phase > 7 || (n && !ids)) return WK_ECONFIG;
  if ((phase & 1) && (!snap_out || !n_out)) return WK_ECONFIG;
  if ((phase & 6) && n && !snap_in) return WK_ECONFIG;
  cache_phase_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*cv, ids, snap_in, n, n_steady, step, phase, snap_out,
                                                         n_out, status);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_cache_offload_step(const wk_cache2_view* cv, const wk_index_view* ix, const wk_steady_view* st,
                          const wk_step_view* sv, int G, int64_t step, int U, void* stream) {
  if (!cv || !ix || !st || !sv || U <= 0 || G < 1 || G > 8 || sv->pstride != 4 || !sv->pieces) return WK_ECONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  cache2_step_kernel<<<U, 512, 0, s>>>(*cv, *ix, *st, *sv, G, step);
  WK_CHECK_LAUNCH();
  return 0;
}

int wk_decode_step(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                   const wk_zone_params* zp, const float* k_new, const float* v_new, int U, int m_max, int S,
                   int store_bf16, void* stream) {
  if (!ix || !st || !sv || !zp || !k_new || !v_new || U <= 0) return WK_ECONFIG;
  if (!v6_ok(ix, sv, zp->d) || sv->pstride != 2 || m_max <= 0) {
    // generic path: separate append
    int rc = wk_append_tokens(st, k_new, v_new, U, zp->d, store_bf16, sv->status, stream);
    if (rc) return rc;
    rc = wk_score_topk(ix, sv, zp, U, m_max, stream);
    if (rc) return rc;
    return wk_tripartite_attn(ix, st, sv, zp, U, S, store_bf16, stream);
  }
  const AppendArgs app = {1, k_new, v_new, *st, store_bf16};
  const int rc = score_topk_impl(ix, sv, zp, U, m_max, 3, &app, (cudaStream_t)stream);
  if (rc) return rc;
  return wk_tripartite_attn(ix, st, sv, zp, U, S, store_bf16, stream);
}

int wk_centroid_scan(const wk_index_view* ix, const wk_step_view* sv, const wk_zone_params* zp, int U, int m_max,
                     void* stream) {
  if (!ix || !sv || !zp || !v6_ok(ix, sv, zp->d)) return WK_ECONFIG;
  const int rc = score_topk_impl(ix, sv, zp, U, m_max, 1, nullptr, (cudaStream_t)stream);
  return rc;
}

int wk_plan_zones(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                  const wk_zone_params* zp, const float* k_new, const float* v_new, int U, int m_max,
                  int store_bf16, void* stream) {
  if (!ix || !sv || !zp || !v6_ok(ix, sv, zp->d)) return WK_ECONFIG;
  AppendArgs app = {0, nullptr, nullptr, {}, 0};
  if (k_new && v_new && st) app = {1, k_new, v_new, *st, store_bf16};
  const int rc = score_topk_impl(ix, sv, zp, U, m_max, 2, &app, (cudaStream_t)stream);
  return rc;
}

int wk_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return WK_ECONFIG;
  return cudaHostAlloc(ptr, bytes, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess ? 0 : WK_ECUDA;
}

int wk_host_free(void* ptr) { return cudaFreeHost(ptr) == cudaSuccess ? 0 : WK_ECUDA; }

int wk_recall_at_k(const wk_index_view* ix, const wk_steady_view* st, const wk_step_view* sv,
                   const int32_t* n_store, int U, int G, int d, int metrics_k, int blas_threads,
                   float* s_scratch, uint8_t* rflag, int64_t n_cap, int store_bf16, float* recall_out,
                   void* stream) {
  if (!ix || !st || !sv || !n_store || U <= 0 || G < 1 || G > 8 || d > 256 || metrics_k < 1) return WK_ECONFIG;
  if (configure_smem()) return WK_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = recall_smem_bytes();
  if (store_bf16)
    recall_kernel<__nv_bfloat16><<<U * G, 512, sm, s>>>(*ix, *st, *sv, n_store, G, d, metrics_k, blas_threads,
                                                        s_scratch, rflag, n_cap, recall_out);
  else
    recall_kernel<float><<<U * G, 512, sm, s>>>(*ix, *st, *sv, n_store, G, d, metrics_k, blas_threads, s_scratch,
                                                rflag, n_cap, recall_out);
  WK_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
