// tu_abi.cu -- translation unit: centroid scan, block caches and the C ABI
// (abi.cu launches every kernel; kernels of the other units are declared there).
#include "score_v5.cu"
#include "cache.cu"
#include "cache_v2.cu"
#include "abi.cu"
