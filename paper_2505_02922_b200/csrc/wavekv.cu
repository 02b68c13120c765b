// wavekv.cu -- unity translation unit: one nvcc invocation builds libwavekv.so
// (sm_100a) from the kernel sources and the C ABI.
#include "kmeans.cu"
#include "decode.cu"
#include "select_v6.cu"
#include "attend_v4.cu"
#include "score_v4.cu"
#include "cache.cu"
#include "cache_v2.cu"
#include "metrics.cu"
#include "abi.cu"
