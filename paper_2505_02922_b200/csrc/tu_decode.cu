// tu_decode.cu -- translation unit: generic decode kernels + recall@k metric
// (metrics.cu shares decode.cu's selection helpers).
#include "decode.cu"
#include "metrics.cu"
