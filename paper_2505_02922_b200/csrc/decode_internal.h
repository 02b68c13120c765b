// decode_internal.h -- per-step device views for the decode kernels.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "wavekv_internal.h"

namespace wk {
using SteadyView = ::wk_steady_view;  // sinks + decode buffer (engine.py:87-96)
using StepView = ::wk_step_view;      // per-step buffers

struct SelParams {
  int G, d, blas_threads;
  double retrieval_fraction, estimation_fraction;
  float inv_sqrt_d;
  int need_tail, need_allc;
  int score_fp64;  // scores came from the fp64-accumulating kernel (score_v3)
  int score_mode;  // wk_zone_params.score_mode of the scores being selected
  int piece_rows;  // rows per retrieval piece (attend_v4 chunk rows)
  // fused append of this step's token (engine.py:178-182), done by the
  // head-0 CTA of each unit; k_new == nullptr: no append
  const float* k_new;
  const float* v_new;
  SteadyView st;
  int store_bf16;
};

struct AttnParams {
  int G, d;
  float inv_sqrt_d;
  int tail_denominator_only, denominator_eq2;
};

size_t attend_smem_bytes(int d, int elem);
}  // namespace wk
