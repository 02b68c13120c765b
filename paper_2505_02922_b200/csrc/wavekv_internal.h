// wavekv_internal.h -- device-side aliases of the public ABI structs plus
// kernel declarations shared between translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/wavekv.h"

namespace wk {
using SegDesc = ::wk_segment;      // one clustering segment
using IndexView = ::wk_index_view; // per-layer index arrays
}  // namespace wk
