// cache_internal.h -- device alias of the block-cache view.
#pragma once
#include "wavekv_internal.h"

namespace wk {
using CacheView = ::wk_cache_view;
}  // namespace wk
