#!/bin/bash
# rebuild attend_v6 with -D overrides and run the 65K x 128-unit reproduction
IFS=";" read -ra CL <<< "${CFGS}"
for f in "${CL[@]}"; do
  WK_EXTRA_NVCC_FLAGS="$f" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  echo "== [$f]"; CUDA_LAUNCH_BLOCKING=1 python tools/repro_attn.py 2>&1 | tail -2
done
