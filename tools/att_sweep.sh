#!/bin/bash
# attend_v4 ring-depth / warps sweep: rebuild with -D overrides (needs ATT4_NST / ATT4_W hooks), bench each
export PYTHONUNBUFFERED=1

for cfg in ${CFGS:-"2,12 3,8 4,6"}; do
  nst=${cfg%,*}; w=${cfg#*,}
  WK_EXTRA_NVCC_FLAGS="-DATT4_NST=$nst -DATT4_W=$w" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  for pk in 0; do
    r=$(python bench.py --layer-bufs 2 --no-cpu --fa-steps 0 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['breakdown_ms_per_layer']['tripartite_attn']*1e3,1))")
    echo "NST=$nst W=$w -> $r"
  done
done
