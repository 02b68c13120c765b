#!/bin/bash
# attend_v5 ring stages x warps sweep: rebuild with -D overrides, bench each (configs[1], 2 layer buffers)
export PYTHONUNBUFFERED=1
CFGS=${CFGS:-"2,12 3,8 4,6 3,12"}
for cfg in $CFGS; do
  IFS=, read nst w <<< "$cfg"
  WK_EXTRA_NVCC_FLAGS="-DATT5_NST=$nst -DATT5_WMAX=$w" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  r=$(python bench.py --layer-bufs 2 --no-cpu --fa-steps 0 --no-e2e --no-extras ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['breakdown_ms_per_layer']['tripartite_attn']*1e3,1))")
  echo "NST=$nst WMAX=$w -> $r"
done
