#!/bin/bash
# attend_v4 chunk-rows / ring / warps sweep for HS=4: rebuild with -D overrides
# (ATT4_RG4 chunk rows, ATT4_NST8 ring stages when RG=8, ATT4_W warps), bench each.
export PYTHONUNBUFFERED=1
CFGS=${CFGS:-"16,3,12 8,3,16 8,2,16 8,3,12"}
for cfg in $CFGS; do
  IFS=, read rg nst w <<< "$cfg"
  WK_EXTRA_NVCC_FLAGS="-DATT4_RG4=$rg -DATT4_NST8=$nst -DATT4_W=$w" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  r=$(WK_RG4=$rg python bench.py --layer-bufs 2 --no-cpu --fa-steps 0 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['breakdown_ms_per_layer']['tripartite_attn']*1e3,1))")
  echo "RG=$rg NST8=$nst W=$w -> $r"
done
