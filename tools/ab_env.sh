#!/bin/bash
# A/B an environment knob on the default bench workload: ab_env.sh VAR "v1 v2 ..." [extra bench args]
var=$1; vals=$2; shift 2
for v in $vals; do
  r=$(env $var=$v python bench.py --layer-bufs 2 --no-cpu --fa-steps 0 --no-e2e "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3))")
  echo "$var=$v -> $r"
done
