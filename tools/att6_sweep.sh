#!/bin/bash
# attend_v6 producer / consumer warp-count sweep (ncu kernel durations, configs[1] workload)
export PYTHONUNBUFFERED=1
IFS=";" read -ra CL <<< "${CFGS:--DATT6_NP=2 -DATT6_NC=10;-DATT6_NP=4 -DATT6_NC=8;-DATT6_NP=3 -DATT6_NC=9;-DATT6_NP=4 -DATT6_NC=10}"
for f in "${CL[@]}"; do
  WK_EXTRA_NVCC_FLAGS="$f" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"attend_v" -c 6 --csv --log-file /tmp/l.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e --no-extras ${BENCH_ARGS} > /dev/null 2>&1
  echo "flags=[$f] $(grep gpu__time /tmp/l.csv | tail -3 | awk -F'","' '{printf "%s ", $NF}')"
done
