#!/bin/bash
# attend_v5 timing split: estimation vs exact chunks (ATT5_SKIP rebuilds; results are not valid outputs)
export PYTHONUNBUFFERED=1
for f in "" "-DATT5_SKIP=1" "-DATT5_SKIP=2" ${EXTRA_CFGS}; do
  WK_EXTRA_NVCC_FLAGS="$f" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"attend_v5" -c 6 --csv --log-file /tmp/l.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
  echo "flags=[$f]"; grep attend_v5 /tmp/l.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
done
