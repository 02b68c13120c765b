#!/bin/bash
# source-level instruction counts + stalls of the decode kernels (one launch each)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for k in ${KERNELS:-select_v6 attend_v4}; do
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"$k" -s ${SKIP:-20} -c 1 -o /tmp/${k}_full python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e --no-extras --no-flashinfer ${BENCH_ARGS} > gpurun_out/ncu_${k}.log 2>&1
  python tools/ncu_lines.py /tmp/${k}_full.ncu-rep 60 "Instructions Executed" > gpurun_out/${k}_inst.txt
  python tools/ncu_lines.py /tmp/${k}_full.ncu-rep 40 > gpurun_out/${k}_lines.txt
  ncu -i /tmp/${k}_full.ncu-rep --page details --csv > gpurun_out/${k}_details.csv 2>/dev/null
  ncu -i /tmp/${k}_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${k}_source.csv 2>/dev/null
done
ls -la gpurun_out
