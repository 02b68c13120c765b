#!/bin/bash
# ncu --set full of the decode kernels; reports summarised on the box (text only comes back)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
[ "${TESTS:-1}" = "1" ] && { timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log; }
for k in ${KERNELS:-score_v5 select_v6 attend_v4 att4_merge}; do
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"$k" -s ${SKIP:-20} -c 1 -o /tmp/${k}_full python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_${k}.log 2>&1
  python tools/ncu_lines.py /tmp/${k}_full.ncu-rep 40 > gpurun_out/${k}_lines.txt
  ncu -i /tmp/${k}_full.ncu-rep --page details --csv > gpurun_out/${k}_details.csv 2>/dev/null
  ncu -i /tmp/${k}_full.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = "1" ] && cp /tmp/${k}_full.ncu-rep gpurun_out/
done
ls -la gpurun_out
