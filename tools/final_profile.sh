#!/bin/bash
# Refresh profiles/: full-set ncu summaries of every decode kernel, the decode
# and build launch lists, and the bench lines of configs[1], [4], [2] (one gpurun call).
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --model qwen2.5-7b > gpurun_out/bench_qwen.log 2>&1
timeout 900 python bench.py --build > gpurun_out/bench_build.log 2>&1
TESTS=0 KERNELS="score_v5 select_v6 attend_v4 att4_merge" bash tools/prof2.sh > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|select|attend|merge|prep" -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 1 --no-cpu --no-e2e --no-flashinfer > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"km_" --csv --log-file gpurun_out/km.csv python tools/build_probe.py > /dev/null 2>&1
ls gpurun_out
