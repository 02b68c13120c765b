#!/bin/bash
# one gpurun call: GPU parity tests, a short bench, the decode-kernel launch list
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --layer-bufs 2 --cpu-steps 2 > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/bench.log
if [ "${PROFILE:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|select|attend|merge|append|prep" -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 1 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
fi
