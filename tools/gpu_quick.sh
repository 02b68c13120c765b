#!/bin/bash
# one gpurun call: GPU tests (no -x: full picture), a short default bench and the decode launch list
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --layer-bufs 2 --cpu-steps 1 --no-extras ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'ms', d['ms_per_step'], 'attn', d['breakdown_ms_per_layer'], 'roof', d['roofline']['achieved'], d['roofline']['frac'], 'fa', d['full_attention'].get('hbm_gbs'), 'par', d.get('parity_sample'))" 2>&1 | tail -3
if [ "${QWEN:-1}" = "1" ]; then
timeout 600 python bench.py --model qwen2.5-7b --steps 5 --warmup 3 --layer-bufs 2 --no-cpu --no-extras --no-e2e > gpurun_out/bench_qwen.log 2>&1
tail -1 gpurun_out/bench_qwen.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qwen value', d['value'], 'ms', d['ms_per_step'], 'attn', d['breakdown_ms_per_layer'], 'roof', d['roofline']['achieved'], 'fa', d['full_attention'].get('speedup_wave_vs_full'))" 2>&1 | tail -3
fi
if [ "${PROFILE:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|select|attend|merge|append|prep" -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 1 --no-cpu --no-e2e --no-extras > gpurun_out/b_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
fi
