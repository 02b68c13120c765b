set -x
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|select|attend|merge|append" -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 1 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select" -s 40 -c 1 -o gpurun_out/select_full python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e > gpurun_out/b_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend" -s 40 -c 1 -o gpurun_out/attend_full python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e > gpurun_out/b_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score" -s 40 -c 1 -o gpurun_out/score_full python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e > gpurun_out/b_ncu4.log 2>&1
ls -la gpurun_out
