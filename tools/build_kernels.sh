#!/bin/bash
# index-build kernel launch list (configs[2]-shaped build, U=128 units at 120K)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
U=${U:-128} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"km_" --csv --log-file gpurun_out/km.csv python tools/build_probe.py > gpurun_out/km.log 2>&1
python tools/launch_summary.py gpurun_out/km.csv | tee gpurun_out/km_summary.txt
U=${U:-128} python tools/build_probe.py
