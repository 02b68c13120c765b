#!/bin/bash
# ncu --set full of the k-means++ seeding kernel on a 16-unit 120K build
mkdir -p gpurun_out
U=${U:-16} timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"km_seed" -c 1 -o /tmp/seed python tools/build_probe.py > gpurun_out/ncu_seed.log 2>&1
ncu -i /tmp/seed.ncu-rep --page details --csv > gpurun_out/seed_details.csv 2>/dev/null
cp /tmp/seed.ncu-rep gpurun_out/
