#!/bin/bash
# tensor-pipe evidence for the tcgen05 k-means assignment (configs[2] build):
# ncu --set full of one km_assign_tc5 launch + the tensor-pipe metrics this
# ncu exposes for sm_100 (queried on the box), summarised to text.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
ncu --query-metrics --chip gb100 2>/dev/null | grep -i -E "tensor|pipe_tc|tmem|utc|tcgen" > gpurun_out/tc_metric_names.txt
M=$(grep -o -E "^sm__[a-z_]*(tensor|tc|utc)[a-z_]*" gpurun_out/tc_metric_names.txt | sort -u | head -30 | sed 's/$/.avg.pct_of_peak_sustained_active/' | paste -sd, -)
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:km_assign_tc5 -s 3 -c 1 \
  -o /tmp/tc5 python bench.py --build --no-extras > gpurun_out/ncu_tc5.log 2>&1
ncu -i /tmp/tc5.ncu-rep --page details --csv > gpurun_out/km_assign_tc5_details.csv 2>/dev/null
ncu -i /tmp/tc5.ncu-rep --page raw --csv > gpurun_out/km_assign_tc5_raw.csv 2>/dev/null
python tools/ncu_lines.py /tmp/tc5.ncu-rep 30 > gpurun_out/km_assign_tc5_lines.txt 2>&1
timeout 600 ncu -f --clock-control none -k regex:km_assign_tc5 -s 3 -c 1 --metrics "$M" --csv \
  python bench.py --build --no-extras > gpurun_out/km_assign_tc5_tensor_metrics.csv 2>&1
cuobjdump -sass paper_2505_02922_b200/build/kmeans.o 2>/dev/null | grep -o -E "UTC[A-Z]*MMA[A-Z0-9.]*|LDTM[A-Z0-9.]*|UBLKCP[A-Z0-9.]*" | sort | uniq -c > gpurun_out/km_sass_tc_ops.txt
ls -la gpurun_out
