#!/bin/bash
# round-2 evidence: ncu --set full summaries of the decode kernels and the build's
# top kernels, the decode and build launch lists, tensor-pipe counters of the
# k-means assignment and the attention (one gpurun call)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TESTS=0 KERNELS="attend_v6 select_v6 score_v5 att6_merge" bash tools/prof2.sh > /dev/null 2>&1
for k in attend_v6 select_v6 score_v5 att6_merge; do python tools/ncu_summary.py gpurun_out/${k}_details.csv > gpurun_out/${k}_summary.txt 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score|select|attend|merge" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layer-bufs 1 --fa-steps 0 --no-cpu --no-e2e --no-extras > gpurun_out/b_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt
bash tools/build_kernels.sh > gpurun_out/build_kernels.txt 2>&1
U=16 timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"km_assign_tc5|km_seed_v3" -c 2 -o /tmp/km python tools/build_probe.py > /dev/null 2>&1
ncu -i /tmp/km.ncu-rep --page details --csv > gpurun_out/km_details.csv 2>/dev/null
ncu -i /tmp/km.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
    d=dict(zip(h,r)); print('==', d.get('Kernel Name','')[:60])
    for k in h:
        if any(x in k for x in ('pipe_tensor','tmem','utc','pipe_fma_cycles','inst_executed_pipe_uniform')) and ('pct' in k or k.endswith('.sum')):
            print('  ', k, d[k])
" > gpurun_out/km_tensor_metrics.txt
ls -la gpurun_out
