mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "split or out_argument" 2>&1 | tail -3
for sp in 1 2 4 8 1; do
  python bench.py --no-extras --no-cpu --no-e2e --no-flashinfer --fa-steps 0 --steps 10 --split $sp 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('split', $sp, round(l['value'],1), round(l['ms_per_step'],3))"
done
