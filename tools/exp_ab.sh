# A/B of default-bench step time: product library vs experiment builds (EXPS="FLAG1 FLAG2;FLAG3")
export PYTHONUNBUFFERED=1
A="${BENCH_A:---steps 10 --warmup 3 --layer-bufs 2 --no-cpu --no-extras --no-e2e}"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), 'ms', round(d['ms_per_step'],4), d['breakdown_ms_per_layer'])"; }
for r in 1 2; do
timeout 300 python bench.py $A 2>/dev/null | show product
IFS=';' read -ra V <<< "$EXPS"
for e in "${V[@]}"; do EXP_FLAGS="$e" timeout 300 python tools/exp_bench.py $A 2>/dev/null | show "$e"; done
done
