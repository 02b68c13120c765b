# e2e leg vs host-I/O group size (layers per H2D / D2H group)
for gr in 2 4 8 16 32; do
  timeout 300 python bench.py --steps 10 --warmup 3 --layer-bufs 2 --no-cpu --no-extras --e2e-group $gr 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('GR', $gr, 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
