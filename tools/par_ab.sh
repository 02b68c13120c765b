# A/B of the bench's parity sample: the in-tree library vs libwavekv_old.so
cd $GRAFT_REPO_ROOT
P="python bench.py --steps 5 --warmup 3 --layer-bufs 2 --cpu-steps 1 --no-extras --no-e2e"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d.get('parity_sample',{}).get('max_rel_l2'))"; }
$P 2>/dev/null | show new
cp paper_2505_02922_b200/libwavekv.so /tmp/libwavekv_new.so
cp paper_2505_02922_b200/libwavekv_old.so paper_2505_02922_b200/libwavekv.so
$P 2>/dev/null | show old
python bench.py --steps 5 --warmup 3 --cpu-steps 1 --no-extras --no-e2e 2>/dev/null | show old_default_bufs
