python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pdl in 0 1; do for i in 1 2; do
MEMSHARE_PDL=$pdl timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; r=json.loads(sys.stdin.read()); print('pdl=$pdl', 'ms/step %.4f'%r['ms_per_step'], 'value %.0f'%r['value'], 'dist %.4f'%r['roofline']['kernel_ms'], 'frac %.3f'%r['roofline']['frac'], 'online', '%.1f'%r['online']['round_us'])"
done; done
