# Tuning probe: single-target stage size cap (MEMSHARE_ST_MAXKRE, 4 KiB units) on c4 (40 KiB slices) and c2.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for k in 10 5; do
  echo "== MAXKRE=$k"
  MEMSHARE_ST_MAXKRE=$k timeout 600 python bench.py --config c4 --seqs-per-gpu 16 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; r=json.loads(sys.stdin.read()); print('c4 dist %.4f frac %.3f'%(r['roofline']['kernel_ms'], r['roofline']['frac']))"
done
timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; r=json.loads(sys.stdin.read()); print('c2 dist %.4f frac %.3f step %.4f'%(r['roofline']['kernel_ms'], r['roofline']['frac'], r['ms_per_step']))"
