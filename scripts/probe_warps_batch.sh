python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
so=$(python paper_2507_21433_b200/build.py --variant w16 MS_CONSUMER_WARPS=16 2>/dev/null | tail -1)
for lib in "" $so; do
  echo "== lib=$lib"
  MEMSHARE_LIB=$lib timeout 600 python bench.py --config c3 --seqs-per-gpu 32 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; r=json.loads(sys.stdin.read()); print('c3 dist %.4f frac %.3f'%(r['roofline']['kernel_ms'], r['roofline']['frac']))"
  MEMSHARE_LIB=$lib timeout 600 python bench.py --config c5 --seqs-per-gpu 32 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; r=json.loads(sys.stdin.read()); print('c5 dist %.4f frac %.3f'%(r['roofline']['kernel_ms'], r['roofline']['frac']))"
done
