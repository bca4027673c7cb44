# Same-box A/B of scripts/bench_rows.py rows (default: f2) for the working tree and the old tree in _old/.
ROWS=${1:-f2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py -q -x -k "cosine" 2>&1 | tail -1
for i in 1 2; do
  timeout 600 python scripts/bench_rows.py --rows $ROWS > gpurun_out/arow_new_$i.jsonl 2>/dev/null
  (cd _old && timeout 600 python scripts/bench_rows.py --rows $ROWS > ../gpurun_out/arow_old_$i.jsonl 2>/dev/null)
done
grep -h '"row"' gpurun_out/arow_*.jsonl | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(d['row'][:40], d.get('us'), d.get('frac_of_peak'))"
