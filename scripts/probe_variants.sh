# Tuning probe: the distance-kernel rows (c2 aligned, CROSS, f3) with compile-time variants.
# usage: bash scripts/probe_variants.sh "name:DEF1,DEF2 name2:DEF3" [rows]
ROWS=${2:-f2,cross,f3}
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
echo "== base"; timeout 300 python scripts/bench_rows.py --rows $ROWS 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(r['row'][:34].ljust(34), 'us=%.1f'%r.get('us',0), 'pairs/s=%.3gM'%(r.get('pairs_per_s',0)/1e6), 'frac=%s'%r.get('frac_of_peak'))"
for v in $1; do
  name=${v%%:*}; defs=${v#*:}
  so=$(python paper_2507_21433_b200/build.py --variant $name $(echo $defs | tr ',' ' ') 2>/dev/null | tail -1)
  echo "== $name ($defs)"
  MEMSHARE_LIB=$so timeout 300 python scripts/bench_rows.py --rows $ROWS 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(r['row'][:34].ljust(34), 'us=%.1f'%r.get('us',0), 'pairs/s=%.3gM'%(r.get('pairs_per_s',0)/1e6), 'frac=%s'%r.get('frac_of_peak'))"
done
