# Tuning probe: online-round phase latencies with segmentation tile variants (NT x ITEMS).
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
echo "== shipped"; timeout 120 python scripts/probe_online.py | head -2
for v in "1024 4" "512 16" "256 32"; do set -- $v
  so=$(python paper_2507_21433_b200/build.py --variant seg$1_$2 MS_SEG_NT=$1 MS_SEG_ITEMS=$2 2>/dev/null | tail -1)
  echo "== NT=$1 ITEMS=$2"; MEMSHARE_LIB=$so timeout 120 python scripts/probe_online.py | head -2
done
timeout 600 python -m pytest tests/test_gpu_path.py -q -x -k "segment" 2>&1 | tail -2
