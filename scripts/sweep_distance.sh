# Tuning sweep of the block-distance kernel (variants built with build.py --variant NAME DEFINES...).
for v in base a2; do
  if [ $v = base ]; then L=""; else L="paper_2507_21433_b200/libmemshare_$v.so"; fi
  echo "== $v"; MEMSHARE_LIB=$L timeout 120 python scripts/probe_distance.py 2>&1 | grep -E "c2|disjoint |chain|subset"
done
