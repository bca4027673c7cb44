# Per-kernel device times of the distance call on the probe's pair lists (ncu launch list).
for v in base a1; do
  if [ $v = base ]; then L=""; else L="paper_2507_21433_b200/libmemshare_$v.so"; fi
  echo "== $v"
  MEMSHARE_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan|distance_kernel|finalize" --csv python scripts/probe_distance.py 2>/dev/null | grep -E "plan_kernel|distance_kernel|finalize_kernel" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | awk '{k=$1; v=$NF; n[k]++; if (n[k]%23==4) print k, v}' | cut -c1-90
done
