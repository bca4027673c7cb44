for v in base st7 st12x16 piece32 piece4 diag w8 st13x16w8; do
  if [ $v = base ]; then L=""; else L="paper_2507_21433_b200/libmemshare_$v.so"; fi
  echo -n "$v: "; MEMSHARE_LIB=$L timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep "breakdown block_distance"
done
for lpi in 1 4 8; do echo -n "lpi$lpi: "; MEMSHARE_LAYERS_PER_ITEM=$lpi timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep "breakdown block_distance"; done
