B="timeout 300 python bench.py --config c2 --no-cpu-baseline --seed-sweep 0,2 --no-e2e --no-online --no-parity"
for v in "" ftnofence ftnofin ftboth; do
  if [ -n "$v" ]; then export MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_$v.so; else unset MEMSHARE_LIB; fi
  MEMSHARE_BENCH_FUSED=0 $B > gpurun_out/ab2_sep_$v.json 2>&1
  MEMSHARE_BENCH_FUSED=0 MEMSHARE_FUSED_TAIL=0 $B > gpurun_out/ab2_old_$v.json 2>&1
done
