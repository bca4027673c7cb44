# Time the front kernels under MEMSHARE_DEBUG_SKIP masks (tuning only; results are not valid outputs).
# The work-skipping masks act only in a tuning build: python -m paper_2507_21433_b200.build --variant tuning MEMSHARE_TUNING
# and MEMSHARE_LIB=paper_2507_21433_b200/libmemshare_tuning.so.
for m in 0 1 2 4 7; do
  MEMSHARE_DEBUG_SKIP=$m timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stage1|encode|fill_kernel|seg_" -s 12 -c 6 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "stage1|encode|fill_kernel|seg_" | awk -F'","' -v m=$m '{print "skip" m, $5, $NF}' | sed 's/"//g' | cut -c1-120
done
