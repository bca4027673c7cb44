# Same-box A/B of the grouped distance schedule (MEMSHARE_DIST_GROUPED) against the single-anchor
# kernel on the CROSS / f3 rows, with a pipeline-only (-DMS_DIST_NOEVAL) build; grouped parity tests first.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1; echo build_rc=$?
python paper_2507_21433_b200/build.py --variant noeval MS_DIST_NOEVAL > /dev/null 2>&1; echo v1=$?
timeout 240 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/g_pytest.log 2>&1; echo grp_rc=$?
rm -f gpurun_out/g5_rows.txt
for v in "" noeval; do
  if [ -z "$v" ]; then L=""; else L="paper_2507_21433_b200/libmemshare_$v.so"; fi
  echo "== $v grouped" >> gpurun_out/g5_rows.txt
  MEMSHARE_GROUPED=1 MEMSHARE_LIB=$L timeout 120 python scripts/bench_rows.py --rows cross,f3 >> gpurun_out/g5_rows.txt 2>> gpurun_out/g5.err
done
echo "== single" >> gpurun_out/g5_rows.txt
timeout 120 python scripts/bench_rows.py --rows cross,f3 >> gpurun_out/g5_rows.txt 2>> gpurun_out/g5.err
