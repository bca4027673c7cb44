# The 3-layer-unit rule for long lists of 32 KiB slices against the session-start tree (_old/), same box.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1 > gpurun_out/lr_tests.txt
rm -f gpurun_out/lr_*.json
for i in 1 2; do
  timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-online > gpurun_out/lr_new_c3_$i.json 2>/dev/null
  (cd _old && timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-online > ../gpurun_out/lr_old_c3_$i.json 2>/dev/null)
  timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --seed-sweep 0,2 > gpurun_out/lr_new_c2_$i.json 2>/dev/null
  (cd _old && timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --seed-sweep 0,2 > ../gpurun_out/lr_old_c2_$i.json 2>/dev/null)
done
