# Same-box A/B of an online-round change (working tree) against the previous commit (_old/): the
# c2 line with its online rounds, after the parity tests that cover LAST / RANGE rounds.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_progress.py -q -x 2>&1 | tail -1 > gpurun_out/fb2_tests.txt
rm -f gpurun_out/fb2_*.json
for i in 1 2; do
  timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --seed-sweep "" > gpurun_out/fb2_new_$i.json 2>/dev/null
  (cd _old && timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --seed-sweep "" > ../gpurun_out/fb2_old_$i.json 2>/dev/null)
done
