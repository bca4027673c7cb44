# Same-box A/B for the stage-1 changes: GPU parity subset, then the c2 bench (incl. the online rounds)
# for the working tree and the old tree in _old/ (prepared as in scripts/ab_rev.sh).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_progress.py -q -x 2>&1 | tail -2
A="--config c2 --no-cpu-baseline --no-e2e --seed-sweep 0"
for i in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/ar_new_c2_$i.json 2>/dev/null
  (cd _old && timeout 300 python bench.py $A > ../gpurun_out/ar_old_c2_$i.json 2>/dev/null)
done
