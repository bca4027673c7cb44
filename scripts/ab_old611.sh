python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old611 && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py -q -x 2>&1 | tail -2
A="--config c2 --no-cpu-baseline --no-e2e --seed-sweep 0,2"
for i in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/ao_new_c2_$i.json 2>/dev/null
  MEMSHARE_BENCH_FUSED=1 timeout 300 python bench.py $A > gpurun_out/ao_newf_c2_$i.json 2>/dev/null
  (cd _old611 && timeout 300 python bench.py $A > ../gpurun_out/ao_old_c2_$i.json 2>/dev/null)
done
C="--config c3 --batch-seqs 16 --steps 5 --no-cpu-baseline --no-e2e --no-online"
timeout 600 python bench.py $C > gpurun_out/ao_new_c3.json 2>/dev/null
(cd _old611 && timeout 600 python bench.py $C > ../gpurun_out/ao_old_c3.json 2>/dev/null)
