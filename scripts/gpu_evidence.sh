# One gpurun call that regenerates the committed evidence under profiles/ (round 1).
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
for wv in 0 1; do
  timeout 900 python bench.py --config c3 --seqs-per-gpu 32 --wave $wv --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_c3_wave$wv.json 2> /dev/null
done
timeout 900 python bench.py --config c4 --seqs-per-gpu 16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_c4.json 2> /dev/null
timeout 900 python bench.py --config c5 --seqs-per-gpu 32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_c5_wave0.json 2> /dev/null
timeout 600 python bench.py --mode headshard --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ev_c2_headshard.json 2> /dev/null
timeout 600 python scripts/bench_rows.py > gpurun_out/ev_rows.jsonl 2> gpurun_out/ev_rows.err
timeout 1200 python scripts/sweep_c4.py --seqs 16 > gpurun_out/ev_sweep_c4.jsonl 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:distance_st_kernel -s 4 -c 1 -o gpurun_out/ev_dist_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:distance_st_kernel -s 3 -c 1 -o gpurun_out/ev_dist_c4 python bench.py --config c4 --seqs-per-gpu 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage1_kernel -s 4 -c 1 -o gpurun_out/ev_s1_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu_s1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_split -s 2 -c 1 -o gpurun_out/ev_attn python scripts/bench_rows.py --rows f1 > gpurun_out/ev_ncu_attn.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.txt 2>&1
ls -la gpurun_out/
