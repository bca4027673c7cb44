# One gpurun call that regenerates the committed evidence under profiles/ (round 1).
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
timeout 900 python bench.py --config c3 --seqs-per-gpu 32 --steps 10 --warmup 3 --no-e2e > gpurun_out/ev_bench_c3.json 2> gpurun_out/ev_bench_c3.err
timeout 600 python scripts/bench_rows.py > gpurun_out/ev_rows.jsonl 2> gpurun_out/ev_rows.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:distance_kernel -s 4 -c 1 -o gpurun_out/ev_dist_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_split -s 2 -c 1 -o gpurun_out/ev_attn python scripts/bench_rows.py --rows f1 > gpurun_out/ev_ncu_attn.log 2>&1
ls -la gpurun_out/
