# one gpurun call: per-call breakdown at c2, the c3 (32 seq/GPU) line, and the c2 ncu launch list
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --breakdown --no-cpu-baseline > gpurun_out/bench_c2_bd.json 2> gpurun_out/bench_c2_bd.err
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep breakdown gpurun_out/bench_c2_bd.err; cat gpurun_out/bench_c3.json | head -c 1500
