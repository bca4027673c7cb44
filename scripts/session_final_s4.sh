# Round 2 session 4, final check: build, smoke, the GPU tests, the default bench line, c2, c4, the rows.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f4_build.log 2>&1; echo build_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/f4_bench_c3.json 2> gpurun_out/f4_bench_c3.err; echo c3_rc=$?
timeout 600 python bench.py --config c2 --steps 300 --warmup 20 > gpurun_out/f4_bench_c2.json 2> gpurun_out/f4_bench_c2.err; echo c2_rc=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/f4_bench_c4.json 2> gpurun_out/f4_bench_c4.err; echo c4_rc=$?
timeout 600 python scripts/bench_rows.py > gpurun_out/f4_rows.jsonl 2> gpurun_out/f4_rows.err; echo rows_rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/f4_bench_reference.json 2> gpurun_out/f4_ref.err; echo ref_rc=$?
