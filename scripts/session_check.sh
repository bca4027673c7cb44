python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s1_build.log 2>&1; echo build_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.log 2>&1; echo pytest_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err; echo bench_rc=$?
timeout 600 python bench.py --config c2 --steps 200 --warmup 20 > gpurun_out/s1_bench_c2.json 2> gpurun_out/s1_bench_c2.err; echo c2_rc=$?
