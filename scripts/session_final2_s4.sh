# Round 2 session 4, final state check after the 3-layer-unit rule: build, smoke, GPU tests, default line, c2.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g2_build.log 2>&1; echo build_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g2_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/g2_bench_c3.json 2> gpurun_out/g2_bench_c3.err; echo c3_rc=$?
timeout 600 python bench.py --config c2 --steps 300 --warmup 20 > gpurun_out/g2_bench_c2.json 2> gpurun_out/g2_bench_c2.err; echo c2_rc=$?
