# Round 2 session 4 evidence: the default bench (c3 batch), c2 with the 5-seed sweep, the GPU tests.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e4_build.log 2>&1; echo build_rc=$?
timeout 900 python bench.py > gpurun_out/e4_bench_c3.json 2> gpurun_out/e4_bench_c3.err; echo c3_rc=$?
timeout 600 python bench.py --config c2 --steps 300 --warmup 20 --seed-sweep 0,1,2,3,4 > gpurun_out/e4_bench_c2.json 2> gpurun_out/e4_bench_c2.err; echo c2_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/e4_pytest.log 2>&1; echo pytest_rc=$?
