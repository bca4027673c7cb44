# A/B of the fused a5-a7 tail (one gpurun call): parity subset, then c2 bench with the fused call,
# the separate calls with the in-kernel finaliser, and the separate calls with the finalize kernel.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_symm.py tests/test_gpu_analysis.py -q -x > gpurun_out/ab_pytest.txt 2>&1
echo pytest_rc=$?
MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftprof.so python scripts/probe_ft.py > gpurun_out/ab_ftprof.txt 2>&1
B="timeout 300 python bench.py --config c2 --no-cpu-baseline --seed-sweep 0,2 --no-e2e"
$B > gpurun_out/ab_fused.json 2> gpurun_out/ab_fused.err; echo fused_rc=$?
MEMSHARE_BENCH_FUSED=0 $B > gpurun_out/ab_sep.json 2> gpurun_out/ab_sep.err; echo sep_rc=$?
MEMSHARE_BENCH_FUSED=0 MEMSHARE_FUSED_TAIL=0 $B > gpurun_out/ab_old.json 2> gpurun_out/ab_old.err; echo old_rc=$?
$B > gpurun_out/ab_fused2.json 2> gpurun_out/ab_fused2.err; echo fused2_rc=$?
