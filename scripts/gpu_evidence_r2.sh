# One gpurun call that regenerates the round-2 evidence (profiles/r2_*): GPU tests, smoke, the
# driver's bench lines (c3 default, c2, reference arm, c4), the c2 launch list, an ncu capture of
# the distance kernel at c2 and the device timeline of the c2 rounds.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev_build.log 2>&1
python paper_2507_21433_b200/build.py --variant tl MS_TIMELINE > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1100 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.txt 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.txt 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/ev_bench_c3.json 2> gpurun_out/ev_bench_c3.err; echo c3_rc=$?
timeout 600 python bench.py --config c2 > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err; echo c2_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo ref_rc=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/ev_bench_c4.json 2> gpurun_out/ev_bench_c4.err; echo c4_rc=$?
MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_tl.so timeout 300 python scripts/probe_timeline.py > gpurun_out/ev_timeline.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --config c2 --steps 10 --warmup 5 --no-cpu-baseline --no-e2e --no-online --no-parity --seed-sweep '' > /dev/null 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:distance_st_kernel -s 4 -c 1 -o gpurun_out/ev_dist_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-online --no-parity --seed-sweep '' > gpurun_out/ev_ncu.log 2>&1; echo ncu2_rc=$?
ls -la gpurun_out/
