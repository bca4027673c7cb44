python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1; echo build_rc=$?
MEMSHARE_GROUPED=1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:distance_grp -c 1 -f -o gpurun_out/g_grp_f3b python scripts/bench_rows.py --rows f3 > gpurun_out/g_ncu.log 2>&1; echo ncu_rc=$?
