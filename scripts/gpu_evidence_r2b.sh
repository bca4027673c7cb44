# Round-2 evidence, part 2: configs[4] (one rank's share of the 8-GPU c5 batch), the f-rows,
# the KV-head-sharded mode at N = 1 and the c2 seed sweep.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python bench.py --config c5 --batch-seqs 64 --steps 5 --no-cpu-baseline > gpurun_out/ev2_c5_64seq.json 2> gpurun_out/ev2_c5.err; echo c5_rc=$?
timeout 900 python scripts/bench_rows.py > gpurun_out/ev2_rows.jsonl 2> gpurun_out/ev2_rows.err; echo rows_rc=$?
timeout 600 python bench.py --config c2 --mode headshard --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ev2_c2_headshard.json 2> gpurun_out/ev2_hs.err; echo hs_rc=$?
