python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m pytest tests/test_gpu_path.py -q -k cosine_metric_vs_oracle"
for i in 1 2 3; do
echo "== l1 loads"; MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftl1.so $T 2>&1 | tail -1
done
B="timeout 300 python bench.py --config c2 --no-cpu-baseline --seed-sweep 0,2 --no-e2e --no-online"
MEMSHARE_BENCH_FUSED=0 MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftgpu.so $B > gpurun_out/ab3_gpu.json 2>&1
MEMSHARE_BENCH_FUSED=0 MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftl1.so $B > gpurun_out/ab3_l1.json 2>&1
MEMSHARE_BENCH_FUSED=0 MEMSHARE_FUSED_TAIL=0 $B > gpurun_out/ab3_old.json 2>&1
