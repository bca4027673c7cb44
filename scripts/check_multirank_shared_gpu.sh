# The N > 1 bench path (torchrun, barriers, max-over-ranks timing, LPT partition, pair sums) with
# 2 ranks sharing cuda:0 over gloo (MEMSHARE_BENCH_SHARED_GPU=1, testing only; a 1-GPU box).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export MEMSHARE_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --batch-seqs 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mr_c3.json 2> gpurun_out/mr_c3.err; echo c3_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --config c2 --steps 20 --warmup 3 --no-cpu-baseline --seed-sweep "" > gpurun_out/mr_c2.json 2> gpurun_out/mr_c2.err; echo c2_rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref_rc=$?
