bash scripts/ab_rev.sh _old --config c2 --no-cpu-baseline --no-e2e --seed-sweep 0 --steps 200 --warmup 20 > gpurun_out/ab_s1.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_path.py tests/test_gpu_progress.py -q -x > gpurun_out/ab_s1_tests.log 2>&1; echo tests=$?
