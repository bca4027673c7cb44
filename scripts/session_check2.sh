python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2_build.log 2>&1; echo build_rc=$?
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mixed_probe scripts/mixed_probe.cu && timeout 300 /tmp/mixed_probe > gpurun_out/s2_mixed.txt 2>&1; echo probe_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2_pytest.log 2>&1; echo pytest_rc=$?
