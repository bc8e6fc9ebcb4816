mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --tb=short > gpurun_out/r2c_tests.log 2>&1
