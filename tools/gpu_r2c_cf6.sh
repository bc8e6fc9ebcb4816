mkdir -p gpurun_out/cf6
timeout 300 python tools/profile_ts.py C3s 20 2>&1 | tail -1
timeout 300 python tools/profile_ts.py C1 50 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_coarse_factor.py -m gpu -q -x 2>&1 | tail -1
