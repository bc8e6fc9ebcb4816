# round 2: interleaved two-dot GEMV in the dataflow kernel; all-GPU exact LU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r2t_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 2>&1 | grep -E "numeric setup|local solve" >> gpurun_out/r2t_ts.log; done
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2t_ts.log 2>&1
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2t_ts.log 2>&1
GDSW_LOCAL_FACTOR=1 GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C3 > gpurun_out/r2t_c3.jsonl 2> gpurun_out/r2t_c3.err
