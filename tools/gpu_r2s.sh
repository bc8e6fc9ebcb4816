# round 2: CTA-cooperative rows in the GPU IKJ LU for separator levels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "numeric_lu or local_solves or golden or factored" > gpurun_out/r2s_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 2>&1 | grep -E "numeric setup|local solve" >> gpurun_out/r2s_ts.log; done
GDSW_HOST_LU=0 GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C3 > gpurun_out/r2s_c3.jsonl 2> gpurun_out/r2s_c3.err
