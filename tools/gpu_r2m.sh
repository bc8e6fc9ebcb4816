# round 2: multi-row warps in the dataflow partitioned-inverse solve
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or factored or supernodal" > gpurun_out/r2m_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2m_ts_${c}.log 2>&1; done
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2m_cf_time.log 2>&1
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2m_cf_time.log 2>&1
GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C3 C1 > gpurun_out/r2m_cfg.jsonl 2> gpurun_out/r2m_cfg.err
