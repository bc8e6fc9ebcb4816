# round 2: partitioned-inverse GEMV with 8 loads in flight, one row per warp
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or gmres_matches or iteration_counts or factored or supernodal" > gpurun_out/r2k_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2k_ts_${c}.log 2>&1; done
for m in 0 1; do GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2k_cf_time.log 2>&1; done
for m in 0 1; do GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2k_cf_time.log 2>&1; done
GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C1 C3 C2ilu > gpurun_out/r2k_cfg.jsonl 2> gpurun_out/r2k_cfg.err
