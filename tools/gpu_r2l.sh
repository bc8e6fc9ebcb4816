# round 2: adaptive dataflow tiles
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or factored or supernodal" > gpurun_out/r2l_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2l_ts_${c}.log 2>&1; done
for c in C1 C3s; do GDSW_LOCAL_FACTOR=0 timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2l_ts_${c}_stream.log 2>&1; done
for m in 1; do GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2l_cf_time.log 2>&1; done
for m in 1; do GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2l_cf_time.log 2>&1; done
GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C3 > gpurun_out/r2l_cfg.jsonl 2> gpurun_out/r2l_cfg.err
