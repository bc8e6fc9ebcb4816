# round 2: dataflow partitioned-inverse solves (local exact LU + coarse)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or gmres_matches or iteration_counts or factored or supernodal" > gpurun_out/r2j_parity.log 2>&1
for lv in 0 1; do
  for c in C1 C3s; do
    GDSW_CF_LEVELS=$lv GDSW_SETUP_TIMES=1 timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2j_ts_${c}_lv$lv.log 2>&1
  done
  for m in 0 1; do GDSW_CF_LEVELS=$lv GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2j_cf_time.log 2>&1; done
  GDSW_CF_LEVELS=$lv GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2j_cf_time.log 2>&1
done
GDSW_COARSE_FACTOR=0 timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2j_cf_time.log 2>&1
GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C1 C3 > gpurun_out/r2j_cfg.jsonl 2> gpurun_out/r2j_cfg.err
