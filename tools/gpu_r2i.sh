# round 2: factored local solves (exact LU), coarse factor kernel launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or gmres_matches or iteration_counts or factored" > gpurun_out/r2i_parity.log 2>&1
for lf in 0 1; do
  for c in C1 C3s; do
    GDSW_LOCAL_FACTOR=$lf GDSW_SETUP_TIMES=1 timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2i_ts_${c}_lf$lf.log 2>&1
  done
done
GDSW_LOCAL_FACTOR=1 timeout 900 python tools/run_configs.py C1 C3 > gpurun_out/r2i_cfg.jsonl 2> gpurun_out/r2i_cfg.err
GDSW_COARSE_FACTOR=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cf|k_coarse|k_restrict" -c 60 --csv --log-file gpurun_out/r2i_cf_launches.csv python tools/profile_coarse.py 8 8 8 2 > gpurun_out/r2i_cf_ncu.log 2>&1
for m in 0 1; do GDSW_COARSE_FACTOR=$m timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2i_cf_time.log 2>&1; done
