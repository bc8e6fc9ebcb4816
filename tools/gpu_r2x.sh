# round 2: column-major backward panels + adaptive column splits
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or factored or partitioned or supernodal or gmres_matches" > gpurun_out/r2x_parity.log 2>&1
for nocm in 0 1; do
  for c in C1 C3s; do GDSW_CF_NOCM=$nocm timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/nocm $nocm: /" >> gpurun_out/r2x_ts.log; done
  GDSW_CF_NOCM=$nocm GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/nocm $nocm: /" >> gpurun_out/r2x_ts.log
  GDSW_CF_NOCM=$nocm GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 2>&1 | sed "s/^/nocm $nocm: /" >> gpurun_out/r2x_ts.log
done
timeout 1200 python tools/run_configs.py C3 C1 > gpurun_out/r2x_cfg.jsonl 2> gpurun_out/r2x_cfg.err
