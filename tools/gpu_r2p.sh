# round 2: producer-staged starting values (PSV) in the streamed SpTRSV
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sptrsv or local_solves or golden or gmres_matches" > gpurun_out/r2p_parity.log 2>&1
for psv in 1 0; do
  GDSW_TS_PSV=$psv timeout 600 python tools/profile_ts.py C2ilu 20 2>&1 | grep "local solve" | sed "s/^/psv $psv: /" >> gpurun_out/r2p_ts.log
  GDSW_TS_PSV=$psv timeout 600 python tools/profile_ts.py ela_ilu1 20 2>&1 | grep "local solve" | sed "s/^/psv $psv: /" >> gpurun_out/r2p_ts.log
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "C2_ilu0 or ilu0_p4" > gpurun_out/r2p_cfg.log 2>&1
timeout 900 python tools/run_configs.py C2ilu > gpurun_out/r2p_c2ilu.jsonl 2>&1
