mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/ts_pytest.log
for c in C1 C3s C2ilu; do
  timeout 300 python tools/profile_ts.py $c
done > gpurun_out/prof_ts.log 2>&1
timeout 600 python tools/run_configs.py C1 C3 >> gpurun_out/prof_ts.log 2>&1
