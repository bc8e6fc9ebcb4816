mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/ts_pytest.log
for c in C1 C3s C2ilu; do
  timeout 300 python tools/profile_ts.py $c
  GDSW_TS_BUDGET_KB=100 timeout 300 python tools/profile_ts.py $c
  GDSW_TS_BUDGET_KB=60 timeout 300 python tools/profile_ts.py $c
done > gpurun_out/prof_ts.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
