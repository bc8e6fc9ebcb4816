mkdir -p gpurun_out
for v in "" "GDSW_TS_BUDGET_KB=56 GDSW_TS_MINCHUNKS=2" "GDSW_TS_BUDGET_KB=72 GDSW_TS_MINCHUNKS=2" "GDSW_TS_BUDGET_KB=72 GDSW_TS_MINCHUNKS=3"; do
  echo "== $v"; env $v timeout 600 python tools/profile_ts.py C3 5
  env $v timeout 600 python tools/profile_ts.py C1 5
done > gpurun_out/c3.log 2>&1
