mkdir -p gpurun_out
for c in C1 C3s C2ilu; do
  for b in 64 100 160 220; do echo "budget $b"; GDSW_TS_BUDGET_KB=$b timeout 300 python tools/profile_ts.py $c; done
  for b in 100 220; do echo "budget $b xglobal"; GDSW_TS_XGLOBAL=1 GDSW_TS_BUDGET_KB=$b timeout 300 python tools/profile_ts.py $c; done
done > gpurun_out/prof_ts2.log 2>&1
