mkdir -p gpurun_out
for fl in 0 1 2 3 0 3; do
  for c in C1 C3s; do GDSW_CF_FLAGS=$fl timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/flags $fl: /" >> gpurun_out/r2r_ts.log; done
  GDSW_CF_FLAGS=$fl GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/flags $fl: /" >> gpurun_out/r2r_ts.log
done
