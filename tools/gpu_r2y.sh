mkdir -p gpurun_out
for cm in 128 512 2048; do
  for c in C1 C3s; do GDSW_CF_CM_MAX=$cm timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/cm $cm: /" >> gpurun_out/r2y_ts.log; done
  GDSW_CF_CM_MAX=$cm GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/cm $cm: /" >> gpurun_out/r2y_ts.log
  GDSW_CF_CM_MAX=$cm GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 2>&1 | sed "s/^/cm $cm: /" >> gpurun_out/r2y_ts.log
done
