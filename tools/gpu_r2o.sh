# round 2: predicated row dots; tiles-per-slot sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local_solves or golden or factored or supernodal" > gpurun_out/r2o_parity.log 2>&1
for tps in 1 2 4 8; do
  for c in C1 C3s; do GDSW_CF_TPS=$tps timeout 900 python tools/profile_ts.py $c 20 2>&1 | grep "local solve" | sed "s/^/tps $tps: /" >> gpurun_out/r2o_ts.log; done
  GDSW_CF_TPS=$tps GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/tps $tps: /" >> gpurun_out/r2o_ts.log
  GDSW_CF_TPS=$tps GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 2>&1 | sed "s/^/tps $tps: /" >> gpurun_out/r2o_ts.log
done
