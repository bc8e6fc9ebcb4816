mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "local_solves or golden or factored or partitioned or supernodal or gmres_matches or sharded" > gpurun_out/r2aa_parity.log 2>&1
for tps in 1 2 4; do
  for c in C1 C3s; do GDSW_CF_TPS=$tps timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/tps $tps: /" >> gpurun_out/r2aa_ts.log; done
  GDSW_CF_TPS=$tps GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/tps $tps: /" >> gpurun_out/r2aa_ts.log
done
