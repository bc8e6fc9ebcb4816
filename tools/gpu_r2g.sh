# round 2: streamed SpTRSV consumer-warp count, block-dot variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sptrsv or local_solves or supernodal or block_dot or sr_update" > gpurun_out/r2g_parity.log 2>&1
for w in 8 16 32; do
  for c in C2ilu C1 C3s; do
    GDSW_TS_WARPS=$w timeout 600 python tools/profile_ts.py $c 20 2>&1 | tail -1 | sed "s/^/warps $w: /" >> gpurun_out/r2g_ts.log
  done
done
timeout 300 tools/micro/bbd2 > gpurun_out/r2g_bbd2.log 2>&1
