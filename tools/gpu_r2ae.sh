mkdir -p gpurun_out
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/cmu4: /" >> gpurun_out/r2ae_ts.log; done
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/cmu4: /" >> gpurun_out/r2ae_ts.log
cp tools/expt/libgdsw_cmu8.so paper_2304_04876_b200/_lib/libgdsw.so
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 30 2>&1 | grep "local solve" | sed "s/^/cmu8: /" >> gpurun_out/r2ae_ts.log; done
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 2>&1 | sed "s/^/cmu8: /" >> gpurun_out/r2ae_ts.log
