mkdir -p gpurun_out
timeout 600 python tools/profile_ts.py C2ilu 20 2>&1 | grep "local solve" > gpurun_out/r2ac_ts.log
cp tools/expt/libgdsw_expt.so paper_2304_04876_b200/_lib/libgdsw.so
timeout 600 python tools/profile_ts.py C2ilu 20 2>&1 | grep "local solve" | sed "s/^/NOSTART: /" >> gpurun_out/r2ac_ts.log
