mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 -o gpurun_out/ts_c2ilu -f python tools/profile_ts.py C2ilu 3 > gpurun_out/ncu_ts2.log 2>&1
