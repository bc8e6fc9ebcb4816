# round 2: ncu of the dataflow partitioned-inverse solve (C3-sized blocks, C1)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cf_dataflow -s 2 -c 1 -o gpurun_out/r2n_cf_c3s -f python tools/profile_ts.py C3s 3 > gpurun_out/r2n_cf_c3s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cf_dataflow -s 2 -c 1 -o gpurun_out/r2n_cf_c1 -f python tools/profile_ts.py C1 3 > gpurun_out/r2n_cf_c1.log 2>&1
