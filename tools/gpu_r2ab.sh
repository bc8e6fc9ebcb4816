mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 -o gpurun_out/r2ab_ts_c2ilu -f python tools/profile_ts.py C2ilu 3 > gpurun_out/r2ab_ts.log 2>&1
GDSW_SETUP_TIMES=1 timeout 1200 python tools/run_configs.py C3 C1 > gpurun_out/r2ab_cfg.jsonl 2> gpurun_out/r2ab_cfg.err
