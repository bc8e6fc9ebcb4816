# sync-free ILU(k) SpTRSV: parity, local-solve time and C2 ILU(0) solve vs the streamed level-set kernel
mkdir -p gpurun_out/sf
timeout 300 python tools/profile_ts.py C2ilu 20 > gpurun_out/sf/ts_sf.txt 2>&1; tail -1 gpurun_out/sf/ts_sf.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py -m gpu -q -x > gpurun_out/sf/pytest.log 2>&1; tail -1 gpurun_out/sf/pytest.log
timeout 600 python tools/run_configs.py C2ilu > gpurun_out/sf/c2ilu_sf.jsonl 2>/dev/null; cut -c1-330 gpurun_out/sf/c2ilu_sf.jsonl
GDSW_SYNCFREE=0 timeout 300 python tools/profile_ts.py C2ilu 20 > gpurun_out/sf/ts_ls.txt 2>&1; tail -1 gpurun_out/sf/ts_ls.txt
timeout 300 python tools/profile_ts.py ela_ilu1 20 > gpurun_out/sf/ela_sf.txt 2>&1; tail -1 gpurun_out/sf/ela_sf.txt
GDSW_SYNCFREE=0 timeout 300 python tools/profile_ts.py ela_ilu1 20 > gpurun_out/sf/ela_ls.txt 2>&1; tail -1 gpurun_out/sf/ela_ls.txt
