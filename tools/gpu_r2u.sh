# round 2: partitioned-inverse blocks computed on the device
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_dist.py -q -x > gpurun_out/r2u_parity.log 2>&1
for c in C1 C3s; do GDSW_SETUP_TIMES=1 timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2u_ts_$c.log 2>&1; done
for c in C1 C3s; do GDSW_PINV_HOST=1 GDSW_SETUP_TIMES=1 timeout 900 python tools/profile_ts.py $c 20 > gpurun_out/r2u_ts_${c}_host.log 2>&1; done
