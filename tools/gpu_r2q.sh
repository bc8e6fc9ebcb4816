# round 2: dataflow staging chains side by side + ticket prefetch
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "local_solves or golden or factored or supernodal or sharded" > gpurun_out/r2q_parity.log 2>&1
for c in C1 C3s; do timeout 900 python tools/profile_ts.py $c 20 2>&1 | grep "local solve" >> gpurun_out/r2q_ts.log; done
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 16 16 8 >> gpurun_out/r2q_ts.log 2>&1
GDSW_COARSE_FACTOR=1 timeout 600 python tools/profile_coarse.py 8 8 8 >> gpurun_out/r2q_ts.log 2>&1
