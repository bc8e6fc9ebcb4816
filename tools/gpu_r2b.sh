# round 2: drift diagnosis, sharded path with graphs + side stream, bench --gpus self-launch
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "drift or thread or identity" -x -q --tb=long > gpurun_out/r2b_drift.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_harness.py -x -q --tb=long > gpurun_out/r2b_dist.log 2>&1
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_sharded1.json 2> gpurun_out/r2b_sharded1.err
GDSW_NO_GRAPH=1 timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_sharded1_nograph.json 2> gpurun_out/r2b_sharded1_nograph.err
GDSW_SAME_DEVICE=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_same2.json 2> gpurun_out/r2b_same2.err
