# round 2: slab (per-rank window) setup of the sharded solve
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_harness.py -q -x > gpurun_out/r2ad_dist.log 2>&1
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2ad_sharded1.json 2> gpurun_out/r2ad_sharded1.err
GDSW_SAME_DEVICE=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ad_same2.json 2> gpurun_out/r2ad_same2.err
