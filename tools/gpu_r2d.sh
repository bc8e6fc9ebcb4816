# round 2 (re-entry): full GPU suite incl. slow reference-pinned configs, smoke, bench, sharded checks
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2d_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rA --durations=40 -p no:randomly > gpurun_out/r2d_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_sharded1.json 2> gpurun_out/r2d_sharded1.err
GDSW_SAME_DEVICE=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_same2.json 2> gpurun_out/r2d_same2.err
