mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/u0.json 2>/dev/null
GDSW_SR_KEEP_ZM=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/u1.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/p.log
