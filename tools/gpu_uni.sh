mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/p.log
timeout 600 python bench.py > gpurun_out/u0.json 2>gpurun_out/u0.err
GDSW_NO_GRAPH=1 timeout 600 python bench.py > gpurun_out/u1.json 2>/dev/null
