# quick GPU check: parity tests + default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/q_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
