mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/ts_pytest.log
timeout 1200 python tools/run_configs.py C1 C2ilu C3 > gpurun_out/ts_configs.jsonl 2>&1
