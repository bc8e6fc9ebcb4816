set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/t1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err
timeout 1200 python tools/run_configs.py C1 C2ilu C2single C4 C5_512 C3 > gpurun_out/t1_configs.jsonl 2>&1
tail -5 gpurun_out/t1_*.log gpurun_out/t1_bench.json gpurun_out/t1_configs.jsonl
