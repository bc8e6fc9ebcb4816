# HEAD check in a fresh container: smoke, GPU suite, bench
mkdir -p gpurun_out/head
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/head/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/head/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/head/bench.json 2> gpurun_out/head/bench.err
tail -3 gpurun_out/head/pytest.log; cat gpurun_out/head/smoke.log; cut -c1-400 gpurun_out/head/bench.json
