# round 2: full GPU suite (incl. reference-pinned config tests) + quick bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=25 -p no:randomly 2>&1 | tail -120 > gpurun_out/r2a_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
