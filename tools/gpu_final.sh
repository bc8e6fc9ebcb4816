# round-end style evidence: gpu tests, smoke, default bench, reference arm, configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 1500 python tools/run_configs.py C1 C2 C2ilu C2single C3 C4 C5_512 > gpurun_out/f_configs.jsonl 2>&1
