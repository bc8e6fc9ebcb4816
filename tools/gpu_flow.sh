mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/fl_pytest.log
for rpt in 1 2; do for mb in 40 80 120; do
GDSW_FLOW_RPT=$rpt GDSW_FLOW_MB=$mb timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/fl_bench_${rpt}_$mb.json 2> gpurun_out/fl_bench_${rpt}_$mb.err
done; done
