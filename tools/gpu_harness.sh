#!/bin/bash
# harness GPU tests + the C1/C2 harness reports
mkdir -p gpurun_out
python -m pytest tests/test_gpu_harness.py -x -q > gpurun_out/h_pytest.log 2>&1
python -m paper_2304_04876_b200.harness solve --config configs/c1.cfg --format json --output gpurun_out/h_c1.json > gpurun_out/h_c1.log 2>&1
python -m paper_2304_04876_b200.harness sweep --config configs/c2.cfg --axis local_solver --values 'fast_ilu(0,3,5),ilu_k(0)' --format json --output gpurun_out/h_c2.json > gpurun_out/h_c2.log 2>&1
python -m paper_2304_04876_b200.harness sweep --config configs/c2.cfg --axis local_solver --values 'fast_ilu(0,3,5),ilu_k(0)' --output gpurun_out/h_c2.csv >> gpurun_out/h_c2.log 2>&1
tail -3 gpurun_out/h_pytest.log; cat gpurun_out/h_c1.log gpurun_out/h_c2.log
