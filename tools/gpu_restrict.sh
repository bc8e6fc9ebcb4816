#!/bin/bash
# restriction kernel change: parity + C2 / C4 phase tables
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -x -q > gpurun_out/rs_pytest.log 2>&1
tail -2 gpurun_out/rs_pytest.log
python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/rs_c2.json 2> gpurun_out/rs_c2.err
python bench.py --grid 200 --boxes 5 --precision single --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/rs_c4.json 2> gpurun_out/rs_c4.err
