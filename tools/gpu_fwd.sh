#!/bin/bash
# previous-chunk forwarding in the streamed SpTRSV: parity + timing with/without
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -x -q > gpurun_out/fwd_pytest.log 2>&1
tail -3 gpurun_out/fwd_pytest.log
for c in C2ilu C1 C3s C3; do
  timeout 300 python tools/profile_ts.py $c 20 2>&1 | grep "local solve"
  GDSW_TS_NOFWD=1 timeout 300 python tools/profile_ts.py $c 20 2>&1 | grep "local solve" | sed 's/^/NOFWD /'
done
