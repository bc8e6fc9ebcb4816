mkdir -p gpurun_out/ts
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/ts/pytest.log 2>&1
timeout 900 python tools/run_configs.py C2ilu C1 > gpurun_out/ts/configs.jsonl 2> gpurun_out/ts/configs.err
tail -1 gpurun_out/ts/pytest.log
python -c "
import json
for l in open('gpurun_out/ts/configs.jsonl'):
    d=json.loads(l); print({k:d.get(k) for k in ('config','iterations','solve_ms','ms_per_iteration','apply_ms')})"
