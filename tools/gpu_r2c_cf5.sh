mkdir -p gpurun_out/cf5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_coarse_factor.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/cf5/pytest.log 2>&1; tail -1 gpurun_out/cf5/pytest.log
timeout 1500 python tools/run_configs.py C1 C1 C3 > gpurun_out/cf5/configs.jsonl 2> gpurun_out/cf5/configs.err
python -c "
import json
for l in open('gpurun_out/cf5/configs.jsonl'):
    d=json.loads(l); print(d['config'], d['iterations'], round(d['solve_ms'],2), round(d['ms_per_iteration'],3), round(d['apply_ms'],3))"
