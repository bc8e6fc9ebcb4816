# verify the five-CTA dataflow kernel: exact-LU parity and the configs that use it
mkdir -p gpurun_out/cfocc
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_coarse_factor.py -m gpu -q -x > gpurun_out/cfocc/pytest.log 2>&1; tail -1 gpurun_out/cfocc/pytest.log
timeout 1500 python tools/run_configs.py C1 C3 C5_2048 > gpurun_out/cfocc/configs.jsonl 2> gpurun_out/cfocc/configs.err
python -c "
import json
for l in open('gpurun_out/cfocc/configs.jsonl'):
    d=json.loads(l); print(d['config'], d['iterations'], round(d['solve_ms'],2), round(d['ms_per_iteration'],3), round(d['apply_ms'],3))"
