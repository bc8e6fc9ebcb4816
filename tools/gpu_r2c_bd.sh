# block-dot change: micro, GPU suite, bench
mkdir -p gpurun_out/bd
timeout 120 tools/micro/bbd3 > gpurun_out/bd/micro.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/bd/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/bd/bench.json 2> gpurun_out/bd/bench.err
tail -2 gpurun_out/bd/pytest.log; python -c "
import json; d=json.load(open('gpurun_out/bd/bench.json')); print(d['value'], d['iterations'], d['e2e']['value'], d['phases']['block_dot'])"
