# sharded path at the round-2c code: world-1 sharded bench, 2 ranks on one device, dist tests
mkdir -p gpurun_out/dist
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dist/sharded1.json 2> gpurun_out/dist/sharded1.err
GDSW_SAME_DEVICE=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dist/same2.json 2> gpurun_out/dist/same2.err
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q > gpurun_out/dist/pytest.log 2>&1
tail -1 gpurun_out/dist/pytest.log
for f in sharded1 same2; do python -c "
import json; d=json.load(open('gpurun_out/dist/$f.json')); print('$f', d['n_gpus'], d['value'], d['iterations'], d.get('ms_per_iteration'), d.get('comm_ms_per_solve'), (d.get('e2e') or {}).get('value'))"; done
