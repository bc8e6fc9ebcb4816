# A/B: single-reduce update sweeping from the end (after the block dot's forward sweep)
mkdir -p gpurun_out/srrev
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('sr_update','block_dot','jacobi_upper')})"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_ops.py -m gpu -q -x > gpurun_out/srrev/pytest.log 2>&1; tail -1 gpurun_out/srrev/pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/srrev/rev$rep.json 2>/dev/null; summ gpurun_out/srrev/rev$rep.json
GDSW_SR_REV=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/srrev/fwd$rep.json 2>/dev/null; summ gpurun_out/srrev/fwd$rep.json
done
