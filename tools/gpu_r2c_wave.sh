# A/B: one-wave grid for the single-reduce update
mkdir -p gpurun_out/wave
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('sr_update','block_dot')})"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gmres or golden" > gpurun_out/wave/pytest.log 2>&1; tail -1 gpurun_out/wave/pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/wave/wave$rep.json 2>/dev/null; summ gpurun_out/wave/wave$rep.json
GDSW_SR_WAVE=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/wave/nowave$rep.json 2>/dev/null; summ gpurun_out/wave/nowave$rep.json
done
