# A/B: one-wave grid-stride SpMV (GDSW_SPMV_WAVE=1) vs a row per thread
mkdir -p gpurun_out/spw
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('spmv','block_dot')})"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "spmv or gmres or golden" > gpurun_out/spw/pytest.log 2>&1; tail -1 gpurun_out/spw/pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/spw/rowpt$rep.json 2>/dev/null; summ gpurun_out/spw/rowpt$rep.json
GDSW_SPMV_WAVE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/spw/wave$rep.json 2>/dev/null; summ gpurun_out/spw/wave$rep.json
done
