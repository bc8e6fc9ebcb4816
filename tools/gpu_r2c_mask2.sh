mkdir -p gpurun_out/mask2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/mask2/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/mask2/bench.json 2> gpurun_out/mask2/bench.err
GDSW_NO_SELL_MASK=1 timeout 900 python bench.py > gpurun_out/mask2/bench_nomask.json 2> gpurun_out/mask2/bench_nomask.err
tail -1 gpurun_out/mask2/pytest.log
for f in bench bench_nomask; do python -c "
import json; d=json.load(open('gpurun_out/mask2/$f.json')); p=d['phases']; print('$f', d['value'], d['iterations'], d['e2e']['value'], d['apply_ms'], d['roofline']['frac'], {k:(round(v['us_per_launch'],1), round(v['gbs'])) for k,v in p.items()})"; done
