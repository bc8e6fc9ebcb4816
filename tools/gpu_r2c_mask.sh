# slot-mask SELL layout: GPU suite, bench A/B, configs
mkdir -p gpurun_out/mask
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/mask/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/mask/bench.json 2> gpurun_out/mask/bench.err
GDSW_NO_SELL_MASK=1 timeout 900 python bench.py > gpurun_out/mask/bench_nomask.json 2> gpurun_out/mask/bench_nomask.err
GDSW_SETUP_TIMES=1 timeout 1800 python tools/run_configs.py C1 C2 C2ilu C2single C3 C4 > gpurun_out/mask/configs.jsonl 2> gpurun_out/mask/configs.err
tail -2 gpurun_out/mask/pytest.log
for f in bench bench_nomask; do python -c "
import json; d=json.load(open('gpurun_out/mask/$f.json')); p=d['phases']; print('$f', d['value'], d['iterations'], d['e2e']['value'], d['apply_ms'], d['roofline']['frac'], {k:(round(v['us_per_launch'],1), round(v['gbs'])) for k,v in p.items()})"; done
