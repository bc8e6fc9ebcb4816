mkdir -p gpurun_out/cfocc
for k in 1 2; do timeout 600 python tools/run_configs.py C1 C1 > gpurun_out/cfocc/c1_$k.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/cfocc/c1_$k.jsonl'):
    d=json.loads(l); print(d['config'], d['iterations'], round(d['solve_ms'],2), round(d['ms_per_iteration'],3), round(d['apply_ms'],3))"; done
timeout 300 python tools/profile_ts.py C1 50 2>&1 | tail -1
