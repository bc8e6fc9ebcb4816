# A/B: k_sr_update register cap (min CTAs per SM) with the one-wave grid
mkdir -p gpurun_out/srocc
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('sr_update',)})"; }
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/srocc/b0.json 2>/dev/null; summ gpurun_out/srocc/b0.json
for mb in 6 8; do
sed -i "s/__global__ void __launch_bounds__(256[^)]*) k_sr_update(/__global__ void __launch_bounds__(256, $mb) k_sr_update(/" paper_2304_04876_b200/csrc/krylov.cuh
python -c "$B" > gpurun_out/srocc/build$mb.log 2>&1; grep -A2 'k_sr_updateILi2ELb0' gpurun_out/srocc/build$mb.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | head -2 | tr '\n' ' '
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/srocc/b$mb.json 2>/dev/null; summ gpurun_out/srocc/b$mb.json
done
