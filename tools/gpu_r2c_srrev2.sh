# A/B: block-dot basis rows with the default L2 policy (instead of evict-first), update sweeping back
mkdir -p gpurun_out/srrev
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('sr_update','block_dot','jacobi_upper')})"; }
sed -i 's/      for (int u = 0; u < KRG; ++u) x\[u\] = ldg_stream(rp\[u\] + i);/      for (int u = 0; u < KRG; ++u) x[u] = __ldg(rp[u] + i);/' paper_2304_04876_b200/csrc/krylov.cuh
grep -c '__ldg(rp\[u\] + i)' paper_2304_04876_b200/csrc/krylov.cuh
python -c "$B" > /dev/null 2>&1
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/srrev/ldg_rev$rep.json 2>/dev/null; summ gpurun_out/srrev/ldg_rev$rep.json
GDSW_SR_REV=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/srrev/ldg_fwd$rep.json 2>/dev/null; summ gpurun_out/srrev/ldg_fwd$rep.json
done
