# A/B: alternating Jacobi sweep directions x factor-value L2 policy; parity incl. the offset-mask test
mkdir -p gpurun_out/alt
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), round(d['apply_ms'],4), {k:round(v['us_per_launch'],1) for k,v in p.items() if 'jacobi' in k or k in ('spmv','prolong')})"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/alt/pytest.log 2>&1; tail -1 gpurun_out/alt/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/alt/alt_norm.json 2>/dev/null; summ gpurun_out/alt/alt_norm.json
GDSW_SWEEP_ALT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/alt/fwd_norm.json 2>/dev/null; summ gpurun_out/alt/fwd_norm.json
sed -i 's/^constexpr bool SWEEP_VAL_EF = false;/constexpr bool SWEEP_VAL_EF = true;/' paper_2304_04876_b200/csrc/sparse.cuh
python -c "$B" > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/alt/alt_ef.json 2>/dev/null; summ gpurun_out/alt/alt_ef.json
GDSW_SWEEP_ALT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/alt/fwd_ef.json 2>/dev/null; summ gpurun_out/alt/fwd_ef.json
