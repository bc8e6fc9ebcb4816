# A/B of build-time knobs on one box: prolongation loads in flight, SpMV occupancy
mkdir -p gpurun_out/ab
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
summ() { python -c "
import json; d=json.load(open('$1')); p=d['phases']; print('$1', round(d['value']*1e3,3), d['iterations'], round(d['e2e']['value']*1e3,3), round(d['apply_ms'],4), {k:round(v['us_per_launch'],1) for k,v in p.items() if k in ('spmv','prolong','jacobi_upper','block_dot')})"; }
timeout 600 python bench.py > gpurun_out/ab/pl16.json 2>/dev/null; summ gpurun_out/ab/pl16.json
sed -i 's/constexpr int PROLONG_PL = 16;/constexpr int PROLONG_PL = 8;/' paper_2304_04876_b200/csrc/coarse.cuh
python -c "$B" > /dev/null 2>&1; timeout 600 python bench.py > gpurun_out/ab/pl8.json 2>/dev/null; summ gpurun_out/ab/pl8.json
sed -i 's/constexpr int PROLONG_PL = 8;/constexpr int PROLONG_PL = 16;/' paper_2304_04876_b200/csrc/coarse.cuh
sed -i 's/__global__ void __launch_bounds__(256) k_sell_spmv(/__global__ void __launch_bounds__(256, 6) k_sell_spmv(/' paper_2304_04876_b200/csrc/sparse.cuh
python -c "$B" > /dev/null 2>&1; timeout 600 python bench.py > gpurun_out/ab/spmv6.json 2>/dev/null; summ gpurun_out/ab/spmv6.json
sed -i 's/__global__ void __launch_bounds__(256, 6) k_sell_spmv(/__global__ void __launch_bounds__(256) k_sell_spmv(/' paper_2304_04876_b200/csrc/sparse.cuh
python -c "$B" > /dev/null 2>&1
timeout 900 python tools/run_configs.py C2ilu > gpurun_out/ab/c2ilu.jsonl 2> gpurun_out/ab/c2ilu.err; cat gpurun_out/ab/c2ilu.jsonl | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 \
  -o gpurun_out/ab/r2c_k_trisolve_stream -f python tools/profile_ts.py C2ilu 3 > gpurun_out/ab/ts_ncu.log 2>&1; tail -2 gpurun_out/ab/ts_ncu.log
