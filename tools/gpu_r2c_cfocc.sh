# A/B: k_cf_dataflow occupancy (register cap via min CTAs per SM)
mkdir -p gpurun_out/cfocc
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cfocc/b4.txt 2>&1; echo "minB 4: $(tail -1 gpurun_out/cfocc/b4.txt)"
for mb in 5 6 8; do
sed -i "s/__launch_bounds__(CF_THREADS[^)]*) k_cf_dataflow/__launch_bounds__(CF_THREADS, $mb) k_cf_dataflow/" paper_2304_04876_b200/csrc/coarse_factor.cuh
python -c "$B" > gpurun_out/cfocc/build$mb.log 2>&1; grep -A2 'k_cf_dataflowIdd' gpurun_out/cfocc/build$mb.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | head -2 | tr '\n' ' '
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cfocc/b$mb.txt 2>&1; echo "minB $mb: $(tail -1 gpurun_out/cfocc/b$mb.txt)"
done
