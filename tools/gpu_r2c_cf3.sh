# A/B: dataflow CTA size (128 threads, 10 per SM) and tiles per slot with the five-CTA kernel
mkdir -p gpurun_out/cf3
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf3/base.txt 2>&1; echo "base: $(tail -1 gpurun_out/cf3/base.txt)"
GDSW_CF_TPS=2 timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf3/tps2.txt 2>&1; echo "tps2: $(tail -1 gpurun_out/cf3/tps2.txt)"
sed -i 's/^constexpr int CF_THREADS = 256;/constexpr int CF_THREADS = 128;/' paper_2304_04876_b200/csrc/coarse_factor.cuh
sed -i 's/__launch_bounds__(CF_THREADS, 5) k_cf_dataflow/__launch_bounds__(CF_THREADS, 10) k_cf_dataflow/' paper_2304_04876_b200/csrc/coarse_factor.cuh
python -c "$B" > gpurun_out/cf3/build128.log 2>&1; grep -A2 'k_cf_dataflowIdd' gpurun_out/cf3/build128.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | head -2 | tr '\n' ' '
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf3/t128.txt 2>&1; echo "t128: $(tail -1 gpurun_out/cf3/t128.txt)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "factor or partitioned or supernodal or exact" 2>&1 | tail -1
