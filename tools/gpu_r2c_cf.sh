# A/B: column-major panel loads in flight per thread in k_cf_dataflow (CF_CMU)
mkdir -p gpurun_out/cf
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf/cmu4.txt 2>&1; tail -1 gpurun_out/cf/cmu4.txt
timeout 600 python tools/profile_ts.py C1 50 > gpurun_out/cf/c1_cmu4.txt 2>&1; tail -1 gpurun_out/cf/c1_cmu4.txt
sed -i 's/^#define CF_CMU 4$/#define CF_CMU 8/' paper_2304_04876_b200/csrc/coarse_factor.cuh
python -c "$B" > /dev/null 2>&1
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf/cmu8.txt 2>&1; tail -1 gpurun_out/cf/cmu8.txt
timeout 600 python tools/profile_ts.py C1 50 > gpurun_out/cf/c1_cmu8.txt 2>&1; tail -1 gpurun_out/cf/c1_cmu8.txt
sed -i 's/^#define CF_CMU 8$/#define CF_CMU 2/' paper_2304_04876_b200/csrc/coarse_factor.cuh
python -c "$B" > /dev/null 2>&1
timeout 600 python tools/profile_ts.py C3s 20 > gpurun_out/cf/cmu2.txt 2>&1; tail -1 gpurun_out/cf/cmu2.txt
