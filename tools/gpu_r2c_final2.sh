# HEAD check: smoke + full GPU suite + bench; then A/B of 64-thread dataflow CTAs for local blocks
mkdir -p gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; cat gpurun_out/final2/smoke.log | tail -1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final2/pytest.log 2>&1; tail -1 gpurun_out/final2/pytest.log
timeout 900 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; cut -c1-200 gpurun_out/final2/bench.json
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
timeout 300 python tools/profile_ts.py C3s 20 2>&1 | tail -1
sed -i 's/^constexpr int CF_NT_LOCAL = 128, CF_NT_COARSE = 256;/constexpr int CF_NT_LOCAL = 64, CF_NT_COARSE = 256;/' paper_2304_04876_b200/csrc/coarse_factor.cuh
python -c "$B" > gpurun_out/final2/build64.log 2>&1; grep -A2 'k_cf_dataflowIddLi64' gpurun_out/final2/build64.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | head -2 | tr '\n' ' '
timeout 300 python tools/profile_ts.py C3s 20 2>&1 | tail -1
