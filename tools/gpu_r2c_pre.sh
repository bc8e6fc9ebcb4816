# A/B: SpTRSV starting-value prefetch one chunk ahead (TR_PREFETCH), parity of the level-set paths
mkdir -p gpurun_out/pre
B='import importlib.util as u; s=u.spec_from_file_location("b","paper_2304_04876_b200/build.py"); b=u.module_from_spec(s); s.loader.exec_module(b); b.build_all()'
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/pre/pytest.log 2>&1; tail -1 gpurun_out/pre/pytest.log
timeout 600 python tools/profile_ts.py C2ilu 20 > gpurun_out/pre/ts_on.txt 2>&1; tail -1 gpurun_out/pre/ts_on.txt
timeout 900 python tools/run_configs.py C2ilu > gpurun_out/pre/c2ilu_on.jsonl 2>/dev/null; cut -c1-330 gpurun_out/pre/c2ilu_on.jsonl
sed -i 's/^constexpr bool TR_PREFETCH = true;/constexpr bool TR_PREFETCH = false;/' paper_2304_04876_b200/csrc/tristream.cuh
python -c "$B" > /dev/null 2>&1
timeout 600 python tools/profile_ts.py C2ilu 20 > gpurun_out/pre/ts_off.txt 2>&1; tail -1 gpurun_out/pre/ts_off.txt
timeout 900 python tools/run_configs.py C2ilu > gpurun_out/pre/c2ilu_off.jsonl 2>/dev/null; cut -c1-330 gpurun_out/pre/c2ilu_off.jsonl
