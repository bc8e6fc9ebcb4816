# round 2: factored coarse solve: parity, configs at n_c = 2,744 / 12,600 both ways, initcheck after the fix
mkdir -p gpurun_out/san
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "factored or coarse or golden" > gpurun_out/r2f_parity.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "p8" > gpurun_out/r2f_configs.log 2>&1
for m in 0 1; do
  GDSW_COARSE_FACTOR=$m timeout 1200 python tools/run_configs.py C5_512 C5_2048 > gpurun_out/r2f_cfg_mode$m.jsonl 2> gpurun_out/r2f_cfg_mode$m.err
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 50 --error-exitcode 9 python tools/sanitize.py > gpurun_out/san/initcheck.log 2>&1
echo "initcheck exit $?" > gpurun_out/san/summary_r2f.txt
