# round 2: extend-add coarse factor + unrolled GEMVs, NW=16 SpTRSV, EP=2 block dot
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2h_parity.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "p8 or C2_fast" > gpurun_out/r2h_configs.log 2>&1
for m in 0 1; do
  GDSW_SETUP_TIMES=1 GDSW_COARSE_FACTOR=$m timeout 1200 python tools/run_configs.py C5_512 C5_2048 > gpurun_out/r2h_cfg_mode$m.jsonl 2> gpurun_out/r2h_cfg_mode$m.err
done
GDSW_TS_WARPS=24 timeout 600 python tools/profile_ts.py C2ilu 20 2>&1 | tail -1 > gpurun_out/r2h_ts24.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
