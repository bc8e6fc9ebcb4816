# round 2: compute-sanitizer over every kernel family (tiny cases), ncu source profiles of the streamed SpTRSV
mkdir -p gpurun_out/san
CS=compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/san/summary.txt
done
timeout 900 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 9 python -m pytest tests/test_gpu_dist.py -x -q -k fast_ilu > gpurun_out/san/memcheck_dist.log 2>&1
echo "memcheck dist exit $?" >> gpurun_out/san/summary.txt
timeout 600 python tools/profile_ts.py C2ilu 20 > gpurun_out/ts_c2ilu_time.log 2>&1
timeout 600 python tools/profile_ts.py C1 20 > gpurun_out/ts_c1_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 -o gpurun_out/r2_ts_c2ilu -f python tools/profile_ts.py C2ilu 3 > gpurun_out/ncu_ts_c2ilu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 -o gpurun_out/r2_ts_c1 -f python tools/profile_ts.py C1 3 > gpurun_out/ncu_ts_c1.log 2>&1
