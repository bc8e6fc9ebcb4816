# round 2 evidence: full GPU suite, smoke, bench (+ reference arm), configs, ncu launch list + captures
mkdir -p gpurun_out/final
R=${R:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/smi.txt 2>&1
lscpu > gpurun_out/final/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/final/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
GDSW_SETUP_TIMES=1 timeout 2400 python tools/run_configs.py C1 C2 C2ilu C2single C3 C4 C5_1 C5_8 C5_64 C5_216 C5_256 C5_512 C5_2048 > gpurun_out/final/configs.jsonl 2> gpurun_out/final/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/final/${R}_launches.csv python tools/profile_c2.py --solves 1 > gpurun_out/final/launch.log 2>&1
for k in k_jacobi_upper k_block_dot k_sr_update k_prolong k_sell_spmv; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$k -s 5 -c 1 -o gpurun_out/final/${R}_$k -f python tools/profile_c2.py --solves 1 --max-iters 10 > gpurun_out/final/${R}_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cf_dataflow -s 2 -c 1 \
  -o gpurun_out/final/${R}_k_cf_dataflow -f python tools/profile_ts.py C3s 3 > gpurun_out/final/${R}_cf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 \
  -o gpurun_out/final/${R}_k_trisolve_stream -f python tools/profile_ts.py C2ilu 3 > gpurun_out/final/${R}_ts.log 2>&1
caps=$(ls gpurun_out/final/${R}_k_*.ncu-rep)
python tools/ncu_summary.py ${R} gpurun_out/final/${R}_launches.csv $caps > gpurun_out/final/summary.log 2>&1
cp profiles/${R}_ncu_summary.* gpurun_out/final/
for f in $caps; do
  case $f in *k_jacobi_upper*|*k_cf_dataflow*|*k_block_dot*) ;; *) rm -f $f ;; esac
done
