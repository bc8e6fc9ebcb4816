# ncu evidence for profiles/: launch list of one C2 solve + full captures
mkdir -p gpurun_out
R=${R:-r1e}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${R}_launches.csv python tools/profile_c2.py --solves 1 > gpurun_out/${R}_launch.log 2>&1
for k in k_jacobi_upper k_sr_update k_block_dot k_sell_spmv k_prolong k_restrict_chunks k_gather_jacobi_lower; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$k -s 5 -c 1 -o gpurun_out/${R}_$k -f python tools/profile_c2.py --solves 1 --max-iters 10 > gpurun_out/${R}_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trisolve_stream -s 2 -c 1 \
  -o gpurun_out/${R}_k_trisolve_stream -f python tools/profile_ts.py C3s 3 > gpurun_out/${R}_ts.log 2>&1
caps=$(ls gpurun_out/${R}_k_*.ncu-rep)
python tools/ncu_summary.py ${R} gpurun_out/${R}_launches.csv $caps > gpurun_out/${R}_summary.log 2>&1
cp profiles/${R}_ncu_summary.* gpurun_out/
# keep only the captures of the two top kernels (64 MiB copy-back cap)
for f in $caps; do
  case $f in *k_jacobi_upper*|*k_trisolve_stream*) ;; *) rm -f $f ;; esac
done
