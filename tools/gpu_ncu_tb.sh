mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_jacobi_tb_lower -s 5 -c 1 -o gpurun_out/tb -f python tools/profile_c2.py --solves 1 --max-iters 10 > gpurun_out/ncu_tb.log 2>&1
