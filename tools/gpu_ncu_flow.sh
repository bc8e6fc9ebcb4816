mkdir -p gpurun_out
GDSW_FLOW_MB=80 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi_flow -s 20 -c 1 -o gpurun_out/flow -f python tools/profile_c2.py --max-iters 30 > gpurun_out/ncu_flow.log 2>&1
