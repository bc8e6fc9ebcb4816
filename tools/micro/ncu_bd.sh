mkdir -p gpurun_out/micro
# nt order: 8 12 16 20 24 ...; per nt: 23 prod launches, 23 read launches
timeout 600 ncu --set full --clock-control none -k regex:'k_block_dot<|k_read' --launch-skip 100 --launch-count 2 -o gpurun_out/micro/bd_ncu -f tools/micro/bbd3 > gpurun_out/micro/bd_ncu.log 2>&1
tail -3 gpurun_out/micro/bd_ncu.log
