mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 28 --launch-count 1 -f -o gpurun_out/aw_op29 python tools/ncu_one.py 5 4096 > gpurun_out/ncu_aw.log 2>&1
