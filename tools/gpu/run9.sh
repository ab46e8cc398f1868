mkdir -p gpurun_out
for k in 28 21; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip $k --launch-count 1 -f -o gpurun_out/x2_op$((k+1)) python tools/ncu_one.py 5 4096 > gpurun_out/ncu_x2_$k.log 2>&1
done
ls gpurun_out
