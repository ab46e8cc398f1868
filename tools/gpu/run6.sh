set -x
mkdir -p gpurun_out
python tools/ncu_one.py 5 2048 > gpurun_out/one.log 2>&1 || exit 1
for k in 28 1; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip $k --launch-count 1 -f -o gpurun_out/hf_op$((k+1)) python tools/ncu_one.py 5 2048 > gpurun_out/ncu_hf_$k.log 2>&1
done
SC_FP32_SPLIT=tf32 timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 28 --launch-count 1 -f -o gpurun_out/tf_op29 python tools/ncu_one.py 5 2048 > gpurun_out/ncu_tf_28.log 2>&1
ls -la gpurun_out
