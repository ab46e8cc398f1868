export SC_SKIP_BUILD=1
NCU_ONE_LIST=1 python tools/ncu_one.py 5 > gpurun_out/names.txt 2>&1
# op29 is the 29th TC launch (op1..op36 are TC, op0 pqmf): skip 28
ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 28 --launch-count 1 -o gpurun_out/op29 -f python tools/ncu_one.py 5 > gpurun_out/ncu52.log 2>&1
ncu -i gpurun_out/op29.ncu-rep --page source --csv --print-source sass > gpurun_out/op29_sass.csv 2>/dev/null
ncu -i gpurun_out/op29.ncu-rep --page raw --csv > gpurun_out/op29_raw.csv 2>/dev/null
ls -la gpurun_out/
