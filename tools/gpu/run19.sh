mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16split.py -q -rf -x -k "fp32 or bit_identity or graph_vs or gain or signals or zero or splits" > gpurun_out/pytest_hf.log 2>&1
tail -3 gpurun_out/pytest_hf.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_vk.json 2> gpurun_out/bench_vk.err
python tools/prof_table.py gpurun_out/bench_vk.json > gpurun_out/prof_vk.txt 2>&1
head -42 gpurun_out/prof_vk.txt
export SC_LIB_PATH=exp/libstreamconv_b200.so
SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_x29.txt 2>&1
