mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "fp32 or bit_identity or graph_vs" > gpurun_out/pytest_hf.log 2>&1
tail -5 gpurun_out/pytest_hf.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_hf_cfg5.json 2> gpurun_out/bench_hf_cfg5.err
python tools/prof_table.py gpurun_out/bench_hf_cfg5.json > gpurun_out/prof_hf.txt 2>&1
head -45 gpurun_out/prof_hf.txt
export SC_LIB_PATH=exp/libstreamconv_b200.so
SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_hf29.txt 2>&1
SC_TC_TRACE_OP=2 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_hf2.txt 2>&1
