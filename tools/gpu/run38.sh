export SC_LIB_PATH=exp/libstreamconv_b200.so SC_SKIP_BUILD=1
SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_a.txt 2>&1
SC_TC_DEBUG=64 SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_b.txt 2>&1
SC_TC_DEBUG=2 SC_TC_TRACE_OP=29 python tools/trace_tc.py 5 fp32 > gpurun_out/trace_c.txt 2>&1
