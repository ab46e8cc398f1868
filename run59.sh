export SC_SKIP_BUILD=1
SC_LIB_PATH=exp/libstreamconv_b200.so SC_TC_TRACE_OP=2 timeout 300 python tools/trace_tc.py 5 fp32 2 | head -52
