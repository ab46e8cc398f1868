# Experiment library: kernels_tc.cu with the per-slab trace hooks compiled in
# (-DSC_TC_EXPERIMENTS=1), linked with the product objects into exp/libstreamconv_b200.so.
# Use: SC_LIB_PATH=exp/libstreamconv_b200.so SC_TC_TRACE_OP=<op> python tools/trace_tc.py ...
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
B=paper_2204_07064_b200/build
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -I include -ccbin /usr/bin/g++ \
  -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DSC_TC_EXPERIMENTS=1 \
  -c paper_2204_07064_b200/csrc/kernels_tc.cu -o exp/kernels_tc_exp.o
objs=$(ls $B/*.o | grep -v kernels_tc.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libstreamconv_b200.so exp/kernels_tc_exp.o $objs -lcuda -lcufft
echo exp/libstreamconv_b200.so
