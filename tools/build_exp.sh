# Experiment library: kernels_tc.cu rebuilt with extra -D flags (default: the per-slab trace
# hooks, -DSC_TC_EXPERIMENTS=1), linked with the product objects into <dir>/libstreamconv_b200.so.
# Use: bash tools/build_exp.sh [dir] [flags...];
#      SC_LIB_PATH=exp/libstreamconv_b200.so SC_TC_TRACE_OP=<op> python tools/trace_tc.py ...
set -e
cd "$(dirname "$0")/.."
D=${1:-exp}
shift || true
FLAGS=${@:--DSC_TC_EXPERIMENTS=1}
mkdir -p $D
B=paper_2204_07064_b200/build
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -I include -ccbin /usr/bin/g++ \
  -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr $FLAGS \
  -c paper_2204_07064_b200/csrc/kernels_tc.cu -o $D/kernels_tc_exp.o
objs=$(ls $B/*.o | grep -v kernels_tc.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libstreamconv_b200.so $D/kernels_tc_exp.o $objs -lcuda -lcufft
echo $D/libstreamconv_b200.so
