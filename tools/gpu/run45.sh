for lib in paper_2204_07064_b200/lib/libstreamconv_b200.so exp2/libstreamconv_b200.so paper_2204_07064_b200/lib/libstreamconv_b200.so exp2/libstreamconv_b200.so; do
SC_LIB_PATH=$lib SC_SKIP_BUILD=1 timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
python -c "import json; a=json.load(open('gpurun_out/b.json')); p=a['profile_ms']; print('$lib', round(a['ms_per_step'],3), round(p['op29 conv 128->128 K3 d1 [tc-3xf16]'],4), round(p['op2 conv 64->64 K3 d1 [tc-3xf16]'],4))"
done
