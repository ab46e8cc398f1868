# drain ablation: exp lib, full drain vs quarter TMEM reads
export SC_SKIP_BUILD=1
mkdir -p gpurun_out
run() { echo "== $1 :: $2"; env $1 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print(round(d['value']/1e6,1), round(d['ms_per_step'],4), {k[:10]:round(v,4) for k,v in p.items()})"; }
for i in 1 2; do
run "SC_LIB_PATH=exp/libstreamconv_b200.so SC_TC_DEBUG=0" "--config 5 --steps 5 --warmup 3"
run "SC_LIB_PATH=exp/libstreamconv_b200.so SC_TC_DEBUG=64" "--config 5 --steps 5 --warmup 3"
done
