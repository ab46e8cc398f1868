export SC_SKIP_BUILD=1
run() { echo "== $1 :: $2"; env $1 timeout 300 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print(round(d['value']/1e6,1), round(d['ms_per_step'],4), round(sum(p.values()),3))"; }
for i in 1 2 3; do
run "X=1" "--config 5 --steps 8 --warmup 3"
run "SC_LIB_PATH=exp2/libstreamconv_b200.so" "--config 5 --steps 8 --warmup 3"
run "SC_LIB_PATH=exp3/libstreamconv_b200.so" "--config 5 --steps 8 --warmup 3"
done
