export SC_SKIP_BUILD=1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/parity_table.py 2>&1 | grep "cfg4\|cfg5"
run() { echo "== $1 :: $2"; env $1 timeout 300 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print(round(d['value']/1e6,1), round(d['ms_per_step'],4), {k[:22]:round(v,3) for k,v in list(p.items())[-3:]})"; }
for i in 1 2; do
run "X=1" "--config 5 --steps 5 --warmup 3"
run "SC_DENSIFY4=0" "--config 5 --steps 5 --warmup 3"
run "X=1" "--config 4 --steps 10 --warmup 3"
run "SC_DENSIFY4=0" "--config 4 --steps 10 --warmup 3"
done
run "X=1" "--config 5 --steps 8 --warmup 4 --frames 512"
run "SC_DENSIFY4=0" "--config 5 --steps 8 --warmup 4 --frames 512"
