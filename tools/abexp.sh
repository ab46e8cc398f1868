# A/B timing experiment: variants via env (outputs one line per run)
export SC_SKIP_BUILD=1
run() { echo "== $1 :: $2"; env $1 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,1))"; }
for cfg in "--config 1 --steps 50 --warmup 5" "--config 2 --steps 20 --warmup 5" "--config 4 --steps 20 --warmup 5" "--config 5 --steps 10 --warmup 5"; do
  run "SC_GRAPHS_PER_PLAN=1" "$cfg"
  run "SC_GRAPHS_PER_PLAN=8" "$cfg"
done
