# A/B timing experiment (outputs one line per run), alternating order
export SC_SKIP_BUILD=1
run() { echo "== $1 :: $2"; env $1 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print(round(d['value']/1e6,1), round(d['ms_per_step'],4), {k[:14]:v for k,v in sorted(p.items(), key=lambda x:-x[1])[:6]})"; }
for cfg in "--config 2 --steps 20 --warmup 5 --precision bf16" "--config 3 --steps 20 --warmup 5 --precision bf16" "--config 4 --steps 20 --warmup 5 --precision bf16" "--config 5 --steps 10 --warmup 5 --precision bf16"; do
  run "X=1" "$cfg"
  run "SC_LIB_PATH=exp_prev/libstreamconv_b200.so" "$cfg"
done
