# A/B timing experiment (outputs one line per run), alternating order:
#   bash tools/abexp.sh "<bench args>" ...   (current build vs exp_prev/libstreamconv_b200.so)
export SC_SKIP_BUILD=1
run() { echo "== $1 :: $2"; env $1 python bench.py $2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print(round(d['value']/1e6,1), round(d['ms_per_step'],4), {k[:14]:round(v,4) for k,v in sorted(p.items(), key=lambda x:-x[1])[:4]})"; }
for cfg in "$@"; do
  for i in 1 2; do
    run "X=1" "$cfg"
    run "SC_LIB_PATH=exp_prev/libstreamconv_b200.so" "$cfg"
  done
done
