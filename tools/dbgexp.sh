# timing-only experiment: SC_TC_DEBUG bits disable parts of the fp32 TC kernel (outputs garbage)
export SC_SKIP_BUILD=1
for d in 0 2 256 512 1024 1026 768 258 770 136; do
  SC_TC_DEBUG=$d python bench.py --config 2 --steps 10 --warmup 4 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); p=d['profile_ms']; print($d, round(d['value']/1e6,1), p['op0 conv 128->128 K3 d1 [tc]'], p['op1 conv 128->128 K1 d1 [tc]'])"
done
