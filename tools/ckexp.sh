export SC_SKIP_BUILD=1
for ck in 1 2 4; do
  echo "== CK=$ck"
  SC_TC_CK=$ck python tools/diag_parity.py 2>&1 | grep "^cfg[0-9] "
  for c in 2 5; do SC_TC_CK=$ck python bench.py --config $c --steps 10 --warmup 4 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print($c, round(d['value']/1e6,1), d['roofline']['kernel'], round(d['roofline']['achieved'],1))"; done
done
