python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -4
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
