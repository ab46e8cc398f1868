for v in 0 1; do
SC_DISABLE_WIN=$v timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_win$v.json 2> /dev/null
python tools/prof_table.py gpurun_out/bench_win$v.json > gpurun_out/prof_win$v.txt 2>&1
done
paste gpurun_out/prof_win0.txt gpurun_out/prof_win1.txt | head -42
timeout 600 python bench.py --no-cpu-baseline --streams 2048 > gpurun_out/bench_2048.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_2048.json')); print('2048 streams', d['ms_per_step'])"
