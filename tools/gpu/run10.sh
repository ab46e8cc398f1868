mkdir -p gpurun_out
for pf in 0 1 2 3 4; do
SC_PF_DIST=$pf timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_pf$pf.json 2> /dev/null
python tools/prof_table.py gpurun_out/bench_pf$pf.json > gpurun_out/prof_pf$pf.txt 2>&1
echo "pf=$pf"; head -12 gpurun_out/prof_pf$pf.txt
done
