mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16split.py -q -rf -x -k "fp32 or bit_identity or graph_vs or gain or signals or zero or splits" > gpurun_out/pytest_hf.log 2>&1
tail -5 gpurun_out/pytest_hf.log
for aw in 1 0; do
SC_AWIN=$aw timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_aw$aw.json 2> gpurun_out/bench_aw$aw.err
python tools/prof_table.py gpurun_out/bench_aw$aw.json > gpurun_out/prof_aw$aw.txt 2>&1
done
paste gpurun_out/prof_aw0.txt gpurun_out/prof_aw1.txt | head -45
