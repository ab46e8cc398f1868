set -x
mkdir -p gpurun_out
SC_SKIP_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "fp32 or bit_identity or graph_vs" > gpurun_out/pytest_hf.log 2>&1
tail -15 gpurun_out/pytest_hf.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_hf_cfg5.json 2> gpurun_out/bench_hf_cfg5.err
SC_FP32_SPLIT=tf32 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_tf_cfg5.json 2> gpurun_out/bench_tf_cfg5.err
python tools/prof_table.py gpurun_out/bench_hf_cfg5.json > gpurun_out/prof_hf.txt 2>&1
python tools/prof_table.py gpurun_out/bench_tf_cfg5.json > gpurun_out/prof_tf.txt 2>&1
paste gpurun_out/prof_tf.txt gpurun_out/prof_hf.txt | head -60
tail -3 gpurun_out/bench_hf_cfg5.err
