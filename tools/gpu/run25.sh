SC_SKIP_BUILD=1 timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b.json 2>/dev/null
python tools/prof_table.py gpurun_out/b.json | grep -E "pqmf|ingest|egress|step"
