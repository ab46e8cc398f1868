#!/bin/bash
# Runs bench.py for every config / precision / buffer size; one JSON line each -> gpurun_out/bench_all.jsonl
export SC_SKIP_BUILD=1
out=gpurun_out/bench_all.jsonl
: > $out
run() { timeout 300 python bench.py "$@" --no-cpu-baseline 2>/dev/null | tail -1 >> $out || echo "{\"failed\": \"$*\"}" >> $out; }
run --config 2 --steps 20 --warmup 5
run --config 2 --steps 20 --warmup 5 --precision bf16
run --config 2 --steps 20 --warmup 5 --precision bf16 --io bf16
run --config 1 --steps 20 --warmup 5
run --config 3 --steps 20 --warmup 5
run --config 3 --steps 20 --warmup 5 --precision bf16
run --config 4 --steps 20 --warmup 5
run --config 4 --steps 20 --warmup 5 --precision bf16
run --config 5 --steps 10 --warmup 4
run --config 5 --steps 10 --warmup 4 --precision bf16
run --config 5 --steps 16 --warmup 8 --frames 512
run --config 5 --steps 6 --warmup 3 --frames 8192
run --config 5 --steps 10 --warmup 4 --streams 2048
SC_FP32_SPLIT=tf32 run --config 5 --steps 10 --warmup 4  # 3xTF32 A/B
