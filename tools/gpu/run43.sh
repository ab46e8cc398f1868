for a in "--config 3" "--config 4" "--config 5 --streams 256" "--config 5 --streams 2048" "--config 5 --streams 8192"; do
timeout 60 python bench.py --no-cpu-baseline --steps 3 --warmup 3 $a > gpurun_out/b.json 2>/dev/null
echo "$a rc=$?"
done
SC_DISABLE_WIN=1 timeout 60 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --config 5 --streams 2048 > /dev/null 2>&1; echo "nowin rc=$?"
SC_AWIN=0 timeout 60 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --config 5 --streams 2048 > /dev/null 2>&1; echo "noawin rc=$?"
