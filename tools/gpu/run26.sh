timeout 600 ncu --set full --import-source on --clock-control none -k regex:pqmf --launch-count 2 -f -o gpurun_out/pqmf python tools/ncu_one.py 5 4096 > gpurun_out/ncu_pq.log 2>&1
