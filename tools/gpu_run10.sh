timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench10s.json 2>&1
