for mb in 400 800 1600; do
AZ_SCRATCH_MB=$mb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mb$mb.json 2>&1
done
