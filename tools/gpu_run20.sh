python tools/tsqr_dbg.py > gpurun_out/tdbg.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_blk.json 2>&1
AZ_TSQR_OLD=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_old.json 2>&1
