timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench21.json 2>&1
timeout 1200 python tools/run_2d_full.py c3 16 --factored > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
timeout 1200 python tools/run_2d_full.py c4 16 --factored > gpurun_out/full_c4.json 2> gpurun_out/full_c4.err
