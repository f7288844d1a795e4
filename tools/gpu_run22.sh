timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solve.py tests/test_gpu_wide.py -m gpu -x -q -k "not full_size or c2" > gpurun_out/pytest22.log 2>&1; echo "rc=$?" >> gpurun_out/pytest22.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench22.json 2>&1
