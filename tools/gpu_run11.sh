timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solve.py -m gpu -x -q > gpurun_out/pytest_ops16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops16.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e16.json 2>&1
