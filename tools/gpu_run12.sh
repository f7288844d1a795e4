AZ_FFT_E=17 timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -x -q > gpurun_out/pytest_ops17.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops17.log
AZ_FFT_E=17 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e17.json 2>&1
