set -x
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/pytest_wide.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wide.log
timeout 600 python -m pytest tests/test_gpu_solve.py -m gpu -x -q > gpurun_out/pytest_solve.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_solve.log
