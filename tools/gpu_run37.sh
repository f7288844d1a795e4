set -x
timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -x -q -k "ellipse or disk or star or helm or box2d" > gpurun_out/pytest_aniso_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_aniso_ops.log
