timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/pytest_wide.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wide.log
timeout 1200 python tools/run_2d_full.py c3 16 --check > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
timeout 1200 python tools/run_2d_full.py c4 16 --check > gpurun_out/full_c4.json 2> gpurun_out/full_c4.err
timeout 1800 python tools/run_2d_full.py c5 8 --check > gpurun_out/full_c5.json 2> gpurun_out/full_c5.err
