set -x
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -x -q -k "factor" > gpurun_out/pytest_fac.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fac.log
timeout 900 python tools/run_2d_full.py c3 16 --factored --fac-only --fac-nrhs=1,2,4,8,16,24,32,64 > gpurun_out/fac_c3.json 2> gpurun_out/fac_c3.err
