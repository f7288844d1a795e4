set -x
timeout 900 python tools/run_2d_full.py c4 16 --check > gpurun_out/full_c4.json 2> gpurun_out/full_c4.err
timeout 1200 python tools/run_2d_full.py c3 16 --check > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
