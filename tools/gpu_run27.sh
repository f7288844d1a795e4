timeout 1200 python tools/run_2d_full.py c3 16 > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
timeout 1200 python tools/run_2d_full.py c4 16 > gpurun_out/full_c4.json 2> gpurun_out/full_c4.err
timeout 1800 python tools/run_2d_full.py c5 6 > gpurun_out/full_c5.json 2> gpurun_out/full_c5.err
