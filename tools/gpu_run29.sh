

timeout 2400 python tools/run_2d_full.py c5 6 --check --factored > gpurun_out/full_c5.json 2> gpurun_out/full_c5.err
