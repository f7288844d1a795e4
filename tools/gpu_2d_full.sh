# Full-size 2-D solves (BASELINE c3, c4, c5 and the anisotropic ellipse) and factorisation reuse; results under gpurun_out/full_*.json.
set -x
timeout 1200 python tools/run_2d_full.py c4 16 --factored > gpurun_out/full_c4.json 2> gpurun_out/full_c4.err
timeout 1200 python tools/run_2d_full.py c3 16 --factored --fac-nrhs=1,8,64 > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
timeout 2400 python tools/run_2d_full.py c5 6 --factored --fac-nrhs=1,8 > gpurun_out/full_c5.json 2> gpurun_out/full_c5.err
timeout 1200 python tools/run_2d_full.py ellipse:256 16 --factored > gpurun_out/full_e256.json 2> gpurun_out/full_e256.err
