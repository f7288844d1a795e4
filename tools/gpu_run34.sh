set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tsgemv' -c 2 -o gpurun_out/prof_tsgemv python tools/run_2d_full.py c3 16 --factored --fac-only > gpurun_out/ncu34.log 2>&1
