AZ_DEBUG_JACOBI=1 python tools/prof_dense.py svd 3072 1 > gpurun_out/dbgj.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_bjac_round' -s 100 -c 1 -o gpurun_out/prof_bjac3 python tools/prof_dense.py svd 3072 1 > gpurun_out/ncu15.log 2>&1
