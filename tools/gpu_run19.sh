timeout 300 python tools/prof_c2.py solve > gpurun_out/plain19.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tsqr' -c 1 -o gpurun_out/prof_tsqr python tools/prof_c2.py solve > gpurun_out/ncu19.log 2>&1
