timeout 300 python tools/prof_c2.py solve > gpurun_out/plain9.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1f_rows|k1f_cols|k_tsqr|k_jacobi' -s 60 -c 14 -o gpurun_out/prof_c2b python tools/prof_c2.py solve > gpurun_out/ncu9.log 2>&1
