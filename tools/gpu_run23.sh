timeout 300 python tools/prof_c2.py solve > gpurun_out/plain23.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1f_rows|k1f_cols' -s 6 -c 5 -o gpurun_out/prof_fft python tools/prof_c2.py solve > gpurun_out/ncu23.log 2>&1
