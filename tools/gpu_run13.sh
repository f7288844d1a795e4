timeout 300 python tools/prof_c2.py solve > gpurun_out/plain13.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1f_' -s 9 -c 8 -o gpurun_out/prof_c2c python tools/prof_c2.py solve > gpurun_out/ncu13.log 2>&1
