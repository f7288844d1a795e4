set -x
timeout 300 python tools/jac_sweep.py star_32 1 > gpurun_out/plain6.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bjac_round|k_qr_upd|k_qr_vtc|k_qr_panel' -s 20 -c 8 -o gpurun_out/prof_bjac python tools/jac_sweep.py star_32 1 > gpurun_out/ncu6.log 2>&1
