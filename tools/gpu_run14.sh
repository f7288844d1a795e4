python tools/prof_dense.py qr 131072 2048 > gpurun_out/dense_plain.log 2>&1
python tools/prof_dense.py svd 3072 1 >> gpurun_out/dense_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bjac_round|k_qr_upd|k_qr_vtc|k_qr_panel' -s 30 -c 6 -o gpurun_out/prof_dense python tools/prof_dense.py qr 131072 2048 > gpurun_out/ncu14.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bjac_round' -s 200 -c 3 -o gpurun_out/prof_bjac2 python tools/prof_dense.py svd 3072 1 > gpurun_out/ncu14b.log 2>&1
