# c1 latency profile on one B200 (run through gpurun from the repo root): the per-kernel breakdown of
# one c1 solve, and ncu --set full of its TSQR, one-CTA Jacobi and chain kernels (summary on the box).
python tools/c1_latency.py c1 1 > gpurun_out/c1_plain.txt 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'k_jacobi_small|k_tsqr|k_chain1s|k_gemm_mn_small' -s 40 -c 6 -o /tmp/prof_c1 \
  python tools/c1_latency.py c1 1 > gpurun_out/c1_ncu.log 2>&1
python tools/summarize_ncu.py full /tmp/prof_c1.ncu-rep > gpurun_out/c1_ncu_full.txt 2>&1
