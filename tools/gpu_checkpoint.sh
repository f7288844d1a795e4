# Round checkpoint on one B200 (run through gpurun from the repo root):
#   the bench line, the ncu launch list of the same bench command, and one `ncu --set full` capture
#   of the c2 hot kernels (each ncu run only after its command exited 0); summaries written on the
#   box (the full report stays there: gpurun_out/ is capped at 64 MiB).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-configs "" > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_c2.py solve > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'k_tsqr|k1f_rows|k1f_cols|k_jacobi_small|k_gemm_mn_small' -c 24 -o /tmp/prof_c2 \
  python tools/prof_c2.py solve > gpurun_out/ncu_full.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
python tools/summarize_ncu.py full /tmp/prof_c2.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
rm -f gpurun_out/launches.csv
bash tools/prof_c1.sh
ls -la gpurun_out
