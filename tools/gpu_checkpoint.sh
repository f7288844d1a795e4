# Round checkpoint on one B200 (run through gpurun from the repo root):
#   full GPU test suite, the bench line, the ncu launch list of the same bench command, and one
#   `ncu --set full` capture of the c2 hot kernels (each ncu run only after its command exited 0).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_c2.py solve > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_tsqr|k1f_rows|k1f_cols|k_jacobi_small|k_gemm_mn_small' -c 24 -o gpurun_out/prof_c2 \
  python tools/prof_c2.py solve > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
# summaries on the box; the full report only travels back when small (gpurun_out/ is capped at 64 MiB)
python tools/summarize_ncu.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
python tools/summarize_ncu.py full gpurun_out/prof_c2.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
[ "$(stat -c %s gpurun_out/prof_c2.ncu-rep 2>/dev/null || echo 0)" -gt 40000000 ] && rm -f gpurun_out/prof_c2.ncu-rep
rm -f gpurun_out/launches.csv.big
ls -la gpurun_out
