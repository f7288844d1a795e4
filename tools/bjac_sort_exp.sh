# Block-Jacobi sweep-level norm ordering experiment (AZ_BJAC_SORT): per-sweep off-diagonal measure and
# bjac_round time of the full-size 2-D solves with and without it.
set -x
for s in 0 1; do
  for c in "c4 16" "c3 16"; do
    set -- $c
    AZ_BJAC_SORT=$s AZ_DEBUG_JACOBI=1 timeout 600 python tools/run_2d_full.py $1 $2 > gpurun_out/sort_$1_$s.json 2> gpurun_out/sort_$1_$s.err
  done
done
AZ_BJAC_SORT=1 AZ_DEBUG_JACOBI=1 timeout 600 python tools/run_2d_full.py c5 6 > gpurun_out/sort_c5_1.json 2> gpurun_out/sort_c5_1.err
AZ_BJAC_SORT=1 timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/sort_wide_tests.log 2>&1
tail -3 gpurun_out/sort_wide_tests.log
