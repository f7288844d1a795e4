timeout 600 python -m pytest tests/test_gpu_wide.py -m gpu -x -q -k "not full_size" > gpurun_out/pw.log 2>&1; echo "rc=$?" >> gpurun_out/pw.log
rm -f gpurun_out/cs.log
for pre in 1 0; do
AZ_BJAC_PRECOND=$pre timeout 600 python tools/prof_dense.py svd 7720 1 >> gpurun_out/cs.log 2>&1
AZ_BJAC_PRECOND=$pre timeout 600 python tools/prof_dense.py svd 3072 1 >> gpurun_out/cs.log 2>&1
done
AZ_DEBUG_JACOBI=1 timeout 1200 python tools/run_2d_full.py c3 16 > gpurun_out/full_c3.json 2> gpurun_out/full_c3.err
