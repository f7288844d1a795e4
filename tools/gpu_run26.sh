for cs in "" 1 2 4; do
AZ_BJAC_CS=$cs timeout 600 python tools/prof_dense.py svd 7720 1 >> gpurun_out/cs.log 2>&1
AZ_BJAC_CS=$cs timeout 600 python tools/prof_dense.py svd 3072 1 >> gpurun_out/cs.log 2>&1
done
