# Block-Jacobi cluster-size experiment on the full-size 2-D solves: the bjac_round time of c5 / c3
# for several AZ_BJAC_CS (CTAs per block pair; the round's waves = ceil(pairs * CS / 148)).
set -x
for cs in 2 3 6; do
  AZ_BJAC_CS=$cs timeout 600 python tools/run_2d_full.py c5 6 > gpurun_out/cs_c5_$cs.json 2> gpurun_out/cs_c5_$cs.err
done
for cs in 1 6; do
  AZ_BJAC_CS=$cs timeout 600 python tools/run_2d_full.py c3 16 > gpurun_out/cs_c3_$cs.json 2> gpurun_out/cs_c3_$cs.err
done
