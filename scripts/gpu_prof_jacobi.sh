#!/bin/bash
mkdir -p gpurun_out
python scripts/profile_c2.py --warm > gpurun_out/prof_plain.txt 2>&1; cat gpurun_out/prof_plain.txt
ncu --set full --clock-control none --import-source on -k regex:jacobi_block -s 0 -c 1 \
    -o gpurun_out/jacobi_full -f python scripts/profile_c2.py > gpurun_out/ncu_jacobi_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"chol_kernel|trinv" -s 0 -c 2 \
    -o gpurun_out/chol_full -f python scripts/profile_c2.py > gpurun_out/ncu_chol_stdout.txt 2>&1
tail -2 gpurun_out/ncu_jacobi_stdout.txt
