#!/bin/bash
mkdir -p gpurun_out
python scripts/dbg_range.py 2>&1 | tail -6
ncu --set full --clock-control none --import-source on -k regex:tcs_gemm -s 0 -c 2 \
    -o gpurun_out/tcs_full -f python scripts/profile_c2.py > gpurun_out/ncu_tcs_stdout.txt 2>&1
tail -2 gpurun_out/ncu_tcs_stdout.txt
