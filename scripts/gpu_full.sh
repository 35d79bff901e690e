#!/bin/bash
# Full GPU session: tests, bench line, launch list and one ncu --set full
# capture of the A-streaming product (fp16-split tcgen05 kernel).  Outputs in gpurun_out/.
mkdir -p gpurun_out
NO_BENCH=1 bash scripts/gpu_check.sh
timeout 900 python bench.py --steps ${STEPS:-5} --warmup ${WARMUP:-3} > gpurun_out/bench.txt 2>&1
tail -1 gpurun_out/bench.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_c2.py > gpurun_out/prof_ncu_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc3_gemm -s 0 -c 1 \
    -o gpurun_out/tc3_full -f python scripts/profile_c2.py > gpurun_out/ncu_full_stdout.txt 2>&1
tail -2 gpurun_out/ncu_full_stdout.txt
ls -la gpurun_out
