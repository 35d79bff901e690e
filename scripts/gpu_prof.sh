#!/bin/bash
# Launch list (per-kernel device time) of one config-2 decomposition.
mkdir -p gpurun_out
python scripts/profile_c2.py --warm > gpurun_out/prof_plain.txt 2>&1
cat gpurun_out/prof_plain.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_c2.py ${PROF_ARGS} > gpurun_out/prof_ncu_stdout.txt 2>&1
tail -3 gpurun_out/prof_ncu_stdout.txt
