#!/bin/bash
# The measurement set of a round (outputs in gpurun_out/, summarised into
# profiles/ by scripts/summarize_ncu.py): the bench line, the launch list of
# one config-2 decomposition, an ncu --set full capture of the dominant
# kernel (the product), and the launch list of three config-5 iterations.
#   R=r02 bash scripts/gpu_round_profiles.sh
R=${R:-rNN}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${R}_smi.txt
timeout 900 python bench.py > gpurun_out/${R}_bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_c2.csv python scripts/profile_c2.py --warm > gpurun_out/${R}_prof_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tc3p_gemm} -s 2 -c 1 \
    -o gpurun_out/${R}_product_full -f python scripts/profile_c2.py > gpurun_out/${R}_ncu_full.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_c5.csv python scripts/probe.py c5 3 > gpurun_out/${R}_prof_c5.txt 2>&1
