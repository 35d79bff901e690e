#!/bin/bash
# ncu --set full capture of one kernel of a config-2 decomposition.
#   KREGEX=<kernel regex> [KSKIP=n] [KOUT=name] bash scripts/gpu_prof_kernel.sh
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${KSKIP:-0} -c 1 \
    -o gpurun_out/${KOUT:-kernel_full} -f python scripts/profile_c2.py ${PROF_ARGS} > gpurun_out/ncu_${KOUT:-kernel_full}.txt 2>&1
tail -3 gpurun_out/ncu_${KOUT:-kernel_full}.txt
