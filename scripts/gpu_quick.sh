#!/bin/bash
# Quick GPU iteration: stage times, launch list, GPU tests (outputs in gpurun_out/).
mkdir -p gpurun_out
BRSVD_DEBUG=1 python scripts/profile_c2.py --warm 2>&1 | tail -${DBG_TAIL:-3}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_c2.py > gpurun_out/prof_ncu_stdout.txt 2>&1
if [ -z "${NO_TESTS}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
  tail -3 gpurun_out/pytest_gpu.txt
fi
