#!/bin/bash
# One GPU session: smoke, GPU parity tests, short bench.  Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
tail -5 gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
tail -40 gpurun_out/pytest_gpu.txt
if [ -z "${NO_BENCH}" ]; then
  timeout 900 python bench.py --steps ${STEPS:-2} --warmup ${WARMUP:-1} ${BENCH_ARGS} > gpurun_out/bench.txt 2>&1
  tail -5 gpurun_out/bench.txt
fi
