#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tcs.py -x -q --timeout 120 > gpurun_out/pytest_tcs.txt 2>&1
tail -12 gpurun_out/pytest_tcs.txt
timeout 300 python scripts/tcs_exp.py 2>&1 | tail -14
