#!/bin/bash
# Product-kernel iteration: tcs tests, product tests, one bench line, launch list.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcs.py tests/test_gpu_tc.py -x -q --timeout 300 > gpurun_out/pytest_tcs.txt 2>&1
tail -15 gpurun_out/pytest_tcs.txt
BRSVD_DEBUG=1 timeout 300 python scripts/profile_c2.py --warm 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_tcs.txt 2>&1
tail -1 gpurun_out/bench_tcs.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'launch_ms', d['roofline']['launch_ms'], 'frac', d['roofline']['frac'], d['stages_s'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_c2.py > gpurun_out/prof_ncu_stdout.txt 2>&1
python scripts/launch_summary.py gpurun_out/launches_c2.csv 2>&1 | head -30
