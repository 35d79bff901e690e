timeout 600 python -m pytest tests/test_gpu_lazy_scales.py tests/test_gpu_tc.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/g41_t.txt 2>&1; echo "exit $?" >> gpurun_out/g41_t.txt
timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 10 > gpurun_out/g41_bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g41_launches.csv python bench.py --no-e2e --no-cpu --no-configs --steps 1 --warmup 1 > gpurun_out/g41_ncu.log 2>&1
