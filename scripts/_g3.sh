timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "shards or overflow" > gpurun_out/g3_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g3_pytest.txt
timeout 600 python scripts/bench_configs.py --configs c4,c3 --c3-rows 50000 --steps 2 > gpurun_out/g3_c4.txt 2>&1
