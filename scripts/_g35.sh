timeout 240 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider > gpurun_out/g35_tc.txt 2>&1; echo "exit $?" >> gpurun_out/g35_tc.txt
timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 10 > gpurun_out/g35_bench.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g35_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/g35_pytest.txt
