timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g12_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g12_pytest.txt
timeout 300 python scripts/probe.py scale > gpurun_out/g12_scale.txt 2>&1
timeout 900 python bench.py > gpurun_out/g12_bench.txt 2>&1
