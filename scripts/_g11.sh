timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/g11_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g11_pytest.txt
timeout 300 python scripts/probe.py products > gpurun_out/g11_products.txt 2>&1
timeout 600 python scripts/bench_configs.py --configs c1,c5 > gpurun_out/g11_configs.txt 2>&1
