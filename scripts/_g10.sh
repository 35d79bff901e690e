timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/g10_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g10_pytest.txt
timeout 300 python scripts/probe.py products > gpurun_out/g10_products.txt 2>&1
BRSVD_SKINNY_SIMT=1 timeout 300 python scripts/probe.py products > gpurun_out/g10_products_simt.txt 2>&1
timeout 600 python scripts/bench_configs.py --configs c1,c5 > gpurun_out/g10_configs.txt 2>&1
