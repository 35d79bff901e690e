timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/g4_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g4_pytest.txt
for v in 0 1; do BRSVD_GRAM_SIMT=$v timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 10 > gpurun_out/g4_bench_simt$v.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gram -c 20 python bench.py --no-e2e --no-cpu --no-configs --steps 1 --warmup 1 > gpurun_out/g4_ncu_gram.txt 2>&1
