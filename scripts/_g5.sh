timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g5_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/g5_pytest.txt
BRSVD_CI_TIMING=1 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 1 --warmup 1 > gpurun_out/g5_citiming.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gram_dmma -s 2 -c 1 -o gpurun_out/g5_gram python bench.py --no-e2e --no-cpu --no-configs --steps 1 --warmup 1 > gpurun_out/g5_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cholinv -s 2 -c 1 -o gpurun_out/g5_chol python bench.py --no-e2e --no-cpu --no-configs --steps 1 --warmup 1 > gpurun_out/g5_ncu2.log 2>&1
