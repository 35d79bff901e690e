timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 10 > gpurun_out/g34_bench.txt 2>&1
BRSVD_TCW=0 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 10 > gpurun_out/g34_bench_p.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc3w -s 0 -c 1 -o gpurun_out/g34_tcw python scripts/profile_c2.py > gpurun_out/g34_ncu.log 2>&1
