timeout 240 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider > gpurun_out/g33_tc.txt 2>&1; echo "exit $?" >> gpurun_out/g33_tc.txt
if grep -q "exit 0" gpurun_out/g33_tc.txt; then
timeout 300 python scripts/probe.py lsweep > gpurun_out/g33_lsweep.txt 2>&1
BRSVD_TCW=0 timeout 300 python scripts/probe.py lsweep > gpurun_out/g33_lsweep_p.txt 2>&1
fi
