BRSVD_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_tcs.py -x -q -k "40000 or 33000" --timeout 300 2>&1 | grep "brsvd\] tcs\|passed\|failed" | head -20
BRSVD_DEBUG=1 timeout 300 python scripts/profile_c2.py 2>&1 | grep "tcs\|wall\|Error" | head
