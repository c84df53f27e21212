BSG_OS_RANK=3 timeout 600 python -m pytest tests/test_radix_gpu.py tests/test_golden_gpu.py -q -x 2>&1 | tail -2
for r in 1 2 3; do for m in 0 3; do BSG_OS_RANK=$m timeout 120 python scripts/probe_pass.py 2>&1 | tail -1; done; done
