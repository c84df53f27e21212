timeout 600 python -m pytest tests/test_radix_gpu.py tests/test_golden_gpu.py tests/test_acceptance_gpu.py -q -x 2>&1 | tail -2
AB_ROUNDS=3 timeout 900 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/e0/libbsg.so | grep SUMMARY
