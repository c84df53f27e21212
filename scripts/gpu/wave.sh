timeout 900 python -m pytest tests/test_radix_gpu.py tests/test_golden_gpu.py tests/test_acceptance_gpu.py -q -x 2>&1 | tail -2
for lg in 16 18 20 21; do echo "n=2^$lg"; AB_N=$((1<<lg)) AB_ROUNDS=3 timeout 300 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/w0/libbsg.so | grep SUMMARY; done
