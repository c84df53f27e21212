timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
AB_ROUNDS=4 timeout 1200 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/head/libbsg.so build/var/e0/libbsg.so | grep SUMMARY
