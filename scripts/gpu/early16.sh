timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for n in 22 23 24 25; do echo "n=2^$n"; AB_ROUNDS=3 AB_N=$((1<<n)) timeout 300 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/head/libbsg.so | grep SUMMARY; done
