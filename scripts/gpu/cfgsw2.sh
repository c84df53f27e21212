for n in 24 25 26 28; do echo "== n=2^$n"; AB_ROUNDS=3 AB_N=$((1<<n)) timeout 400 python scripts/ab.py paper_1708_09495_b200/libbsg.so:6 paper_1708_09495_b200/libbsg.so:1 | grep SUMMARY; done
