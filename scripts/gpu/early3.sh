timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
AB_ROUNDS=4 timeout 900 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/e0/libbsg.so | grep SUMMARY
for v in "" ; do timeout 200 python scripts/probe_sorted.py 2>&1 | tail -4; done
