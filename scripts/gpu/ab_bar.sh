AB_ROUNDS=4 timeout 1000 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/sn/libbsg.so | grep SUMMARY
