AB_ROUNDS=3 timeout 900 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/c1/libbsg.so build/var/c2/libbsg.so build/var/c1w8/libbsg.so build/var/c2w8/libbsg.so | grep SUMMARY
