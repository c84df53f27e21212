AB_ROUNDS=3 timeout 1000 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/w2/libbsg.so build/var/w3/libbsg.so build/var/w6/libbsg.so build/var/w8/libbsg.so | grep SUMMARY
