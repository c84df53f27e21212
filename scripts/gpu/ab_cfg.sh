AB_ROUNDS=3 timeout 1000 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/m4/libbsg.so:7 build/var/m3/libbsg.so:7 build/var/m4w8/libbsg.so:7 build/var/m4w2/libbsg.so:7 | grep SUMMARY
