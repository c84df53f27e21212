for v in s0 s1 s1w8 s2; do BSG_LIB=$PWD/build/var/$v/libbsg.so timeout 120 python scripts/probe_lb.py; done
AB_ROUNDS=2 timeout 600 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/mb3/libbsg.so:1 paper_1708_09495_b200/libbsg.so:1 | grep SUMMARY
