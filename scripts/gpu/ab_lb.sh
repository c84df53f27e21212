for v in se1; do BSG_LIB=$PWD/build/var/$v/libbsg.so timeout 120 python scripts/probe_lb.py; done
V="paper_1708_09495_b200/libbsg.so"; for v in e1 e1w2 e1w6 e1w8; do V="$V build/var/$v/libbsg.so"; done
AB_ROUNDS=3 timeout 1000 python scripts/ab.py $V | grep SUMMARY
