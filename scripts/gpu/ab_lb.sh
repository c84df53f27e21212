V="paper_1708_09495_b200/libbsg.so"; for v in lam w2 w6 w8 c2 c1w8; do V="$V build/var/$v/libbsg.so"; done
AB_ROUNDS=3 timeout 1000 python scripts/ab.py $V | grep SUMMARY
