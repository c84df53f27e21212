timeout 120 python scripts/probe_phases.py
BSG_LIB=$PWD/build/var/sleep100/libbsg.so timeout 120 python scripts/probe_phases.py | tail -1
AB_ROUNDS=3 timeout 600 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/sleep100/libbsg.so build/var/sleep400/libbsg.so | grep SUMMARY
