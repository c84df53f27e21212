timeout 900 python scripts/ab_net.py paper_1708_09495_b200/libbsg.so build/var/mk8/libbsg.so build/var/mk32/libbsg.so build/var/minb4/libbsg.so build/var/minb6/libbsg.so 2>&1 | tail -24
