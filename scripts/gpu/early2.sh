timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
AB_ROUNDS=3 timeout 900 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/e0/libbsg.so | grep SUMMARY
timeout 600 python scripts/bench_suite.py --only C2 --out gpurun_out/suite_c2.json 2>&1 | tail -8 | cut -c1-100
