timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for lg in 16 20 21; do echo "n=2^$lg"; AB_N=$((1<<lg)) AB_ROUNDS=3 timeout 400 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/prev/libbsg.so | grep SUMMARY; done
timeout 600 python scripts/bench_suite.py --only PR --out gpurun_out/suite_pr.json 2>&1 | tail -6 | cut -c1-100
