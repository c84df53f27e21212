timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python scripts/bench_suite.py --only PR --out gpurun_out/suite_pr.json 2>&1 | tail -6
