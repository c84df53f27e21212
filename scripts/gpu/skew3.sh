timeout 900 python -m pytest tests/test_pr_gpu.py tests/test_golden_gpu.py -q -x 2>&1 | tail -2
timeout 600 python scripts/bench_suite.py --only PR --out gpurun_out/suite_pr.json 2>&1 | tail -6 | cut -c1-100
