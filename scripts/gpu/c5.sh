timeout 1200 python -m pytest tests/test_pr_gpu.py tests/test_golden_gpu.py tests/test_peer_ipc_gpu.py -q -x 2>&1 | tail -3
timeout 900 python scripts/bench_suite.py --only C5,PR --out gpurun_out/suite_c5.json 2>&1 | tail -9
