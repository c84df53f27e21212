timeout 900 python -m pytest tests/test_pr_gpu.py tests/test_peer_ipc_gpu.py -q -x 2>&1 | tail -3
