timeout 300 python -m pytest tests/test_pr_gpu.py -q -x -k "peer or fused or world1" 2>&1 | grep -v "^\[rank" | tail -30
