timeout 900 python -m pytest tests/test_pr_gpu.py tests/test_peer_ipc_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do timeout 120 python scripts/probe_peer.py 2>&1 | tail -1; BSG_LIB=$PWD/build/var/prev/libbsg.so timeout 120 python scripts/probe_peer.py 2>&1 | tail -1; done
