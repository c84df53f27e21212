# register block network: parity tests + optional A/B of variant libraries
timeout 600 python -m pytest tests/test_netsort_gpu.py tests/test_fullsize_gpu.py -k "netsort or c4 or network or btn or oet or merge" -x -q > gpurun_out/net_test.log 2>&1; echo rc=$?; tail -3 gpurun_out/net_test.log
if [ $# -gt 0 ]; then python scripts/dev/ab_net.py "$@"; fi
