timeout 600 python -m pytest tests/test_netsort_gpu.py tests/test_fullsize_gpu.py -k "netsort or c4 or network or btn or oet or merge" -x -q > gpurun_out/net_test.log 2>&1; echo rc=$?; tail -3 gpurun_out/net_test.log
timeout 300 python scripts/bench_suite.py --only C4 > gpurun_out/net_suite.log 2>&1; cut -c1-110 gpurun_out/net_suite.log
