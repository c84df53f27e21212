timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do for m in 0 2; do BSG_OS_RANK=$m timeout 120 python scripts/probe_pass.py 2>&1 | tail -1; done; done
timeout 600 python scripts/bench_suite.py --only C2 --out gpurun_out/suite_c2.json 2>&1 | tail -8 | cut -c1-120
BSG_OS_RANK=2 timeout 600 python scripts/bench_suite.py --only C2 --out gpurun_out/suite_c2_r2.json 2>&1 | tail -8 | cut -c1-120
