# Round artifacts: bench line, reference arm, launch list, one-sweep ncu capture, config suite
set -x
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-inflight 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:onesweep_kernel -s 4 -c 1 -o gpurun_out/os_bench python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-inflight 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 1200 python scripts/bench_suite.py --out gpurun_out/bench_suite.json > gpurun_out/bench_suite.log 2>&1; echo "suite rc=$?"
