# Round-2 measurement pass: bench line, config suite, launch list, ncu captures.
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo bench=$?
timeout 1200 python scripts/bench_suite.py --out gpurun_out/r02_suite.jsonl > gpurun_out/r02_suite.log 2>&1
echo suite=$?
timeout 900 python scripts/bench_csv.py --sizes 2^20,2^24 --procs 2,4,8 --reps 2 --out gpurun_out/r02_bench.csv > gpurun_out/r02_csv.log 2>&1
echo csv=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_bench.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:onesweep_kernel -s 6 -c 1 -o gpurun_out/r02_onesweep python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_os.log 2>&1
echo ncu_os=$?
ncu --set full --clock-control none --import-source on -k regex:block_network_reg -s 1 -c 1 -o gpurun_out/r02_netreg python scripts/dev/prof_net.py 0 8 > gpurun_out/r02_ncu_net.log 2>&1
echo ncu_net=$?
