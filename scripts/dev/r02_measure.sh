# Round-2 measurement pass: bench line (driver settings), reference arm, config suite, CSV,
# launch list and ncu captures of bench.py's passes; only text summaries come back.
set -x
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo bench=$?
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
echo ref=$?
timeout 1200 python scripts/bench_suite.py --out gpurun_out/r02_suite.jsonl > gpurun_out/r02_suite.log 2>&1
echo suite=$?
timeout 900 python scripts/bench_csv.py --sizes 2^20,2^24 --procs 2,4,8 --reps 2 --out gpurun_out/r02_bench.csv > gpurun_out/r02_csv.log 2>&1
echo csv=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02_ncu_bench.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k 'regex:onesweep_kernel|first_pass_kernel' -s 16 -c 4 -o /tmp/r02_passes python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02_ncu_passes.log 2>&1
echo ncu_passes=$?
ncu -i /tmp/r02_passes.ncu-rep --page details > gpurun_out/r02_passes_ncu_details.txt
ncu -i /tmp/r02_passes.ncu-rep --page raw --csv > gpurun_out/r02_passes_ncu_raw.csv
python scripts/dev/srcprof.py /tmp/r02_passes.ncu-rep 60 > gpurun_out/r02_passes_ncu_source_hotspots.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:block_network_reg -s 1 -c 1 -o /tmp/r02_netreg python scripts/dev/prof_net.py 0 8 > gpurun_out/r02_ncu_net.log 2>&1
echo ncu_net=$?
ncu -i /tmp/r02_netreg.ncu-rep --page details > gpurun_out/r02_block_network_reg_ncu_details.txt
ncu -i /tmp/r02_netreg.ncu-rep --page raw --csv > gpurun_out/r02_block_network_reg_ncu_raw.csv
ls -la gpurun_out
