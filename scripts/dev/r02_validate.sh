# HEAD validation: GPU tests, then the bench line, launch list and ncu captures of both passes.
set -x
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
echo tests=$?
tail -5 gpurun_out/gputests.log
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo bench=$?
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02_ncu_bench.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:onesweep_kernel -s 6 -c 1 -o gpurun_out/r02_onesweep python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02_ncu_os.log 2>&1
echo ncu_os=$?
ncu --set full --clock-control none --import-source on -k regex:first_pass_kernel -s 2 -c 1 -o gpurun_out/r02_firstpass python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02_ncu_fp.log 2>&1
echo ncu_fp=$?
