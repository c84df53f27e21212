# GPU box session: gpu tests, bench line, one-sweep ncu capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:onesweep_kernel -s 2 -c 1 -o gpurun_out/os_full python scripts/prof_pass.py > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?"
