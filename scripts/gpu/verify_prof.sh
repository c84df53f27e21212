timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:onesweep_kernel -s 2 -c 1 -o gpurun_out/os_full2 python scripts/prof_pass.py > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
