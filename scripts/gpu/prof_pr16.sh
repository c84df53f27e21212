BITS=16 P=8 REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pr16_launches.csv python scripts/probe_pr.py > /dev/null 2>&1; echo rc=$?
