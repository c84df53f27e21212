# ncu --set full capture of the four passes of one 2^28 sort; text summaries only come back
set -x
ncu --set full --clock-control none --import-source on -k 'regex:onesweep_kernel|first_pass_kernel' -s 4 -c 4 -o /tmp/passes python scripts/dev/prof_pass.py 268435456 sort > gpurun_out/ncu_passes.log 2>&1
echo ncu=$?
ncu -i /tmp/passes.ncu-rep --page details > gpurun_out/passes_details.txt
ncu -i /tmp/passes.ncu-rep --page raw --csv > gpurun_out/passes_raw.csv
python scripts/dev/ncu_brief.py /tmp/passes.ncu-rep > gpurun_out/passes_brief.txt
ncu -i /tmp/passes.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/passes_source.csv 2>/dev/null
ls -la gpurun_out /tmp/passes.ncu-rep
