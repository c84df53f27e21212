"""Print the headline counters of an .ncu-rep (details page)."""
import csv, subprocess, sys

KEYS = ['Duration', 'DRAM Throughput', 'Issue Slots', 'Executed Ipc A', 'Registers Per', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Warp Cycles Per Issued', 'Bank Conflicts', 'Executed Instructions',
        'L1/TEX Hit', 'Memory Throughput', 'Compute (SM) Throughput', 'Shared Memory']
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for x in rows[1:]:
    n = x[h.index('Metric Name')]
    if any(k in n for k in KEYS):
        print(x[h.index('Kernel Name')][:40], '|', x[h.index('Section Name')][:28], '|', n, x[h.index('Metric Unit')],
              x[h.index('Metric Value')])
