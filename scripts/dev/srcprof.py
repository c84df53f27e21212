"""Aggregate an ncu source page (sass+cuda) by CUDA source line."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            ex = int(r[7]); st = int(r[4])
        except ValueError:
            continue
        k = (fname, int(r[0]))
        agg[k][0] += ex; agg[k][1] += st; agg[k][2] = r[1].strip()[:90]
tot = sum(v[0] for v in agg.values()); tst = sum(v[1] for v in agg.values())
print("total warp-instr", tot, "stall samples", tst)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / tot + kv[1][1] / max(tst, 1)))[:n]:
    print(f"ins {v[0]/tot*100:5.1f}%  stall {v[1]/max(tst,1)*100:5.1f}%  {k[0]}:{k[1]:<4d} {v[2]}")
