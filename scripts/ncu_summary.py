"""Summarise an .ncu-rep (details page) and a launch-list CSV."""
import csv, subprocess, sys
from collections import defaultdict

def details(rep, keys=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ks, ns, us, vs = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    res = []
    for r in rows[1:]:
        if len(r) <= vs:
            continue
        if keys is None or any(k in r[ns] for k in keys):
            res.append((r[hdr.index("Kernel Name")][:60], r[ks], r[ns], r[us], r[vs]))
    return res

def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = {}
    for m in metrics:
        if m in hdr:
            res[m] = [(rows[1][hdr.index(m)], r[hdr.index(m)]) for r in rows[2:]]
    return res

def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0][-60:]].append(float(r[vi]))
    tot = sum(sum(v) for v in d.values())
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:62s} n={len(v):4d} avg={sum(v)/len(v)/1e3:9.1f}us share={sum(v)/tot*100:5.1f}%")

if __name__ == "__main__":
    if sys.argv[1].endswith(".csv"):
        launches(sys.argv[1])
    else:
        keys = sys.argv[2].split(",") if len(sys.argv) > 2 else None
        for r in details(sys.argv[1], keys):
            print(" | ".join(r[1:]))
