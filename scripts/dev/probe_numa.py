"""Host topology vs pinned-copy bandwidth: copy rates with the process bound to each NUMA node (development aid)."""
import os, subprocess, sys, glob
print(subprocess.run("nvidia-smi topo -m; lscpu | grep -i -E 'numa|socket|model name|^CPU\\(s\\)'; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c",
                     shell=True, capture_output=True, text=True).stdout)
print("affinity", sorted(os.sched_getaffinity(0)))
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes", nodes)
child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe_pcie.py")
def cpus_of(node):
    s = open(node + "/cpulist").read().strip(); out = []
    for part in s.split(","):
        a, _, b = part.partition("-"); out += list(range(int(a), int(b or a) + 1))
    return out
for node in nodes or [None]:
    if node:
        cp = [c for c in cpus_of(node) if c in os.sched_getaffinity(0)]
        if not cp: print(node, "no allowed cpus"); continue
        pre = "import os; os.sched_setaffinity(0, %r); " % cp
    else:
        pre = ""
    r = subprocess.run([sys.executable, "-c", pre + "exec(open(%r).read())" % child], capture_output=True, text=True)
    print(node, r.stdout.strip().replace("\n", " | "), r.stderr[-300:])
