# one-sweep timing with debug bits (results invalid, timing only):
# 1 = skip look-back, 2 = trivial ranks, 4 = skip write-out, 16 = skip staging
for d in ${DBG_LIST:-0 1 2 3 4 16 20}; do echo "dbg=$d"; BSG_OS_DBG=$d python scripts/probe_phases.py | head -1; done
