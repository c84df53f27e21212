# one-sweep timing with debug bits (1 = skip look-back, 2 = trivial ranks); results invalid, timing only
for d in 0 1 2 3; do echo "dbg=$d"; BSG_OS_DBG=$d python scripts/probe_phases.py | head -1; done
