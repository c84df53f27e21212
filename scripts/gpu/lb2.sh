for v in "" w2 w8 w16; do
  if [ -n "$v" ]; then export BSG_LIB=$PWD/build/var/$v/libbsg.so; fi
  echo "== $v"; timeout 120 python scripts/probe_phases.py | tail -1
done
unset BSG_LIB
AB_ROUNDS=3 timeout 900 python scripts/ab.py paper_1708_09495_b200/libbsg.so build/var/w2/libbsg.so build/var/w8/libbsg.so build/var/w16/libbsg.so build/var/old/libbsg.so | grep SUMMARY
