#!/bin/bash
# onesweep config sweep over sizes (development aid)
for n in 20 22 24 26; do
  echo "== n=2^$n"
  AB_ROUNDS=2 AB_N=$((1<<n)) python scripts/ab.py "$@" | grep SUMMARY
done
