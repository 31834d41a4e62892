#!/bin/bash
# A/B of library builds on the headline sorted sum: whole-range kernel time and 8 tile parts
for v in "$@"; do
  PAIRCOUNT_LIB=build/ab/$v.so python scripts/ab_sorted.py 5 | sed "s/^/$v /"
  PAIRCOUNT_LIB=build/ab/$v.so python scripts/part_overhead.py | grep sorted | sed "s/^/$v /"
done
