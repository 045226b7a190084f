#!/bin/bash
# A/B per-cycle timing of library variants built under paper_1508_03235_b200/ab/
# usage: tools/ab_cycle.sh ENGINE [variant ...]
e=$1; shift
for v in "$@"; do
  echo "== $v"
  NOCSIM_LIB=$PWD/paper_1508_03235_b200/ab/$v.so timeout 300 python tools/cycle_time.py $e
done
