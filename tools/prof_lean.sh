#!/bin/bash
# ncu --set full of one 2000-cycle TILED launch (engine ${2:-3}) at C3; report -> gpurun_out/prof_$1_c3.ncu-rep
tag=$1; eng=${2:-3}; wl=${3:-c3}
ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 1 -c 1 -o gpurun_out/prof_${tag}_${wl} -f \
  python tools/prof_run.py --workload $wl --engine $eng --warm 6000 --cycles 2000 --launches 1 > gpurun_out/prof_${tag}.log 2>&1
