set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export NOCSIM_LIB=$PWD/paper_1508_03235_b200/_build/ab/trace.so
timeout 300 python tools/trace_tiled.py c3 6000 > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_tiled.py c2 6000 > gpurun_out/trace_c2.txt 2>&1
timeout 300 python tools/trace_tiled.py ur0 1000 > gpurun_out/trace_ur0.txt 2>&1
unset NOCSIM_LIB
timeout 300 python tools/ab_c3.py > gpurun_out/ab_base.txt 2>&1
cat gpurun_out/trace_*.txt gpurun_out/ab_base.txt
