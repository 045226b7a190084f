cd $GRAFT_REPO_ROOT
NOCSIM_LIB=$PWD/paper_1508_03235_b200/_build/ab/trace.so timeout 300 python tools/trace_tiled.py c3 6000 > gpurun_out/trace2_c3.txt 2>&1
NOCSIM_LIB=$PWD/paper_1508_03235_b200/_build/ab/trace.so timeout 300 python tools/trace_tiled.py ur0 1000 > gpurun_out/trace2_ur0.txt 2>&1
cat gpurun_out/trace2_c3.txt gpurun_out/trace2_ur0.txt
bash tools/gpu/tests.sh 3000
