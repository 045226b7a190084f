# per-cycle times for several meshes (incl. the idle floor) + ncu --set full of the C3 TILED launch
cd $GRAFT_REPO_ROOT
timeout 300 python tools/cycle_time.py 3 > gpurun_out/cycle.log 2>&1
bash tools/gpu/prof.sh ${1:-r02a}
