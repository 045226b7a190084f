cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -k "small_mesh or virtual_ranks or odd_tilings or edge_config or c1a or c1b or launch_bound or drain or scripted or virtual_bands_match" > gpurun_out/sub.log 2>&1; tail -3 gpurun_out/sub.log
bash tools/gpu/sanitize.sh
