# compute-sanitizer memcheck / racecheck / synccheck over the UR split-barrier TILED path
cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/scripts/sanitize_split.py ${1:-60} > gpurun_out/san_split_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_split_$tool.log
  tail -4 gpurun_out/san_split_$tool.log
done
