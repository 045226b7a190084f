# compute-sanitizer memcheck / racecheck / synccheck over every engine (small meshes)
cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py 60 > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
  tail -4 gpurun_out/san_$tool.log
done
