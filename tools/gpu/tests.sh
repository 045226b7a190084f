# full GPU test suite on the box; log + junit summary into gpurun_out/
cd $GRAFT_REPO_ROOT
timeout ${1:-3000} python -m pytest tests -m gpu -q -x --durations=15 ${2:-} > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
tail -40 gpurun_out/gputest.log
