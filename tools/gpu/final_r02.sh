# round-2 measurement pass: smoke, default bench (C3) + launch list, the other bench workloads, C5 ncu, GPU tests
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fresh 0 > gpurun_out/bench_ncu.log 2>&1
for w in ${1:-c4ur c5 c1a c1b c2}; do
  echo "# bench.py --workload $w" >> gpurun_out/bench_all.jsonl
  timeout 900 python bench.py --workload $w --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl
done
[ -n "$2" ] && bash tools/gpu/prof_c5.sh $2
timeout ${3:-2400} python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
tail -30 gpurun_out/gputest.log
tail -n 3 gpurun_out/bench.log gpurun_out/smoke.log
