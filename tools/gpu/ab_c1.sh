# A/B of library variants on the C1 bench workloads (per-cycle times from bench.py) + C1 parity with the last
cd $GRAFT_REPO_ROOT
for v in $1; do
  for w in c1a c1b; do
    NOCSIM_LIB=$PWD/abl/$v timeout 300 python bench.py --workload $w --steps 5 --no-cpu-baseline --fresh 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w %.3f us/cycle block %d' % (d['ms_per_step']*1e3/d['config']['cycles_per_step'], d['config']['block']))"
  done
done | tee gpurun_out/ab_c1.txt
NOCSIM_LIB=$PWD/abl/${2:-def.so} timeout 900 python -m pytest tests -m gpu -q -x -k "c1 or smoke or 4x4 or maximum" > gpurun_out/abtest.log 2>&1; tail -2 gpurun_out/abtest.log
