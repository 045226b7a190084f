# A/B of library variants: C1a / C1b / C2 bench per-cycle times and C3 steady state
cd $GRAFT_REPO_ROOT
for v in $1; do
  for w in c1a c1b c2; do
    NOCSIM_LIB=$PWD/abl/$v timeout 300 python bench.py --workload $w --steps 5 --no-cpu-baseline --fresh 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w %.3f us/cycle block %d' % (d['ms_per_step']*1e3/d['config']['cycles_per_step'], d['config']['block']))"
  done
  NOCSIM_LIB=$PWD/abl/$v timeout 300 python tools/ab_c3.py 3 2>&1 | head -1 | sed "s/^/$v /"
done | tee gpurun_out/ab_small.txt
[ -n "$2" ] && NOCSIM_LIB=$PWD/abl/$2 timeout 1500 python -m pytest tests -m gpu -q -x -k "c1 or c2 or 4x4 or smoke or small or maximum or tiled" > gpurun_out/abtest.log 2>&1; tail -2 gpurun_out/abtest.log
