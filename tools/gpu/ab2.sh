# A/B per-cycle timing of library variants under ab/ (or "cur") + an optional pytest subset
# usage: bash tools/gpu/ab2.sh "base.so cur" [pytest -k expr]
cd $GRAFT_REPO_ROOT
for v in $1; do
  if [ "$v" = cur ]; then lib=$PWD/paper_1508_03235_b200/libnocsim.so; else lib=$PWD/ab/$v; fi
  NOCSIM_LIB=$lib timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
if [ -n "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/abtest.log 2>&1; tail -15 gpurun_out/abtest.log
fi
