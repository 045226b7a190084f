# A/B of library variants in abl/ (per-cycle timing at C3 + idle 208x208, C2, C1) then a GPU test subset
# usage: bash tools/gpu/ab_split.sh "base.so cur" [pytest -k expr]
cd $GRAFT_REPO_ROOT
for v in $1; do
  if [ "$v" = cur ]; then lib=$PWD/paper_1508_03235_b200/libnocsim.so; else lib=$PWD/abl/$v; fi
  NOCSIM_LIB=$lib timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
  NOCSIM_LIB=$lib timeout 300 python tools/cycle_time.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
if [ -n "$2" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/abtest.log 2>&1; tail -5 gpurun_out/abtest.log
fi
