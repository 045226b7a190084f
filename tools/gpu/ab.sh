# A/B per-cycle timing of library variants + trace of the current build + TILED parity subset
# usage: bash tools/gpu/ab.sh "base.so cur" [pytest -k expr]
cd $GRAFT_REPO_ROOT
AB=paper_1508_03235_b200/_build/ab
for v in $1; do
  if [ "$v" = cur ]; then lib=$PWD/paper_1508_03235_b200/libnocsim.so; else lib=$PWD/$AB/$v; fi
  NOCSIM_LIB=$lib timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
if [ -f $AB/trace.so ]; then
  NOCSIM_LIB=$PWD/$AB/trace.so timeout 300 python tools/trace_tiled.py c3 6000 > gpurun_out/trace_cur_c3.txt 2>&1
  tail -4 gpurun_out/trace_cur_c3.txt
fi
if [ -n "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/abtest.log 2>&1; tail -3 gpurun_out/abtest.log
fi
