# A/B of library variants in abl/ at C3 / idle / small meshes, then C5 (PERSIST), then the GPU tests
# usage: bash tools/gpu/ab_all.sh "base.so cur v.so" "base.so cur" [pytest -k expr | all]
cd $GRAFT_REPO_ROOT
lib_of() { if [ "$1" = cur ]; then echo $PWD/paper_1508_03235_b200/libnocsim.so; else echo $PWD/abl/$1; fi; }
for v in $1; do
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/cycle_time.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
for v in $2; do
  NOCSIM_LIB=$(lib_of $v) timeout 600 python tools/ab_c5.py 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab_c5.txt
if [ "$3" = all ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/abtest.log 2>&1; tail -5 gpurun_out/abtest.log
elif [ -n "$3" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x -k "$3" > gpurun_out/abtest.log 2>&1; tail -5 gpurun_out/abtest.log
fi
