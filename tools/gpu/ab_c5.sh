# A/B of PERSIST variants at C5 (tools/ab_c5.py) + a GPU test subset with the current library
cd $GRAFT_REPO_ROOT
lib_of() { if [ "$1" = cur ]; then echo $PWD/paper_1508_03235_b200/libnocsim.so; else echo $PWD/abl/$1; fi; }
for v in $1; do
  NOCSIM_LIB=$(lib_of $v) timeout 600 python tools/ab_c5.py 2>&1 | tail -1 | sed "s/^/$v /"
done | tee gpurun_out/ab_c5.txt
if [ -n "$2" ]; then
  NOCSIM_LIB=$(lib_of ${3:-cur}) timeout 1800 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/abtest.log 2>&1; tail -3 gpurun_out/abtest.log
fi
