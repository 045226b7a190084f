# A/B of library variants under ab/ at C5 (PERSIST)
cd $GRAFT_REPO_ROOT
for v in $1; do
  if [ "$v" = cur ]; then lib=$PWD/paper_1508_03235_b200/libnocsim.so; else lib=$PWD/ab/$v; fi
  NOCSIM_LIB=$lib timeout 300 python tools/ab_c5.py 2>&1 | tail -1
done | tee gpurun_out/ab5.txt
