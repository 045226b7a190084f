# repeat the streamed-script parity tests (PERSIST) to measure a flaky failure; then A/B timings
cd $GRAFT_REPO_ROOT
lib_of() { if [ "$1" = cur ]; then echo $PWD/paper_1508_03235_b200/libnocsim.so; else echo $PWD/abl/$1; fi; }
for v in $1; do
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/cycle_time.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
for v in $2; do
  for r in $(seq 1 ${3:-10}); do
    NOCSIM_LIB=$(lib_of $v) timeout 300 python -m pytest tests -m gpu -q -k "streamed_script_gpu and 1-2" 2>&1 | tail -1 | sed "s/^/$v run$r /"
  done
done | tee gpurun_out/flaky.txt
