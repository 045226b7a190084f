# which library variants fail the streamed-script parity test; then A/B timings
cd $GRAFT_REPO_ROOT
lib_of() { if [ "$1" = cur ]; then echo $PWD/paper_1508_03235_b200/libnocsim.so; else echo $PWD/abl/$1; fi; }
for v in base.so cur; do
  for r in 1 2; do
    NOCSIM_LIB=$(lib_of $v) timeout 600 python -m pytest tests -m gpu -q -k "streamed_script" 2>&1 | tail -2 | sed "s/^/$v run$r /"
  done
done | tee gpurun_out/dbg_script.txt
for v in $1; do
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/ab_c3.py 3 2>&1 | sed "s/^/$v /"
  NOCSIM_LIB=$(lib_of $v) timeout 300 python tools/cycle_time.py 3 2>&1 | sed "s/^/$v /"
done | tee gpurun_out/ab.txt
