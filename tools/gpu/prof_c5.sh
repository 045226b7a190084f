# ncu --set full of one 200-cycle PERSIST launch at C5 (1024x1024 LSPD) + per-line export and summary
cd $GRAFT_REPO_ROOT
tag=${1:-c5}
ncu --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_${tag} -f \
  python tools/prof_run.py --workload c5 --engine 2 --warm 3000 --cycles 200 --launches 2 > gpurun_out/prof_${tag}.log 2>&1
ncu -i gpurun_out/prof_${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${tag}_src.csv 2>/dev/null
python tools/ncu_lines2.py gpurun_out/prof_${tag}_src.csv $((1048576*200/32)) 100 > gpurun_out/prof_${tag}_lines.txt
ncu -i gpurun_out/prof_${tag}.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
python tools/summarize_ncu.py gpurun_out/prof_${tag}_raw.csv gpurun_out/prof_${tag}_src.csv gpurun_out/prof_${tag}_summary.txt gpurun_out/traffic_${tag}.json "k_persist C5 $tag" 200 1048576 > /dev/null 2>&1
rm -f gpurun_out/prof_${tag}_src.csv
