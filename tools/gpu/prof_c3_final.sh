# ncu --set full of one 2000-cycle TILED launch at C3 (after 6000 warm-up cycles) + per-line export + summary
cd $GRAFT_REPO_ROOT
tag=${1:-r02c}
bash tools/prof_lean.sh $tag 3 c3
ncu -i gpurun_out/prof_${tag}_c3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${tag}_src.csv 2>/dev/null
python tools/ncu_lines2.py gpurun_out/prof_${tag}_src.csv $((147*12*2000)) 80 > gpurun_out/prof_${tag}_lines.txt
ncu -i gpurun_out/prof_${tag}_c3.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
python tools/summarize_ncu.py gpurun_out/prof_${tag}_raw.csv gpurun_out/prof_${tag}_src.csv gpurun_out/prof_${tag}_summary.txt gpurun_out/traffic_${tag}.json "k_tiled C3 $tag (12 warps per CTA)" 2000 43264 > /dev/null 2>&1
rm -f gpurun_out/prof_${tag}_src.csv
head -40 gpurun_out/prof_${tag}_summary.txt
