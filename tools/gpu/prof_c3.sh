# ncu --set full of one 2000-cycle TILED launch at C3 with source, plus the per-line export
set -x
bash tools/prof_lean.sh base 3 c3
ncu -i gpurun_out/prof_base_c3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_base_c3_src.csv 2>/dev/null
python tools/ncu_lines2.py gpurun_out/prof_base_c3_src.csv $((1470*2000)) 80 > gpurun_out/prof_base_c3_lines.txt
ncu -i gpurun_out/prof_base_c3.ncu-rep --page raw --csv > gpurun_out/prof_base_c3_raw.csv 2>/dev/null
ls -la gpurun_out
