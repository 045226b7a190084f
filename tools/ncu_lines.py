"""Rank CUDA source lines of an ncu report by warp instructions executed.
usage: ncu_lines.py REPORT.ncu-rep [top]   (needs ncu on PATH, -lineinfo build)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, rows, tot_i, tot_t, tot_s = None, None, [], 0.0, 0.0, 0.0
for row in csv.reader(io.StringIO(txt)):
    if len(row) >= 2 and row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        ii, it, isamp = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), \
            hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not row or not row[0].isdigit() or len(row) < len(hdr) or row[2] != "-":
        continue
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    wi, ti, s = f(row[ii]), f(row[it]), f(row[isamp])
    tot_i += wi; tot_t += ti; tot_s += s
    rows.append((wi, ti, s, cur, int(row[0]), row[1].strip()[:90]))
rows.sort(key=lambda r: -r[0])
print("total warp instr %.4g  thread instr %.4g  (avg lanes %.1f)" % (tot_i, tot_t, tot_t / max(tot_i, 1)))
print("%6s %6s %5s %6s  %s" % ("%inst", "lanes", "%stl", "cum", "line"))
cum = 0.0
for wi, ti, s, fn, ln, src in rows[:top]:
    cum += wi
    print("%5.1f%% %6.1f %4.1f%% %5.1f%%  %s:%d  %s" % (100 * wi / tot_i, ti / max(wi, 1), 100 * s / max(tot_s, 1),
                                                     100 * cum / tot_i, fn, ln, src))
