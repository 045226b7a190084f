"""Per-source-line instruction counts and stall samples from an ncu
`--page source --csv --print-source cuda,sass` export.
usage: ncu_lines2.py SRC.csv warps_x_cycles [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
per = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None; h2 = None; res = collections.defaultdict(lambda: [0.0, 0.0, '']); ti = ts = 0
for row in rows:
    if len(row) == 2 and row[0] == "File Path":
        cur = row[1].split('/')[-1]; continue
    if row and row[0] == "Line No":
        h2 = row; ie = h2.index("Instructions Executed"); isa = h2.index("Warp Stall Sampling (All Samples)"); continue
    if h2 is None or len(row) < len(h2) or not row[0].isdigit():
        continue
    try:
        v = float(row[ie]); s = float(row[isa])
    except ValueError:
        continue
    ti += v; ts += s
    r = res[(cur, int(row[0]))]; r[0] += v; r[1] += s; r[2] = row[1][:84]
print("instructions per warp-cycle %.1f" % (ti / per))
for k, v in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
    print("%6.1f %5.1f%%  %s:%d  %s" % (v[0] / per, 100 * v[1] / ts, k[0], k[1], v[2]))
