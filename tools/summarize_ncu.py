"""Summarise an ncu --set full report (raw + source CSV exports) into profiles/.
usage: summarize_ncu.py RAW.csv SRC.csv OUT.txt TRAFFIC.json "title" cycles nodes"""
import collections
import csv
import json
import sys

raw, src, out, traffic, title, cycles, nodes = sys.argv[1:8]
cycles, nodes = int(cycles), int(nodes)
r = list(csv.reader(open(raw)))
hdr, units, vals = r[0], r[1], r[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
lines = ["# " + title]
keys = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__cycles_elapsed.avg.per_second', 'sm__inst_executed.sum.per_cycle_active',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__average_warp_latency_per_inst_issued.ratio', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed']
for k in keys:
    if k in d:
        lines.append("%-60s %s %s" % (k, d[k], u[k]))


def tob(k):
    v = float(d[k].replace(',', ''))
    return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u[k], 1)


dram = tob('dram__bytes_read.sum') + tob('dram__bytes_write.sum')
lts = float(d['lts__t_sectors.sum'].replace(',', '')) * 32
lines.append("%-60s %.3f" % ("DRAM bytes per node-cycle", dram / cycles / nodes))
lines.append("%-60s %.3f" % ("L2 (lts) bytes per node-cycle", lts / cycles / nodes))
stalls = sorted(((h.split('stalled_')[1], float(d[h])) for h in hdr
                 if h.startswith('smsp__pcsamp_warps_issue_stalled_') and 'not_issued' not in h and d[h]),
                key=lambda x: -x[1])
tot = sum(v for _, v in stalls)
lines += ["", "# warp stall sampling (all samples)"]
lines += ["%-30s %6.1f%%" % (k, 100 * v / tot) for k, v in stalls[:12]]
rows = list(csv.reader(open(src)))
cur = None; h2 = None; res = collections.defaultdict(lambda: [0.0, 0.0, '']); ti = ts = 0


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for row in rows:
    if len(row) == 2 and row[0] == "File Path":
        cur = row[1].split('/')[-1]; continue
    if row and row[0] == "Line No":
        h2 = row; ie = h2.index("Instructions Executed"); isa = h2.index("Warp Stall Sampling (All Samples)"); continue
    if h2 is None or len(row) < len(h2) or not row[0].isdigit():
        continue
    v, s = fl(row[ie]), fl(row[isa]); ti += v; ts += s
    res[(cur, int(row[0]))][0] += v; res[(cur, int(row[0]))][1] += s; res[(cur, int(row[0]))][2] = row[1][:80]
lines += ["", "# top source lines by stall samples (% stall, % instructions executed)"]
for k, v in sorted(res.items(), key=lambda x: -x[1][1])[:20]:
    lines.append("%5.1f%% stall %5.1f%% instr  %s:%d  %s" % (100 * v[1] / ts, 100 * v[0] / ti, k[0], k[1], v[2]))
open(out, "w").write("\n".join(lines) + "\n")
inst = float(d['smsp__inst_executed.sum'].replace(',', '')) if 'smsp__inst_executed.sum' in d else 0.0
l2hit = float(d['lts__t_sector_hit_rate.pct'].replace(',', '')) if 'lts__t_sector_hit_rate.pct' in d else None
json.dump({"kernel": title, "dram_bytes_per_launch": dram, "lts_bytes_per_launch": lts, "cycles_per_launch": cycles,
           "nodes": nodes, "dram_bytes_per_node_cycle": dram / cycles / nodes,
           "lts_bytes_per_node_cycle": lts / cycles / nodes,
           "warp_inst_per_node_cycle": inst / cycles / nodes, "l2_hit_rate_pct": l2hit,
           "summary": out}, open(traffic, "w"), indent=1)
print(open(out).read())
