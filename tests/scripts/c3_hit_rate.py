"""SURVEY d.1 check: local-L2 hit rate of the C3 workload over 20k cycles on the CPU oracle
(usage: python tools/c3_hit_rate.py PRIV_TAGS; 96 = the C3 workload).  Test infrastructure only."""
import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import Oracle
from paper_1508_03235_b200 import workloads as W
pt = int(sys.argv[1])
cfg = W.c3() if pt == 96 else W.c3(priv_tags=pt)
o = Oracle(cfg)
prev = None
t0 = time.time()
for k in range(10):
    o.run(2000)
    s = o.stats()[0]
    if prev:
        da = s['accesses'] - prev['accesses']; dh = s['l2_hits'] - prev['l2_hits']
        print(pt, 'cycles %d-%d accesses %d local hits %d (%.1f%%) misses %d evictions %d hops/node-cycle %.3f' % (
            s['cycle']-2000, s['cycle'], da, dh, 100.0*dh/max(da,1), s['l2_misses']-prev['l2_misses'],
            s['evictions']-prev['evictions'], (s['hops']-prev['hops'])/2000/43264), flush=True)
    prev = s
print('done', time.time()-t0)
