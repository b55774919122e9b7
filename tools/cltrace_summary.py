"""Summarise RAMA_CLEANUP_STATS=2 per-round cleanup traces (last solve in the log)."""
import collections
import re
import sys

pat = re.compile(r'\[rama\] cl launch (\d+) round (\d+) np (\d+) pairs (\d+) nt (\d+) asum (\d+) \w+ (\d+) dt_us ([\d.]+)')
for f in sys.argv[1:]:
    solves, cur = [], []
    for line in open(f):
        m = pat.match(line)
        if m:
            r = [float(x) for x in m.groups()]
            if r[1] == 0 and cur:
                solves.append(cur)
                cur = []
            cur.append(r)
    if cur:
        solves.append(cur)
    rows = solves[-1]
    print(f, len(rows), 'rounds, sum dt %.2f ms' % (sum(r[7] for r in rows) / 1e3))
    for r in rows[:6]:
        print('  np %d pairs %d nt %d asum %d rrep %d dt %.1f us' % tuple(r[2:8]))
    b = collections.defaultdict(lambda: [0, 0.0, 0, 0])
    for r in rows:
        k = int(r[2]).bit_length()
        b[k][0] += 1
        b[k][1] += r[7]
        b[k][2] += r[4]
        b[k][3] += r[5]
    for k in sorted(b):
        n = b[k][0]
        print('  np<2^%-2d %4d rounds %7.2f ms (%.1f us/round) avg nt %d avg asum %d' % (k, n, b[k][1] / 1e3, b[k][1] / n, b[k][2] // n, b[k][3] // n))
