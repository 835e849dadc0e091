"""Per-role stall breakdown from an ncu source-page CSV (ncu -i X --page source --csv --print-source sass)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
isrc, iex = h.index('Source'), h.index('Instructions Executed')
reasons = [x for x in h if x.startswith('stall_') and '(Not Issued)' not in x]
by_count = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try:
        e = int(r[iex])
    except ValueError:
        continue
    for k in reasons:
        try:
            by_count[e][k] += int(r[h.index(k)])
        except ValueError:
            pass
key = int(sys.argv[2]) if len(sys.argv) > 2 else None
for e, c in sorted(by_count.items(), key=lambda x: -sum(x[1].values()))[:8]:
    if key and e != key:
        continue
    tot = sum(c.values())
    print(e, tot, [(k, v) for k, v in c.most_common(8)])
