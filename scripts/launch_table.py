"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum CSV launch list.
Usage: launch_table.py launches.csv [--last N]  (N = keep only the last N launches)."""
import collections, csv, sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index('--last') + 1]) if '--last' in sys.argv else 0
rows, hdr = [], None
for r in csv.reader(open(path)):
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            v *= {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(d['Metric Unit'], 1.0)
            rows.append((d['Kernel Name'].split('(')[0].replace('bbs::<unnamed>::', '')[:58], v))
if last:
    rows = rows[-last:]
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in rows:
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v for _, v in rows)
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:58s} n={n:5d} total={v:9.1f} us avg={v / n:8.2f} us {100 * v / tot:5.1f}%")
print(f"launches {len(rows)} total {tot:.1f} us")
