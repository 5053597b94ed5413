"""Per-kernel table of the last search in an ncu launch list (starts at the last root_hist_kernel)."""
import collections, csv, sys
rows, hdr = [], None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        rows.append((d['Kernel Name'].split('(')[0].replace('bbs::<unnamed>::', '')[:50],
                     float(d['Metric Value'].replace(',', '')) / 1e3))
idx = [i for i, (n, _) in enumerate(rows) if n.startswith('root_hist') or n.startswith('score_box')]
rows = rows[idx[-1]:] if idx else rows
if '--seq' in sys.argv:
    t = 0
    for n, v in rows:
        t += v
        print(f"{n:50s} {v:8.1f} {t:8.1f}")
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in rows:
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v for _, v in rows)
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} n={n:5d} total={v:9.1f} us avg={v / n:7.2f} us {100 * v / tot:5.1f}%")
print(f"launches {len(rows)} total {tot:.1f} us")
