"""Summarise an .ncu-rep: headline metrics, stall reasons, top SASS lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


r = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = r[0]
keys = ['Duration', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit', 'L2 Hit', 'Registers',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Issued Ipc Active', 'No Eligible',
        'Warp Cycles Per Issued', 'Grid Size', 'Block Size', 'Issued Instructions',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput']
for x in r[1:]:
    d = dict(zip(h, x))
    if any(k in d.get('Metric Name', '') for k in keys):
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
r = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(r[0], r[2]))
st = [(k, float(d[k] or 0)) for k in r[0] if 'smsp__average_warps_issue_stalled' in k and k.endswith('.ratio')]
print('stalls:', ', '.join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
    print(k, d.get(k))
r = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:] if len(x) >= len(h) - 1]
S = lambda x: int(x['Warp Stall Sampling (All Samples)'] or 0)
tot = sum(S(x) for x in rows)
print('samples', tot, 'sass lines', len(rows))
for i in sorted(sorted(range(len(rows)), key=lambda i: -S(rows[i]))[:top]):
    print(f"{i:5d} {S(rows[i]):6d} {rows[i]['Instructions Executed']:>9s}  {rows[i]['Source'].strip()[:70]}")
