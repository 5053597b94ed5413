"""Per-kernel DRAM traffic and duration from an ncu CSV launch list taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
Usage: traffic.py launches.csv [--last N] [--json out.json --config c2]
Groups the bench's roofline kernels and prints bytes per launch."""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
        "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
GROUPS = {
    "root": ("root_hist_kernel", "root_colpad_kernel", "root_col_kernel"),
    "flush": ("cache_probe_kernel", "score_cube8_kernel", "cache_build_kernel"),
}


def load(path, last=0):
    launches = collections.OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = (d["ID"], d["Kernel Name"].split("(")[0].split("::")[-1].replace("void ", "").split("<")[0])
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        launches.setdefault(k, {})[d["Metric Name"]] = v
    items = list(launches.items())
    return items[-last:] if last else items


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
    items = load(path, last)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in items:
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    for name, (n, us, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:40s} n={n:5d} us/launch={us / n:9.2f} dram MB/launch={by / n / 1e6:9.3f}")
    if "--json" in sys.argv:
        out = {}
        for g, names in GROUPS.items():
            n = max(agg[k][0] for k in names)
            by = sum(agg[k][2] for k in names)
            out[g] = {"dram_bytes_per_launch": by / max(n, 1), "launches": n,
                      "kernels": [k for k in names if agg[k][0]]}
        js = sys.argv[sys.argv.index("--json") + 1]
        cfg = sys.argv[sys.argv.index("--config") + 1]
        try:
            allj = json.load(open(js))
        except (OSError, ValueError):
            allj = {}
        allj[cfg] = out
        json.dump(allj, open(js, "w"), indent=1)
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
