"""Per-kernel DRAM traffic and duration from an ncu CSV launch list taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
Usage: traffic.py launches.csv [--last N] [--json out.json --config c2]
                  [--sol kernel=report.ncu-rep ...]
Groups the bench's roofline kernels, prints bytes per launch, and (--json)
writes per-kernel and per-group entries; --sol adds the speed-of-light
percentages of a kernel from a `ncu --set full` report."""
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


# the search's own kernels (map build and CUB launches excluded from shares)
SEARCH_KERNELS = {"root_hist_kernel", "root_colpad_kernel", "root_col_kernel", "score_box_kernel",
                  "root_select_kernel", "root_pass_kernel", "stage_window_kernel",
                  "cache_prebuild_list_kernel", "cache_build_kernel", "cache_probe_kernel",
                  "score_cube8_kernel", "frontier_kernel", "branch_kernel", "survivors_kernel",
                  "rank_sort_kernel", "merge_kernel", "soa_kernel", "score_runs_kernel",
                  "frontier_auto_kernel", "frontier_spec_kernel", "survivors_auto_kernel",
                  "survivors_spec_kernel", "rank_sort_auto_kernel", "merge_auto_kernel", "pad_keys_kernel",
                  "cache_prebuild_kernel", "scatter_own_kernel"}


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


def sol(rep):
    """Speed-of-light numbers of the first kernel in an ncu --set full report."""
    import io
    import subprocess
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    want = {"Compute (SM) Throughput": "sm_throughput_pct", "Memory Throughput": "memory_throughput_pct",
            "L1/TEX Cache Throughput": "l1tex_throughput_pct", "L2 Cache Throughput": "l2_throughput_pct",
            "Issued Ipc Active": "ipc_active", "Achieved Occupancy": "achieved_occupancy_pct",
            "Duration": "ncu_duration", "Registers Per Thread": "registers"}
    out = {"source": rep}
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = want.get(d.get("Metric Name"))
        if k and k not in out and (d.get("Metric Unit") != "Gbyte/s"):
            try:
                out[k] = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                pass
    return out


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
        search_us = sum(v[1] for k, v in agg.items() if k in SEARCH_KERNELS)
        for name, (n, us, by) in agg.items():
            if n == 0:
                continue
            out[name] = {"dram_bytes_per_launch": by / n, "us_per_launch": us / n, "launches": n}
            if name in SEARCH_KERNELS:
                out[name]["share_of_search_device_time"] = us / max(search_us, 1e-9)
        for spec in [a for i, a in enumerate(sys.argv) if i and sys.argv[i - 1] == "--sol"]:
            kname, rep = spec.split("=", 1)
            out.setdefault(kname, {}).update(sol(rep))
        allj[cfg] = out
        json.dump(allj, open(js, "w"), indent=1)
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
