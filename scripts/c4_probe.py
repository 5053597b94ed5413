"""Throughput probe: C2 map, n scans, bbs_search_scans at several concurrencies."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import harness as H  # noqa: E402  (synthetic inputs)
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS["c4"]
spec = H.SceneSpec.default(**cfgd["spec"])
m, _, _ = H.gen_scene(spec, cfgd["seed"])
scans, poses = H.gen_scans(spec, cfgd["seed"], 1000, int(os.environ.get("C4_N", "32")))
scans = [H.cut_scan(s, min(cfgd["K"], s.shape[0]), 7) for s in scans]
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = [B.DeviceScan(vm, s) for s in scans]
cfg = bench.search_config(B, cfgd)
shares = [int(x) for x in os.environ.get("C4_SHARES", "0").split(",")]
concs = [int(x) for x in os.environ.get("C4_CONCS", "1,2,4,8,16").split(",")]
print("host cores", os.cpu_count(), flush=True)
for share in shares:
    if share:
        os.environ["BBS_GRID_SHARE"] = str(share)
    else:
        os.environ.pop("BBS_GRID_SHARE", None)
    for conc in concs:
        B.search_scans(vm, ds, cfg, concurrency=conc)
        c0 = time.process_time()
        best = 1e9
        for _ in range(int(os.environ.get("C4_REPS", "3"))):
            t = time.perf_counter()
            res = B.search_scans(vm, ds, cfg, concurrency=conc)
            best = min(best, time.perf_counter() - t)
        if best == 1e9:
            continue
        dev = sum(r.device_ms for r in res)
        print(f"share {share or 'T'} concurrency {conc}: {len(ds) / best:.0f} scans/s, wall {1e3 * best:.1f} ms, "
              f"sum device {dev:.1f} ms, mean device {dev / len(ds):.2f} ms, cpu {1e3 * (time.process_time() - c0):.0f} ms", flush=True)
