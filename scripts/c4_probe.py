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
scans, poses = H.gen_scans(spec, cfgd["seed"], 1000, 32)
scans = [H.cut_scan(s, min(cfgd["K"], s.shape[0]), 7) for s in scans]
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = [B.DeviceScan(vm, s) for s in scans]
cfg = bench.search_config(B, cfgd)
for conc in (1, 2, 4, 8, 16):
    B.search_scans(vm, ds, cfg, concurrency=conc)
    t = time.perf_counter()
    res = B.search_scans(vm, ds, cfg, concurrency=conc)
    dt = time.perf_counter() - t
    dev = sum(r.device_ms for r in res)
    print(f"concurrency {conc}: {len(ds) / dt:.0f} scans/s, wall {1e3 * dt:.1f} ms, sum device {dev:.1f} ms, "
          f"mean device {dev / len(ds):.2f} ms", flush=True)
