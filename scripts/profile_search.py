"""Profiling driver: the bench workload (C2 campus) searched N times."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2310_10023_b200 as B
ap = argparse.ArgumentParser()
ap.add_argument("--searches", type=int, default=3)
ap.add_argument("--config", default="c2")
ap.add_argument("--layout", default="auto")
ap.add_argument("--k", type=int, default=0, help="override the scan size K")
ap.add_argument("--flush", action="store_true", help="write 256 MiB before every search (cold L2, as bench.py)")
a = ap.parse_args()
cfgd = dict(bench.CONFIGS[a.config])
if a.k:
    cfgd["K"] = a.k
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"], layout=B.Layout[a.layout.upper()])
ds = B.DeviceScan(vm, s)
cfg = bench.search_config(B, cfgd)
flush = None
if a.flush:
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(a.searches):
    if flush is not None:
        flush.fill_(1)
        torch.cuda.synchronize()
    r = B.search_scan(vm, ds, cfg)
    print(f"search {i}: best {r.best_score} evals {r.stats.nodes_generated} epochs {r.epochs} "
          f"device {r.device_ms:.3f} ms root {r.root_score_ms:.3f} epoch-score {r.epoch_score_ms:.3f} "
          f"init {r.stats.initial_nodes_ms:.3f} launches {r.kernel_launches} qpeak {r.queue_peak} per-level {list(r.evals_per_level[:8])}", flush=True)
