import os, sys, time
sys.path.insert(0, '.')
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS["c2"]
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = B.DeviceScan(vm, s)
for b in (10000, 500):
    cfg = B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"], branch_mode=B.BranchMode.TRANS_ONLY, batch_size=b)
    for rep in range(2):
        r = B.search_scan(vm, ds, cfg)
    print(os.environ.get("BBS_ROT_CACHE"), b, r.best_score, r.stats.nodes_generated, r.epochs, f"{r.device_ms:.1f} ms root {r.root_score_ms:.1f} init {r.stats.initial_nodes_ms:.1f} epoch-score {r.epoch_score_ms:.1f}", flush=True)
