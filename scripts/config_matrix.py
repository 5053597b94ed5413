"""Run the device search over a matrix of configs (strategy x branch mode x
roll/pitch range x batch size) on the C2 campus scene; prints one line each.
A robustness sweep (no reference: C2 searches take the reference minutes)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = B.DeviceScan(vm, s)
for strat in ("BFS", "DFS"):
    for mode in ("ROTO_TRANS", "TRANS_ONLY"):
        for rp in (0.02, 0.0873):
            for b in (10000, 500):
                if mode == "TRANS_ONLY" and rp != 0.02:
                    continue
                cfg = B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                                     roll_pitch_half_range=rp, strategy=B.Strategy[strat],
                                     branch_mode=B.BranchMode[mode], batch_size=b)
                t = time.time()
                r = B.search_scan(vm, ds, cfg)
                print(f"{strat} {mode} rp={rp} b={b}: best {r.best_score} matched {r.matched} "
                      f"evals {r.stats.nodes_generated} epochs {r.epochs} device {r.device_ms:.2f} ms "
                      f"wall {time.time() - t:.2f} s", flush=True)
