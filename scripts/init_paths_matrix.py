"""Device vs host initial-queue build (BBS_ROOT_INIT) over the config matrix
of config_matrix.py on a bench scene: every search result must be identical
(best score, pose, Stats, incumbent trace).  Prints one line per config."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = B.DeviceScan(vm, s)
bad = 0
for strat in ("BFS", "DFS"):
    for rp in (0.02, 0.0873):
        for b in (10000, 500):
            for frac in (0.98, 0.95, 0.8):
                cfg = B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                                     roll_pitch_half_range=rp, strategy=B.Strategy[strat], batch_size=b,
                                     score_threshold_fraction=frac, collect_trace=True)
                out = {}
                for init in ("host", "device"):
                    os.environ["BBS_ROOT_INIT"] = init
                    r = B.search_scan(vm, ds, cfg)
                    out[init] = (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated,
                                 r.stats.nodes_pruned, r.stats.batches_flushed, tuple(r.best_score_trace))
                same = out["host"] == out["device"]
                bad += not same
                print(f"{strat} rp={rp} b={b} frac={frac}: best {out['device'][0]} evals {out['device'][2]} "
                      f"{'same' if same else 'DIFFERENT'}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
