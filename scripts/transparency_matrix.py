"""Exactness sweep of the fast paths: every config of a matrix (strategy x
branch mode x roll/pitch x batch size) searched with the defaults and with
the fast paths off (host-switched rounds, no direct runs, no flush cache, no
device root init, the rank-sort kernel before the merge, every merge CTA
ranking) and with the merge's two-phase tiled sort forced; score, pose,
Stats and trace must be identical."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2310_10023_b200 as B

OFF = {"BBS_SPEC_AUTO": "0", "BBS_DIRECT_RUNS": "0", "BBS_ROT_CACHE": "0", "BBS_ROOT_INIT": "host",
       "BBS_FUSE_SORT": "0", "BBS_MERGE_IDLE": "0"}
TILED = {"BBS_TILE_RANK_MIN": "256"}
KEYS = set(OFF) | set(TILED)
cfgd = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
if len(sys.argv) > 2:
    cfgd["K"] = int(sys.argv[2])  # scan size override (e.g. 70000: hash-built histograms)
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = B.DeviceScan(vm, s)
bad = 0
for strat in ("BFS", "DFS"):
    for mode in ("ROTO_TRANS", "TRANS_ONLY"):
        for rp in (0.02, 0.0873):
            for b in (10000, 500, 37):
                if mode == "TRANS_ONLY" and rp != 0.02:
                    continue
                cfg = B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                                     roll_pitch_half_range=rp, strategy=B.Strategy[strat],
                                     branch_mode=B.BranchMode[mode], batch_size=b, collect_trace=True)
                out = []
                for env in ({}, OFF, TILED):
                    for k in KEYS:
                        os.environ.pop(k, None)
                    os.environ.update(env)
                    r = B.search_scan(vm, ds, cfg)
                    out.append((r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated,
                                r.stats.nodes_pruned, r.stats.batches_flushed, tuple(r.best_score_trace)))
                ok = out[0] == out[1] == out[2]
                bad += not ok
                print(f"{strat} {mode} rp={rp} b={b}: {'same' if ok else 'DIFFERENT'} best {out[0][0]} "
                      f"evals {out[0][2]} flushed {out[0][4]}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
