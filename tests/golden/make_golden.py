"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
itself (oracle/_ref/libbnbloc_ref.so = the unmodified bnbloc headers behind a
C shim).  Inputs come from the reference's own gen_scene.  Run here, where
/root/reference exists:

    python tests/golden/make_golden.py [--skip-campus]

Outputs (small, committed):
  scenes.json            scene specs + seeds + digests of the generated clouds
  <case>_levels.json     per-level occupied-voxel counts and sha256 digests
  <case>_batch.npz       seeded node batches and their reference scores
  <case>_search.json     reference search() results (score, pose, Stats, trace)
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Reference, default_config  # noqa: E402

# scene cases: (name, spec overrides, seed, r, max_level, scan cut K or None)
CASES = {
    "small": dict(spec=dict(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4, min_box_side=2.5,
                            max_box_side=6.0, min_box_height=3.0, map_spacing=0.3,
                            scan_spacing=0.45, scan_range=14.0, min_scan_points=300),
                  seed=42, r=0.25, max_level=4, K=None, ct=0.01),
    "tiny": dict(spec=dict(size_x=8.0, size_y=8.0, size_z=4.0, num_boxes=2, min_box_side=1.5,
                           max_box_side=3.0, min_box_height=1.5, map_spacing=0.15,
                           scan_spacing=0.25, scan_range=9.0, min_scan_points=250),
                 seed=11, r=1.0, max_level=2, K=None, ct=0.01),
    # BASELINE configs[0] / SURVEY C1 room (CPU-runnable)
    "room": dict(spec=dict(size_x=20.0, size_y=20.0, size_z=4.0, num_boxes=8, min_box_side=1.0,
                           max_box_side=4.0, min_box_height=1.0, map_spacing=0.058,
                           scan_spacing=0.1, scan_range=10.0, min_scan_points=400),
                 seed=1, r=0.1, max_level=5, K=2000, ct=0.3, rp=0.0873),
    # BASELINE configs[1] / SURVEY C2 campus (the bench workload)
    "campus": dict(spec=dict(size_x=300.0, size_y=300.0, size_z=30.0, num_boxes=60,
                             min_box_side=6.0, max_box_side=30.0, min_box_height=8.0,
                             map_spacing=0.19, scan_spacing=0.3, scan_range=60.0,
                             min_scan_points=400),
                   seed=1, r=0.2, max_level=5, K=10000, ct=0.3, rp=0.02),
}

# search configurations checked per case: (label, overrides)
SEARCHES = {
    "small": [("bfs_roto_b10000", dict(strategy=1, branch_mode=1, batch_size=10000)),
              ("bfs_roto_b7", dict(strategy=1, branch_mode=1, batch_size=7)),
              ("dfs_roto_b500", dict(strategy=0, branch_mode=1, batch_size=500)),
              ("dfs_roto_b10000", dict(strategy=0, branch_mode=1, batch_size=10000)),
              ("bfs_trans_b10000", dict(strategy=1, branch_mode=0, batch_size=10000,
                                        roll_pitch_half_range=0.0)),
              ("dfs_trans_b7", dict(strategy=0, branch_mode=0, batch_size=7,
                                    roll_pitch_half_range=0.0)),
              ("bfs_roto_thr80", dict(strategy=1, branch_mode=1, batch_size=2000,
                                      score_threshold_fraction=0.8))],
    "tiny": [("bfs_trans", dict(strategy=1, branch_mode=0, roll_pitch_half_range=0.0,
                                score_threshold_fraction=0.9)),
             ("dfs_trans", dict(strategy=0, branch_mode=0, roll_pitch_half_range=0.0,
                                score_threshold_fraction=0.9)),
             ("bfs_roto", dict(strategy=1, branch_mode=1, roll_pitch_half_range=0.0,
                               score_threshold_fraction=0.9))],
    "room": [("bfs_roto_b10000", dict(strategy=1, branch_mode=1, batch_size=10000))],
    "campus": [("bfs_roto_b10000", dict(strategy=1, branch_mode=1, batch_size=10000))],
}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cut_scan(scan, k, seed):
    """Fisher-Yates prefix with the reference's splitmix64 Rng (restated in
    csrc/scene.cpp as bbs_cut_scan); pure-Python copy for the generator."""
    mask = (1 << 64) - 1
    state = seed & mask

    def next_u64():
        nonlocal state
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        return z ^ (z >> 31)

    n = scan.shape[0]
    idx = list(range(n))
    for i in range(k):
        span = n - 1 - i + 1
        j = i + next_u64() % span
        idx[i], idx[j] = idx[j], idx[i]
    return scan[idx[:k]].copy()


def search_cfg(case, overrides):
    kw = dict(min_resolution=case["r"], max_level=case["max_level"],
              roll_pitch_half_range=case.get("rp", 0.02), collect_trace=1)
    kw.update(overrides)
    return default_config(**kw)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-campus", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    ref = Reference()
    scenes = {}
    for name, case in CASES.items():
        if args.only and name != args.only:
            continue
        if name == "campus" and args.skip_campus:
            continue
        t0 = time.time()
        spec = ref.default_spec()
        for k, v in case["spec"].items():
            setattr(spec, k, v)
        m, s, gt = ref.gen_scene(spec, case["seed"])
        if case["K"] is not None:
            s = cut_scan(s, min(case["K"], s.shape[0]), 7)
        scenes[name] = dict(spec=case["spec"], seed=case["seed"], r=case["r"],
                            max_level=case["max_level"], K=case["K"], cut_seed=7,
                            map_points=int(m.shape[0]), map_digest=digest(m),
                            scan_points=int(s.shape[0]), scan_digest=digest(s), gt=list(gt))
        rmap = ref.map_build(m, case["r"], case["max_level"], case["ct"], 8 << 30)
        levels = []
        for lv in range(case["max_level"] + 1):
            occ = rmap.occupied(lv)
            levels.append(dict(level=lv, count=int(occ.shape[0]), digest=digest(occ)))
        with open(os.path.join(HERE, f"{name}_levels.json"), "w") as f:
            json.dump(levels, f, indent=1)
        # seeded node batches (search_test.cpp:121-129 pattern, all levels)
        cfg = search_cfg(case, {})
        d_max = ref.max_range(s)
        grid = ref.angular_grid(cfg, d_max)
        L = case["max_level"]
        rng = np.random.default_rng(1234)
        bb = rmap.bbox()
        n_nodes = 4000 if name != "campus" else 2000
        nodes = np.zeros((n_nodes, 8), np.int32)
        for i in range(n_nodes):
            lv = int(rng.integers(0, L + 1))
            cell = case["r"] * 2 ** lv
            nodes[i, 0] = rng.integers(int(np.floor(bb.min.x / cell)) - 1, int(np.ceil(bb.max.x / cell)) + 2)
            nodes[i, 1] = rng.integers(int(np.floor(bb.min.y / cell)) - 1, int(np.ceil(bb.max.y / cell)) + 2)
            nodes[i, 2] = rng.integers(int(np.floor(bb.min.z / cell)) - 1, int(np.ceil(bb.max.z / cell)) + 2)
            for a in range(3):
                g = grid[a * (L + 1) + lv]
                mi = 0 if g.segments == 0 else (g.segments - 1 if g.periodic else g.segments)
                nodes[i, 3 + a] = rng.integers(0, mi + 1)
            nodes[i, 6] = lv
            nodes[i, 7] = -1
        scored = rmap.batch_evaluate(s, cfg, nodes, d_max=d_max, workers=os.cpu_count())
        np.savez_compressed(os.path.join(HERE, f"{name}_batch.npz"), nodes=nodes,
                            scores=scored[:, 7].astype(np.int32))
        results = {}
        for label, ov in SEARCHES[name]:
            c = search_cfg(case, ov)
            c.workers = os.cpu_count()
            t = time.time()
            r, trace = rmap.search(s, c, trace_cap=1 << 16)
            results[label] = dict(
                overrides=ov, best_score=r.best_score, score_threshold=r.score_threshold,
                matched=bool(r.matched), best_pose=list(r.best_pose.as_tuple()),
                nodes_generated=r.stats.nodes_generated, nodes_pruned=r.stats.nodes_pruned,
                batches_flushed=r.stats.batches_flushed, trace=trace,
                ref_seconds=time.time() - t)
            print(name, label, r.best_score, r.stats.nodes_generated, f"{time.time() - t:.1f}s",
                  flush=True)
        with open(os.path.join(HERE, f"{name}_search.json"), "w") as f:
            json.dump(results, f, indent=1)
        print(name, f"done in {time.time() - t0:.1f}s", flush=True)
    path = os.path.join(HERE, "scenes.json")
    old = {}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f)
    old.update(scenes)
    with open(path, "w") as f:
        json.dump(old, f, indent=1)


if __name__ == "__main__":
    main()
