"""Extra reference searches on the C2 campus workload (DFS, small batch,
+-5 deg roll/pitch), appended to campus_search.json.  Runs the UNMODIFIED
reference (oracle/_ref) — several CPU minutes each; the device replays them in
tests/test_search_gpu.py::test_search_matches_reference_golden (every label)."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from make_golden import CASES, cut_scan, search_cfg  # noqa: E402
from pyoracle import Reference  # noqa: E402

EXTRA = [("dfs_roto_b10000", dict(strategy=0, branch_mode=1, batch_size=10000)),
         ("bfs_roto_b1000", dict(strategy=1, branch_mode=1, batch_size=1000)),
         ("bfs_roto_rp5deg", dict(strategy=1, branch_mode=1, batch_size=10000, roll_pitch_half_range=0.0873))]


def main():
    case = CASES["campus"]
    ref = Reference()
    spec = ref.default_spec()
    for k, v in case["spec"].items():
        setattr(spec, k, v)
    m, s, _ = ref.gen_scene(spec, case["seed"])
    s = cut_scan(s, min(case["K"], s.shape[0]), 7)
    rmap = ref.map_build(m, case["r"], case["max_level"], case["ct"], 8 << 30)
    path = os.path.join(HERE, "campus_search.json")
    with open(path) as f:
        results = json.load(f)
    for label, ov in EXTRA:
        if label in results:
            continue
        c = search_cfg(case, ov)
        c.workers = os.cpu_count()
        t = time.time()
        r, trace = rmap.search(s, c, trace_cap=1 << 16)
        results[label] = dict(
            overrides=ov, best_score=r.best_score, score_threshold=r.score_threshold,
            matched=bool(r.matched), best_pose=list(r.best_pose.as_tuple()),
            nodes_generated=r.stats.nodes_generated, nodes_pruned=r.stats.nodes_pruned,
            batches_flushed=r.stats.batches_flushed, trace=trace, ref_seconds=time.time() - t)
        print(label, r.best_score, r.stats.nodes_generated, f"{time.time() - t:.1f}s", flush=True)
        with open(path, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
