"""Dev check: small-scene parity of the device path against the reference
(oracle/_ref) and the C restatement.  Prints one line per check."""
import sys, time, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'oracle'))
import harness as H  # noqa: E402  (synthetic inputs)
import paper_2310_10023_b200 as B
from pyoracle import Reference, Restated, default_config

ref = Reference(); orc = Restated()
spec = H.SceneSpec.default(size_x=24, size_y=24, size_z=10, num_boxes=4, min_box_side=2.5,
                           max_box_side=6.0, min_box_height=3.0, map_spacing=0.3,
                           scan_spacing=0.45, scan_range=14.0, min_scan_points=300)
m, s, gt = H.gen_scene(spec, 42)
r, L = 0.25, 4
for layout in (B.Layout.BITMAP, B.Layout.HASH):
    t = time.time(); dm = B.MultiResVoxelMap.build(m, r, L, layout=layout); bt = time.time() - t
    om = orc.map_build(m, r, L)
    ok = all(np.array_equal(dm.level(l).occupied_voxels(), om.occupied(l)) for l in range(L + 1))
    print('map', layout.name, 'sets equal', ok, 'build_s %.3f' % bt, 'dev_ms %.2f' % dm.build_ms(),
          [dm.level(l).layout().name for l in range(L + 1)], flush=True)
    rm = ref.map_build(m, r, L, 0.3)
    cfg = B.SearchConfig(min_resolution=r, max_level=L, roll_pitch_half_range=0.02)
    dmax = B.max_range(s)
    grids = B.AngularGrid(cfg, dmax)
    rng = np.random.default_rng(0)
    nodes = []
    for i in range(20000):
        l = int(rng.integers(0, L + 1))
        nodes.append([int(rng.integers(-4, 100 >> l)), int(rng.integers(-4, 100 >> l)),
                      int(rng.integers(-2, 40 >> l)),
                      int(rng.integers(0, grids.axis(0, l).max_index() + 1)),
                      int(rng.integers(0, grids.axis(1, l).max_index() + 1)),
                      int(rng.integers(0, grids.axis(2, l).max_index() + 1)), l, -1])
    nodes = np.array(nodes, np.int32)
    t = time.time(); got = B.batch_evaluate(nodes, dm, s, grids); gt_ = time.time() - t
    want = rm.batch_evaluate(s, cfg.to_c(), nodes, workers=8)
    print('batch_evaluate', layout.name, 'equal', np.array_equal(got[:, 7], want[:, 7]),
          'mismatches', int((got[:, 7] != want[:, 7]).sum()), 'gpu_s %.3f' % gt_, flush=True)
    for mode in (B.BranchMode.ROTO_TRANS, B.BranchMode.TRANS_ONLY):
        for strat in (B.Strategy.BFS, B.Strategy.DFS):
            for b in (7, 500, 10000):
                c = B.SearchConfig(min_resolution=r, max_level=L, roll_pitch_half_range=0.0 if mode == 0 else 0.02,
                                   branch_mode=mode, strategy=strat, batch_size=b, collect_trace=True)
                t = time.time(); g = B.search(dm, s, c); gs = time.time() - t
                w, wt = rm.search(s, c.to_c())
                same = (g.best_score == w.best_score and g.matched == bool(w.matched) and
                        g.best_pose.as_tuple() == w.best_pose.as_tuple() and
                        (g.stats.nodes_generated, g.stats.nodes_pruned, g.stats.batches_flushed) ==
                        (w.stats.nodes_generated, w.stats.nodes_pruned, w.stats.batches_flushed) and
                        g.best_score_trace == wt)
                print('search', layout.name, mode.name, strat.name, 'b', b, 'SAME' if same else 'DIFF',
                      g.best_score, w.best_score, (g.stats.nodes_generated, g.stats.nodes_pruned, g.stats.batches_flushed),
                      (w.stats.nodes_generated, w.stats.nodes_pruned, w.stats.batches_flushed),
                      'dev_ms %.2f wall_s %.3f' % (g.device_ms, gs), flush=True)
