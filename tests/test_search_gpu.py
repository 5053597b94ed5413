"""Device search (K5/K6 + epoch loop) parity: best score, best pose, the
Stats counters (nodes_generated / nodes_pruned / batches_flushed) and the
incumbent trace equal the reference's search() exactly — the device replays
the reference's pop/flush schedule — on the golden cases up to the full C2
campus workload, plus the behavioural tests of proj/tests/search_test.cpp."""
import math

import numpy as np
import pytest
import harness as H  # noqa: E402  (synthetic inputs)

from conftest import golden_json, load_case

pytestmark = pytest.mark.gpu


def make_cfg(B, sc, name, ov):
    kw = dict(min_resolution=sc["r"], max_level=sc["max_level"],
              roll_pitch_half_range=0.0873 if name == "room" else 0.02, collect_trace=True)
    kw.update(ov)
    return B.SearchConfig(**kw)


def assert_same(res, want, label):
    assert res.best_score == want["best_score"], label
    assert res.score_threshold == want["score_threshold"], label
    assert res.matched == want["matched"], label
    assert list(res.best_pose.as_tuple()) == want["best_pose"], label
    assert (res.stats.nodes_generated, res.stats.nodes_pruned, res.stats.batches_flushed) == \
        (want["nodes_generated"], want["nodes_pruned"], want["batches_flushed"]), label
    assert res.best_score_trace == want["trace"], label


@pytest.mark.parametrize("layout", ["AUTO", "HASH"])
@pytest.mark.parametrize("name", ["tiny", "small", "room", "campus"])
def test_search_matches_reference_golden(B, golden_scenes, name, layout):
    if name not in golden_scenes:
        pytest.skip("golden case not generated")
    m, s, _, sc = load_case(B, golden_scenes, name)
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"], layout=B.Layout[layout])
    for label, want in golden_json(f"{name}_search.json").items():
        res = B.search(vm, s, make_cfg(B, sc, name, want["overrides"]))
        assert_same(res, want, f"{name}/{label}/{layout}")


@pytest.mark.parametrize("init", ["device", "host"])
@pytest.mark.parametrize("name", ["small", "room", "campus"])
def test_root_queue_init_paths(B, golden_scenes, name, init, monkeypatch):
    """Both builds of the initial queue (root survivors -> sorted queue) match
    the reference: the device path (root_select + root_pass kernels, no host
    round trip) and the host path (CUB select + sort after a sync); the
    default picks one per search (DESIGN §3 K5/K6)."""
    monkeypatch.setenv("BBS_ROOT_INIT", init)
    m, s, _, sc = load_case(B, golden_scenes, name)
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    for label, want in golden_json(f"{name}_search.json").items():
        res = B.search(vm, s, make_cfg(B, sc, name, want["overrides"]))
        assert_same(res, want, f"{name}/{label}/{init}")


def test_device_scan_equals_host_scan(B, golden_scenes):
    m, s, _, sc = load_case(B, golden_scenes, "small")
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    cfg = make_cfg(B, sc, "small", dict(batch_size=500))
    a = B.search(vm, s, cfg)
    ds = B.DeviceScan(vm, s)
    b = B.search_scan(vm, ds, cfg)
    c = B.search_scan(vm, ds, cfg)  # workspace reuse
    for r in (b, c):
        assert (r.best_score, r.best_pose, r.stats.nodes_generated, r.best_score_trace) == \
            (a.best_score, a.best_pose, a.stats.nodes_generated, a.best_score_trace)


# ---- search_test.cpp behaviours ---------------------------------------------
def mini_scene(B, seed, gt):
    """search_test.cpp:16-58 box world, rendered through gen_scene-like
    sampling in numpy (independent map and scan samples)."""
    rng = np.random.default_rng(seed)

    def rect(o, du, dv, nu, nv):
        u, v = np.meshgrid(np.arange(nu + 1) / nu, np.arange(nv + 1) / nv, indexing="ij")
        return (np.array(o)[None] + u.reshape(-1, 1) * np.array(du)[None] +
                v.reshape(-1, 1) * np.array(dv)[None])

    def world(d):
        return np.concatenate([rect((0, 0, 0), (16, 0, 0), (0, 16, 0), 4 * d, 4 * d),
                               rect((2, 3, 0), (6, 0, 0), (0, 0, 5), 2 * d, d),
                               rect((11, 5, 0), (0, 7, 0), (0, 0, 7), 2 * d, 2 * d),
                               rect((4, 12, 0), (5, 2, 0), (0, 0, 3), 2 * d, d)])

    m = world(12)
    w = world(9) + rng.uniform(-1e-6, 1e-6, size=(1, 3))
    R, t = B.pose_to_transform(gt)
    R = np.array(R).reshape(3, 3)
    q = (w - np.array(t)) @ R  # inverse rigid transform
    q = q[np.linalg.norm(q, axis=1) <= 20.0]
    return m, q


def small_cfg(B, mode, **kw):
    c = dict(min_resolution=1.0, max_level=2, roll_pitch_half_range=0.0, branch_mode=mode,
             strategy=B.Strategy.BFS, score_threshold_fraction=0.9)
    c.update(kw)
    return B.SearchConfig(**c)


def test_self_localization_recovers_identity(B):
    m, s = mini_scene(B, 3, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    r = B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY))
    assert r.matched and r.best_score >= r.score_threshold
    assert math.dist(r.best_pose.as_tuple()[:3], (0, 0, 0)) <= math.sqrt(3.0)


def test_recovers_offset_pose(B):
    gt = B.Pose6(5.0, 7.0, 0.5, 0, 0, 2.2)
    m, s = mini_scene(B, 4, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    r = B.search(vm, s, small_cfg(B, B.BranchMode.ROTO_TRANS))
    assert r.matched
    assert math.dist(r.best_pose.as_tuple()[:3], gt.as_tuple()[:3]) < 2.0


def test_disjoint_scan_does_not_match(B):
    m, _ = mini_scene(B, 5, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    rng = np.random.default_rng(99)
    far = np.stack([rng.uniform(-3, 3, 200), rng.uniform(-3, 3, 200), rng.uniform(11, 14, 200)], 1)
    r = B.search(vm, far, small_cfg(B, B.BranchMode.TRANS_ONLY))
    assert not r.matched and r.best_score == r.score_threshold


def test_transonly_matches_exhaustive_oracle_both_strategies(B, orc):
    # search_test.cpp:178-205 with the C restatement's exhaustive leaf oracle
    for seed in range(10, 14):
        prng = np.random.default_rng(seed * 131)
        gt = B.Pose6(prng.uniform(2, 12), prng.uniform(2, 12), prng.uniform(0, 1), 0, 0,
                     prng.uniform(0, 2 * math.pi))
        m, s = mini_scene(B, seed, gt)
        vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
        om = orc.map_build(m, 1.0, 2)
        y = B.normalize_angle(gt.yaw) if hasattr(B, "normalize_angle") else gt.yaw
        cfg = small_cfg(B, B.BranchMode.TRANS_ONLY, yaw_min=y - 0.3, yaw_max=y + 0.3)
        best, _, _ = om.exhaustive(s, cfg.to_c())
        for st in (B.Strategy.DFS, B.Strategy.BFS):
            cfg.strategy = st
            r = B.search(vm, s, cfg)
            if best >= r.score_threshold:
                assert r.matched and r.best_score == best, (seed, st)
            else:
                assert not r.matched


def test_batch_size_does_not_change_transonly_best(B):
    gt = B.Pose6(4.0, 3.0, 0.2, 0, 0, 1.1)
    m, s = mini_scene(B, 21, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    scores = set()
    for b in (1, 7, 10000):
        r = B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, yaw_min=gt.yaw - 0.3,
                                      yaw_max=gt.yaw + 0.3, batch_size=b))
        assert r.matched
        scores.add(r.best_score)
    assert len(scores) == 1


def test_incumbent_trace_is_monotone(B):
    gt = B.Pose6(6.0, 5.0, 0.3, 0, 0, 0.4)
    m, s = mini_scene(B, 22, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    r = B.search(vm, s, small_cfg(B, B.BranchMode.ROTO_TRANS, collect_trace=True))
    assert r.matched and r.best_score_trace
    assert r.best_score_trace == sorted(r.best_score_trace)
    assert r.best_score_trace[0] >= r.score_threshold and r.best_score_trace[-1] == r.best_score


def test_stats_are_populated(B):
    m, s = mini_scene(B, 23, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    r = B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY))
    assert r.stats.nodes_generated > 0 and r.stats.batches_flushed > 0
    assert r.stats.initial_nodes_ms >= 0 and r.stats.find_best_score_ms >= 0
    assert r.stats.pop_remaining_queue_ms >= 0 and r.scan_points == s.shape[0]
    assert r.kernel_launches > 0 and r.lookups == r.stats.nodes_generated * s.shape[0]


def test_validation_errors(B):
    # search_test.cpp:256-273, same exception types
    m, s = mini_scene(B, 24, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    cfg = small_cfg(B, B.BranchMode.TRANS_ONLY)
    with pytest.raises(B.DegenerateScanError):
        B.search(vm, np.zeros((0, 3)), cfg)
    with pytest.raises(B.DegenerateScanError):
        B.search(vm, np.zeros((2, 3)), cfg)
    with pytest.raises(B.ConfigError, match="config r does not match"):
        B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, min_resolution=0.5))
    with pytest.raises(B.ConfigError, match="max_level must be in"):
        B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, max_level=5))
    with pytest.raises(B.ConfigError, match="batch_size"):
        B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, batch_size=0))
    with pytest.raises(B.ConfigError, match="score_threshold_fraction"):
        B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, score_threshold_fraction=1.5))


def test_empty_search_space(B):
    m, s = mini_scene(B, 25, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    cfg = small_cfg(B, B.BranchMode.TRANS_ONLY, translation_range=((5, 5, 5), (-5, 5, 5)))
    with pytest.raises(B.EmptySearchSpaceError):
        B.search(vm, s, cfg)


def test_yaw_result_is_normalized(B):
    gt = B.Pose6(5, 5, 0.3, 0, 0, 1.3)
    m, s = mini_scene(B, 30, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    r1 = B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY))
    r2 = B.search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY))
    assert r1.matched and r1.best_score == r2.best_score and r1.best_pose.yaw == r2.best_pose.yaw
    assert 0.0 <= r1.best_pose.yaw < 2 * math.pi


def test_localize_scan_matches_reference(B, ref):
    spec = H.SceneSpec.default(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4,
                               min_box_side=2.5, max_box_side=6.0, min_box_height=3.0,
                               map_spacing=0.3, scan_spacing=0.2, scan_range=14.0,
                               min_scan_points=300)
    m, raw, _ = H.gen_scene(spec, 9)
    vm = B.MultiResVoxelMap.build(m, 0.5, 3)
    rm = ref.map_build(m, 0.5, 3, 0.05)
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, batch_size=1000)
    for target in (0, 1000):
        got = B.localize_scan(vm, raw, cfg, target)
        want = rm.localize_scan(raw, cfg.to_c(), target)
        assert got.best_score == want.best_score and got.scan_points == want.scan_points
        assert got.best_pose.as_tuple() == want.best_pose.as_tuple()
        assert got.stats.nodes_generated == want.stats.nodes_generated
        assert got.stats.set_source_ms >= 0


def test_rotation_cache_is_transparent(B, golden_scenes, monkeypatch):
    """The flush histogram cache (epoch_cache.cu) and its fallbacks (uncached
    levels, rotations whose offsets do not de-duplicate) must not change any
    result: campus (K = 10000 >= the cache threshold) with +-5 deg roll/pitch,
    so level 0 has > 2^20 rotations and stays uncached while coarser levels
    are cached."""
    m, s, _, sc = load_case(B, golden_scenes, "campus")
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    ds = B.DeviceScan(vm, s)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("BBS_ROT_CACHE", flag)
        for strat in ("BFS", "DFS"):
            cfg = B.SearchConfig(min_resolution=sc["r"], max_level=sc["max_level"],
                                 roll_pitch_half_range=0.0873, collect_trace=True,
                                 strategy=B.Strategy[strat])
            r = B.search_scan(vm, ds, cfg)
            out[(flag, strat)] = (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated,
                                  r.stats.nodes_pruned, r.stats.batches_flushed, r.best_score_trace,
                                  tuple(r.evals_per_level))
    for strat in ("BFS", "DFS"):
        assert out[("1", strat)] == out[("0", strat)], strat
    assert out[("1", "BFS")][6][0] > 0  # the search reached the uncached level 0


def test_dense_histograms_are_transparent(B, golden_scenes, monkeypatch):
    """Dense-box histograms (root batch and flush cache, constant eps per
    level) and the shared-memory hash they replace give identical searches."""
    m, s, _, sc = load_case(B, golden_scenes, "campus")
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    ds = B.DeviceScan(vm, s)
    out = {}
    for flag in (None, "1"):
        if flag is None:
            monkeypatch.delenv("BBS_DENSE_HIST", raising=False)
        else:
            monkeypatch.setenv("BBS_DENSE_HIST", flag)
        cfg = B.SearchConfig(min_resolution=sc["r"], max_level=sc["max_level"], collect_trace=True)
        r = B.search_scan(vm, ds, cfg)
        out[flag] = (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated, r.stats.nodes_pruned,
                     r.stats.batches_flushed, tuple(r.best_score_trace), r.root_probes)
    assert out[None][:6] == out["1"][:6]


def test_large_scan_paths_are_transparent(B, golden_scenes, monkeypatch):
    """K = 70,000 (> 65535: no 16-bit dense histograms, hash builds; the
    root batch's early column exit, prebuild and probe chunks at a size the
    C2 bench never uses): cache on/off give identical searches."""
    m, raw, _ = H.gen_scene(H.SceneSpec.default(**golden_scenes["campus"]["spec"]),
                            golden_scenes["campus"]["seed"])
    s = H.cut_scan(raw, min(70000, raw.shape[0]), 3)
    sc = golden_scenes["campus"]
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    ds = B.DeviceScan(vm, s)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("BBS_ROT_CACHE", flag)
        cfg = B.SearchConfig(min_resolution=sc["r"], max_level=sc["max_level"], collect_trace=True)
        r = B.search_scan(vm, ds, cfg)
        out[flag] = (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated, r.stats.nodes_pruned,
                     r.stats.batches_flushed, tuple(r.best_score_trace))
    assert out["1"] == out["0"]
    assert s.shape[0] > 65535


@pytest.mark.parametrize("strategy", ["BFS", "DFS"])
@pytest.mark.parametrize("cobatch", ["1", "0", "0-tiled"])
def test_search_scans_throughput_mode_matches_single_searches(B, monkeypatch, strategy, cobatch):
    """bbs_search_scans (native workers, workspaces leased concurrently; the
    flushes of the searches in flight co-batched into one launch per epoch
    kernel, or each search on its own stream) returns each scan's search()
    result: Stats, trace, pose.  "0-tiled": concurrent streams with the merge
    kernel's claimed-task sort in its two-phase form from 257 survivors (the
    concurrent merges' CTAs share the SMs; no co-residency is assumed)."""
    cobatch, _, tiled = cobatch.partition("-")
    monkeypatch.setenv("BBS_COBATCH", cobatch)
    if tiled:
        monkeypatch.setenv("BBS_TILE_RANK_MIN", "256")
    spec = H.SceneSpec.default(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4, min_box_side=2.5,
                               max_box_side=6.0, min_box_height=3.0, map_spacing=0.3,
                               scan_spacing=0.45, scan_range=14.0, min_scan_points=300)
    m, _, _ = H.gen_scene(spec, 42)
    scans, _ = H.gen_scans(spec, 42, 1000, 9)
    vm = B.MultiResVoxelMap.build(m, 0.5, 3)
    ds = [B.DeviceScan(vm, s) for s in scans]
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, batch_size=400, collect_trace=True,
                         strategy=getattr(B.Strategy, strategy))
    many = B.search_scans(vm, ds, cfg, concurrency=4, trace_capacity=1 << 12)
    for d, r in zip(ds, many):
        one = B.search_scan(vm, d, cfg)
        assert (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated, r.stats.nodes_pruned,
                r.stats.batches_flushed, r.best_score_trace) == (
                    one.best_score, one.best_pose.as_tuple(), one.stats.nodes_generated, one.stats.nodes_pruned,
                    one.stats.batches_flushed, one.best_score_trace)
        assert one.group_checks == 0
    if cobatch == "1":
        assert sum(r.group_checks for r in many) > 0
    else:
        assert all(r.group_checks == 0 for r in many)


@pytest.mark.parametrize("strategy", ["BFS", "DFS"])
def test_large_batch_uses_radix_sorted_survivors(B, ref, golden_scenes, strategy):
    """batch_size above 16384 sorts each flush's survivors with a radix sort
    (not the O(n^2) rank sort): results equal the reference's search()."""
    m, s, _, sc = load_case(B, golden_scenes, "small")
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    cfg = make_cfg(B, sc, "small", dict(batch_size=40000, strategy=getattr(B.Strategy, strategy)))
    got = B.search(vm, s, cfg)
    rm = ref.map_build(m, sc["r"], sc["max_level"], 0.01)
    want, trace = rm.search(s, cfg.to_c(), trace_cap=1 << 16)
    assert got.best_score == want.best_score
    assert got.best_pose.as_tuple() == want.best_pose.as_tuple()
    assert (got.stats.nodes_generated, got.stats.nodes_pruned, got.stats.batches_flushed) == \
        (want.stats.nodes_generated, want.stats.nodes_pruned, want.stats.batches_flushed)
    assert got.best_score_trace == trace


@pytest.mark.parametrize("spec", ["1", "2", "5", "16", "16-host", "16-votes1"])
@pytest.mark.parametrize("name", ["small", "room"])
def test_speculative_rounds_match_reference(B, golden_scenes, name, spec, monkeypatch):
    """Speculative flush rounds (BFS; frontier_spec_kernel + survivors_spec_
    kernel): any round depth gives the reference's search() exactly -- score,
    pose, Stats, incumbent trace -- on searches with many flushes (small b=7:
    ~1.9k flushes; room: 73), with the rounds switched on by the device votes
    (default; after one vote) or by the host after its first check."""
    depth, _, mode = spec.partition("-")
    monkeypatch.setenv("BBS_SPEC", depth)
    if mode == "host":
        monkeypatch.setenv("BBS_SPEC_AUTO", "0")
    if mode == "votes1":
        monkeypatch.setenv("BBS_SPEC_VOTES", "1")
    m, s, _, sc = load_case(B, golden_scenes, name)
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    for label, want in golden_json(f"{name}_search.json").items():
        res = B.search(vm, s, make_cfg(B, sc, name, want["overrides"]))
        assert_same(res, want, f"{name}/{label}/spec{spec}")


@pytest.mark.parametrize("variant", ["rank-kernel", "fused-tiled", "fused", "fused-tiled-3ctas"])
@pytest.mark.parametrize("name", ["small", "room"])
def test_survivor_sort_variants_match_reference(B, golden_scenes, name, variant, monkeypatch):
    """The flush survivors' sort: a separate rank-sort kernel
    (BBS_FUSE_SORT=0), the merge kernel's claimed-tile rank sort (default), or
    its two-phase variant (tiles sorted in place, then ranked by binary
    searches in the other tiles; forced from 257 survivors), also on a
    3-CTA merge grid -- all give the reference's search() exactly, plain
    epochs and speculative rounds."""
    if variant == "rank-kernel":
        monkeypatch.setenv("BBS_FUSE_SORT", "0")
    if variant.startswith("fused-tiled"):
        monkeypatch.setenv("BBS_TILE_RANK_MIN", "256")
    if variant.endswith("3ctas"):  # a 3-CTA merge grid: every CTA loops over many tiles and sort tasks
        monkeypatch.setenv("BBS_MERGE_CTAS", "3")
    m, s, _, sc = load_case(B, golden_scenes, name)
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    for label, want in golden_json(f"{name}_search.json").items():
        res = B.search(vm, s, make_cfg(B, sc, name, want["overrides"]))
        assert_same(res, want, f"{name}/{label}/{variant}")


_FAST_PATHS_OFF = {"BBS_SPEC_AUTO": "0", "BBS_DIRECT_RUNS": "0", "BBS_ROT_CACHE": "0", "BBS_ROOT_INIT": "host"}


@pytest.mark.parametrize("strategy", ["BFS", "DFS"])
@pytest.mark.parametrize("b", [10000, 37])
def test_fast_paths_are_transparent(B, golden_scenes, monkeypatch, strategy, b):
    """The room scene (K = 2000: flush cache, device-switched rounds, direct
    runs all active) searched with the fast paths on and off: score, pose,
    Stats and trace identical (scripts/transparency_matrix.py sweeps 36
    configs on the C1 and C2 maps)."""
    m, s, _, sc = load_case(B, golden_scenes, "room")
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    ds = B.DeviceScan(vm, s)
    cfg = make_cfg(B, sc, "room", dict(batch_size=b, strategy=getattr(B.Strategy, strategy)))
    out = []
    for env in ({}, _FAST_PATHS_OFF):
        for k in _FAST_PATHS_OFF:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        r = B.search_scan(vm, ds, cfg)
        out.append((r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated, r.stats.nodes_pruned,
                    r.stats.batches_flushed, tuple(r.best_score_trace)))
    assert out[0] == out[1]
    assert s.shape[0] >= 2000  # the flush cache is on at this size


def test_cobatched_group_mixes_cached_and_uncached_slots(B, golden_scenes, monkeypatch):
    """Co-batched flushes with scans of K = 1,000 (no flush cache) and
    K = 3,000 (flush cache, speculative rounds) in the same group: every
    result equals the scan's own search."""
    monkeypatch.setenv("BBS_COBATCH", "1")
    m, _, _, sc = load_case(B, golden_scenes, "room")
    spec = H.SceneSpec.default(**sc["spec"])
    scans, _ = H.gen_scans(spec, sc["seed"], 500, 6)
    scans = [H.cut_scan(s, min(1000 if j % 2 else 3000, s.shape[0]), 11) for j, s in enumerate(scans)]
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
    ds = [B.DeviceScan(vm, s) for s in scans]
    cfg = make_cfg(B, sc, "room", dict(batch_size=2000))
    many = B.search_scans(vm, ds, cfg, concurrency=6, trace_capacity=1 << 14)
    assert sum(r.group_checks for r in many) > 0
    for d, r in zip(ds, many):
        one = B.search_scan(vm, d, cfg)
        assert (r.best_score, r.best_pose.as_tuple(), r.stats.nodes_generated, r.stats.nodes_pruned,
                r.stats.batches_flushed, r.best_score_trace) == (
                    one.best_score, one.best_pose.as_tuple(), one.stats.nodes_generated, one.stats.nodes_pruned,
                    one.stats.batches_flushed, one.best_score_trace)
