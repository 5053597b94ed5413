"""Device oracle_search (oracle.hpp:29-95) against the
reference's own oracle_search compiled from its sources (oracle/_ref): best
score, leaf count and every argmax pose (in the reference's enumeration
order) identical; the reference's validation errors; block-size invariance."""
import math

import numpy as np
import pytest

from test_search_gpu import mini_scene, small_cfg

pytestmark = pytest.mark.gpu


def _same(got, want, label):
    best, leaves, poses = want
    assert got.best_score == best, label
    assert got.leaf_count == leaves, label
    assert len(got.argmax_poses) == poses.shape[0], label
    for p, q in zip(got.argmax_poses, poses):
        assert p.as_tuple() == tuple(q), label


@pytest.mark.parametrize("mode", ["TRANS_ONLY", "ROTO_TRANS"])
@pytest.mark.parametrize("seed", [40, 41, 42])
def test_oracle_search_matches_reference(B, ref, seed, mode):
    prng = np.random.default_rng(seed * 7)
    gt = B.Pose6(prng.uniform(2, 12), prng.uniform(2, 12), prng.uniform(0, 1), 0, 0,
                 prng.uniform(0, 2 * math.pi))
    m, s = mini_scene(B, seed, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    rm = ref.map_build(m, 1.0, 2, 0.01)
    y = B.normalize_angle(gt.yaw)
    kw = dict(yaw_min=y - 0.3, yaw_max=y + 0.3,  # a window around gt keeps the CPU oracle fast
              translation_range=((gt.x - 2, gt.y - 2, 0.0), (gt.x + 2, gt.y + 2, 1.0)))
    if mode == "ROTO_TRANS":
        kw["roll_pitch_half_range"] = 0.05
    cfg = small_cfg(B, getattr(B.BranchMode, mode), **kw)
    got = B.oracle_search(vm, s, cfg)
    _same(got, rm.oracle_search(s, cfg.to_c()), (seed, mode))
    assert got.best_score > 0
    # the search's TransOnly best equals the exhaustive best (search_test.cpp:178-205)
    if mode == "TRANS_ONLY":
        r = B.search(vm, s, cfg)
        if got.best_score >= r.score_threshold:
            assert r.matched and r.best_score == got.best_score


def test_oracle_search_block_size_invariant(B, monkeypatch):
    gt = B.Pose6(6.0, 5.0, 0.4, 0, 0, 0.7)
    m, s = mini_scene(B, 43, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    cfg = small_cfg(B, B.BranchMode.ROTO_TRANS, yaw_min=0.4, yaw_max=1.0,
                    roll_pitch_half_range=0.03, translation_range=((5, 4, 0), (7, 6, 0.5)))
    a = B.oracle_search(vm, s, cfg)
    for blk in ("97", "4096"):
        monkeypatch.setenv("BBS_LEAF_BLOCK", blk)
        b = B.oracle_search(vm, s, cfg)  # one pass, every argmax leaf
        assert (b.best_score, b.leaf_count) == (a.best_score, a.leaf_count), blk
        assert np.array_equal(b.argmax_nodes, a.argmax_nodes), blk
        c = B.oracle_search(vm, s, cfg, argmax_capacity=1)  # the capped entry point
        assert (c.best_score, c.leaf_count) == (a.best_score, a.leaf_count), blk
        assert np.array_equal(c.argmax_nodes, a.argmax_nodes[:1]), blk
    # argmax nodes are level-0 leaves carrying the best score
    assert (a.argmax_nodes[:, 6] == 0).all() and (a.argmax_nodes[:, 7] == a.best_score).all()


def test_oracle_search_ties_keep_enumeration_order(B, ref):
    # a scan far from every voxel scores 0 everywhere: every leaf is an argmax
    m, _ = mini_scene(B, 44, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    rm = ref.map_build(m, 1.0, 2, 0.01)
    far = np.array([[0.0, 0.0, 400.0], [1.0, 0.0, 401.0]])
    cfg = small_cfg(B, B.BranchMode.TRANS_ONLY, yaw_min=0.0, yaw_max=0.2,
                    translation_range=((0, 0, 0), (3, 3, 1)))
    got = B.oracle_search(vm, far, cfg)
    want = rm.oracle_search(far, cfg.to_c(), cap=1 << 16)
    _same(got, want, "ties")
    assert got.best_score == 0 and len(got.argmax_poses) == got.leaf_count


def test_oracle_search_errors(B):
    # oracle.hpp:31-57, same exception types and order
    m, s = mini_scene(B, 45, B.Pose6())
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    cfg = small_cfg(B, B.BranchMode.TRANS_ONLY)
    with pytest.raises(B.DegenerateScanError, match="empty scan"):
        B.oracle_search(vm, np.zeros((0, 3)), cfg)
    with pytest.raises(B.ConfigError, match="config r does not match"):
        B.oracle_search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY, min_resolution=0.5))
    with pytest.raises(B.DegenerateScanError, match="zero scan range"):
        B.oracle_search(vm, np.zeros((2, 3)), cfg)
    with pytest.raises(B.TooLargeError, match="exceeds the 1e8 guard"):
        B.oracle_search(vm, s, small_cfg(B, B.BranchMode.ROTO_TRANS, roll_pitch_half_range=0.5,
                                         translation_range=((-200, -200, -20), (200, 200, 20))))
    with pytest.raises(B.EmptySearchSpaceError, match="empty leaf grid"):
        B.oracle_search(vm, s, small_cfg(B, B.BranchMode.TRANS_ONLY,
                                         translation_range=((4, 5, 5), (-1, 5, 5))))


def test_oracle_search_inverted_range_matches_reference(B, ref):
    """Two inverted translation axes: the reference's unsigned leaf count
    wraps to a small positive number that passes its guards (oracle.hpp:50-57)
    and its loops score nothing -> best_score -1, no argmax."""
    gt = B.Pose6(6.0, 5.0, 0.4, 0, 0, 0.7)
    m, s = mini_scene(B, 44, gt)
    vm = B.MultiResVoxelMap.build(m, 1.0, 2, 0.01)
    rm = ref.map_build(m, 1.0, 2, 0.01)
    # root cell 4 m: x and y index ranges [5, 2] -> leaf ranges [20, 12)
    cfg = small_cfg(B, B.BranchMode.TRANS_ONLY, yaw_min=0.4, yaw_max=0.6,
                    translation_range=((20, 20, 0), (5, 5, 0.5)))
    got = B.oracle_search(vm, s, cfg)
    want = rm.oracle_search(s, cfg.to_c())
    assert want[0] == -1 and want[2].shape[0] == 0
    _same(got, want, "inverted")
