"""Pins the CPU oracle (oracle/bbs_oracle.c, the plain-C restatement) to the
reference: against the committed golden fixtures (generated from the
reference itself by tests/golden/make_golden.py) and, where oracle/_ref is
built, against the reference live on fresh seeded inputs.  CPU only."""
import hashlib

import numpy as np
import pytest
import harness as H  # noqa: E402  (synthetic inputs)

from conftest import golden_json, golden_npz, load_case


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["tiny", "small", "room"])
def test_restated_map_matches_golden_sets(B, orc, golden_scenes, name):
    m, s, _, sc = load_case(B, golden_scenes, name)
    om = orc.map_build(m, sc["r"], sc["max_level"])
    for lv in golden_json(f"{name}_levels.json"):
        occ = om.occupied(lv["level"])
        assert occ.shape[0] == lv["count"]
        assert digest(occ) == lv["digest"]


@pytest.mark.parametrize("name", ["tiny", "small", "room"])
def test_restated_batch_scores_match_golden(B, orc, golden_scenes, name):
    m, s, _, sc = load_case(B, golden_scenes, name)
    om = orc.map_build(m, sc["r"], sc["max_level"])
    g = golden_npz(f"{name}_batch.npz")
    from pyoracle import default_config
    cfg = default_config(min_resolution=sc["r"], max_level=sc["max_level"],
                         roll_pitch_half_range=0.0873 if name == "room" else 0.02)
    got = om.batch_evaluate(s, cfg, g["nodes"][:1500])
    np.testing.assert_array_equal(got[:, 7], g["scores"][:1500])


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_restated_search_matches_golden(B, orc, golden_scenes, name):
    m, s, _, sc = load_case(B, golden_scenes, name)
    om = orc.map_build(m, sc["r"], sc["max_level"])
    from pyoracle import default_config
    for label, want in golden_json(f"{name}_search.json").items():
        if want["nodes_generated"] > 100000:
            continue  # keep the CPU suite fast; the GPU suite checks all of them
        kw = dict(min_resolution=sc["r"], max_level=sc["max_level"], roll_pitch_half_range=0.02,
                  collect_trace=1)
        kw.update(want["overrides"])
        r, trace = om.search(s, default_config(**kw))
        assert r.best_score == want["best_score"], label
        assert bool(r.matched) == want["matched"], label
        assert list(r.best_pose.as_tuple()) == want["best_pose"], label
        assert (r.stats.nodes_generated, r.stats.nodes_pruned, r.stats.batches_flushed) == \
            (want["nodes_generated"], want["nodes_pruned"], want["batches_flushed"]), label
        assert trace == want["trace"], label


def test_restatement_vs_reference_live(B, ref, orc):
    """Fresh seeds: map sets, scores and full searches agree exactly."""
    spec = H.SceneSpec.default(size_x=16, size_y=16, size_z=8, num_boxes=3, min_box_side=2.0,
                               max_box_side=5.0, min_box_height=2.0, map_spacing=0.3,
                               scan_spacing=0.5, scan_range=10.0, min_scan_points=200)
    from pyoracle import default_config
    for seed in (3, 5):
        m, s, _ = H.gen_scene(spec, seed)
        rm = ref.map_build(m, 0.5, 3, 0.05)
        om = orc.map_build(m, 0.5, 3)
        for lv in range(4):
            np.testing.assert_array_equal(rm.occupied(lv), om.occupied(lv))
        for strat in (0, 1):
            cfg = default_config(min_resolution=0.5, max_level=3, strategy=strat, batch_size=300,
                                 collect_trace=1)
            r1, t1 = rm.search(s, cfg)
            r2, t2 = om.search(s, cfg)
            assert r1.best_score == r2.best_score and t1 == t2
            assert r1.best_pose.as_tuple() == r2.best_pose.as_tuple()
            assert (r1.stats.nodes_generated, r1.stats.nodes_pruned) == \
                (r2.stats.nodes_generated, r2.stats.nodes_pruned)


def test_restated_voxel_index_x86_semantics(orc):
    # point_cloud.hpp:39 on x86: cvttsd2si gives INT32_MIN out of range / NaN
    assert orc.voxel_index(3e9, 1.0) == -2147483648
    assert orc.voxel_index(-3e9, 1.0) == -2147483648
    assert orc.voxel_index(float("nan"), 1.0) == -2147483648
    assert orc.voxel_index(-0.5, 1.0) == -1
    assert orc.voxel_index(2147483647.5, 1.0) == 2147483647


def test_reference_voxel_kats(ref):
    """voxel_map_test.cpp:78-96: a single point inflates to the 8 voxels {-1,0}^3."""
    rm = ref.map_build([[0.5, 0.5, 0.5]], 1.0, 1, 0.001)
    occ = rm.occupied(0)
    assert occ.shape[0] == 8
    assert {tuple(v) for v in occ} == {(x, y, z) for x in (-1, 0) for y in (-1, 0) for z in (-1, 0)}
