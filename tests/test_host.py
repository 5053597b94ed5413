"""Host-side logic of the product library (no GPU): the AngularGrid /
prepare_source / bounding-box restatements and the synthetic scene
generator, each checked against the reference (oracle/_ref) and against the
known-answer tests of proj/tests/angular_grid_test.cpp."""
import math

import numpy as np
import pytest
import harness as H  # noqa: E402  (synthetic inputs)

PI = 3.14159265358979323846


def grid_tuple(g):
    return (g.w_min, g.w_max, g.step, g.segments, bool(g.periodic))


# ---- angular_grid_test.cpp known answers -----------------------------------
def test_kat_roots_desk_scale(B):
    # angular_grid_test.cpp:196-211: yaw segments at level 3 = 24; 9*9*3*24 roots
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3, roll_pitch_half_range=0.0)
    g = B.AngularGrid(cfg, 30.0)
    assert g.axis(2, 3).segments == 24
    assert B.initial_node_count(cfg, 30.0, ((0, 0, 0), (64, 64, 16))) == 9 * 9 * 3 * 24


def test_kat_root_range_floor_ceil(B):
    # angular_grid_test.cpp:177-194
    cfg = B.SearchConfig(min_resolution=1.0, max_level=6, roll_pitch_half_range=0.0)
    g = B.AngularGrid(cfg, 0.26)
    assert g.axis(2, 6).index_count() == 2
    assert B.initial_node_count(cfg, 0.26, ((0, 0, 0), (100, 100, 100))) == 27 * 2
    cfg2 = B.SearchConfig(min_resolution=1.0, max_level=2, roll_pitch_half_range=0.0)
    g2 = B.AngularGrid(cfg2, 0.26)
    assert B.initial_node_count(cfg2, 0.26, ((-5, -5, -5), (5, 5, 5))) == \
        125 * g2.axis(2, 2).index_count()


def test_kat_transonly_uses_leaf_step(B):
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3, branch_mode=B.BranchMode.TRANS_ONLY)
    g = B.AngularGrid(cfg, 30.0)
    for lv in range(4):
        assert g.axis(2, lv).step == g.axis(2, 0).step
        if lv > 0:
            assert g.divisions(2, lv) == 1


def test_kat_divisions_overshoot(B):
    # angular_grid_test.cpp:266-291: d_max 1.4 -> yaw segments 4 (level 1), 9 (level 0), a = 3
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3, roll_pitch_half_range=0.0)
    g = B.AngularGrid(cfg, 1.4)
    assert g.axis(2, 1).segments == 4 and g.axis(2, 0).segments == 9
    assert g.divisions(2, 1) == 3


def test_kat_roll_pitch_endpoints(B):
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3, roll_pitch_half_range=0.02)
    g = B.AngularGrid(cfg, 30.0)
    roll = g.axis(0, 0)
    assert roll.index_count() == roll.segments + 1
    assert roll.angle(0) == -0.02
    assert abs(roll.angle(roll.max_index()) - 0.02) <= 1e-15
    yaw = g.axis(2, 0)
    assert yaw.index_count() == yaw.segments and yaw.angle(yaw.max_index()) < 2 * PI


def test_kat_node_pose(B):
    # angular_grid_test.cpp:134-150
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3, roll_pitch_half_range=0.02)
    g = B.AngularGrid(cfg, 30.0)
    p0 = B.node_pose((0, 0, 0, 0, 0, 0, 0, -1), g, 1.0)
    assert (p0.x, p0.roll, p0.pitch, p0.yaw) == (0.0, -0.02, -0.02, 0.0)
    p1 = B.node_pose((3, -1, 2, 0, 0, 0, 2, -1), g, 1.0)
    assert (p1.x, p1.y, p1.z) == (12.0, -4.0, 8.0)


# ---- bit-identity against the reference -------------------------------------
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("d_max", [0.3, 1.4, 25.0, 37.3, 61.0])
def test_angular_grid_bit_identical(B, ref, mode, d_max):
    cfg = B.SearchConfig(min_resolution=0.2, max_level=6, roll_pitch_half_range=0.0873,
                         branch_mode=mode)
    ours = [grid_tuple(a) for a in B.AngularGrid(cfg, d_max)._axes]
    theirs = [grid_tuple(a) for a in ref.angular_grid(cfg.to_c(), d_max)]
    assert ours == theirs
    for lv in range(1, 7):
        for ax in range(3):
            assert B.AngularGrid(cfg, d_max).divisions(ax, lv) == \
                ref.divisions(cfg.to_c(), d_max, ax, lv)


def test_pose_to_transform_bit_identical(B, ref):
    rng = np.random.default_rng(3)
    for _ in range(200):
        p = B.Pose6(*rng.uniform(-10, 10, 3), *rng.uniform(-0.2, 0.2, 2), rng.uniform(0, 7))
        R, t = B.pose_to_transform(p)
        R2, t2 = ref.pose_to_transform(p.as_tuple())
        assert list(R) == list(R2) and list(t) == list(t2)


@pytest.mark.parametrize("seed", [1, 7, 42])
def test_gen_scene_bit_identical(B, ref, seed):
    kw = dict(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4, min_box_side=2.5,
              max_box_side=6.0, min_box_height=3.0, map_spacing=0.3, scan_spacing=0.45,
              scan_range=14.0, min_scan_points=300)
    m1, s1, gt1 = H.gen_scene(H.SceneSpec.default(**kw), seed)
    spec = ref.default_spec()
    for k, v in kw.items():
        setattr(spec, k, v)
    m2, s2, gt2 = ref.gen_scene(spec, seed)
    np.testing.assert_array_equal(m1, m2)
    np.testing.assert_array_equal(s1, s2)
    assert gt1.as_tuple() == gt2


def test_gen_scene_deterministic_and_feasible(B):
    # harness_test.cpp:31-62
    spec = H.SceneSpec.default(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4,
                               min_box_side=2.5, max_box_side=6.0, min_box_height=3.0,
                               map_spacing=0.3, scan_spacing=0.45, scan_range=14.0,
                               min_scan_points=300)
    a = H.gen_scene(spec, 42)
    b = H.gen_scene(spec, 42)
    np.testing.assert_array_equal(a[0], b[0])
    assert a[2].as_tuple() == b[2].as_tuple()
    assert a[1].shape[0] >= 300
    assert abs(a[2].roll) <= 0.01 and abs(a[2].pitch) <= 0.01


def test_gen_scans_match_gen_scene_layout(B):
    spec = H.SceneSpec.default(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4,
                               min_box_side=2.5, max_box_side=6.0, min_box_height=3.0,
                               map_spacing=0.3, scan_spacing=0.45, scan_range=14.0,
                               min_scan_points=300)
    scans, poses = H.gen_scans(spec, 42, 1000, 3)
    assert len(scans) == 3 and all(s.shape[0] >= 300 for s in scans)
    assert len({p.as_tuple() for p in poses}) == 3


def test_cut_scan_is_a_seeded_prefix(B):
    pts = np.arange(300, dtype=np.float64).reshape(100, 3)
    a = H.cut_scan(pts, 40, 7)
    b = H.cut_scan(pts, 40, 7)
    np.testing.assert_array_equal(a, b)
    rows = {tuple(r) for r in pts}
    assert all(tuple(r) in rows for r in a) and len({tuple(r) for r in a}) == 40
    # same as the golden generator's pure-Python Fisher-Yates
    from golden.make_golden import cut_scan
    np.testing.assert_array_equal(a, cut_scan(pts, 40, 7))


@pytest.mark.parametrize("target", [0, 300, 1000, 5000])
def test_prepare_source_bit_identical(B, ref, target):
    spec = H.SceneSpec.default(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4,
                               min_box_side=2.5, max_box_side=6.0, min_box_height=3.0,
                               map_spacing=0.3, scan_spacing=0.2, scan_range=14.0,
                               min_scan_points=300)
    _, raw, _ = H.gen_scene(spec, 9)
    ours = B.prepare_source(raw, target)
    scan, leaf, conv, dmax = ref.prepare_source(raw, target)
    np.testing.assert_array_equal(ours.scan, scan)
    assert (ours.leaf, ours.leaf_converged, ours.d_max) == (leaf, conv, dmax)


def test_prepare_source_campus_raw_scan_bit_identical(B, ref):
    """C2 raw scan (~236k points -> target 10k): the packed-key replay of the
    reference's introsort gives its per-voxel summation order exactly."""
    spec = H.SceneSpec.default(size_x=300.0, size_y=300.0, size_z=30.0, num_boxes=60,
                               min_box_side=6.0, max_box_side=30.0, min_box_height=8.0,
                               map_spacing=0.19, scan_spacing=0.3, scan_range=60.0,
                               min_scan_points=400)
    _, raw, _ = H.gen_scene(spec, 1)
    ours = B.prepare_source(raw, 10000)
    scan, leaf, conv, dmax = ref.prepare_source(raw, 10000)
    np.testing.assert_array_equal(ours.scan, scan)
    assert (ours.leaf, ours.leaf_converged, ours.d_max) == (leaf, conv, dmax)


def test_prepare_source_unpackable_voxels_bit_identical(B, ref):
    """Voxel indices spanning more than 64 packed bits take the reference's
    own record layout; NaN coordinates map to INT64_MIN voxels as on x86."""
    rng = np.random.default_rng(8)
    raw = rng.normal(size=(3000, 3))
    raw[:40] *= 1e17  # ~2^57 voxels apart on every axis at the chosen leaf
    raw[40:43, 1] = np.nan
    ours = B.prepare_source(raw, 500)
    scan, leaf, conv, dmax = ref.prepare_source(raw, 500)
    np.testing.assert_array_equal(ours.scan, scan)
    assert (ours.leaf, ours.leaf_converged) == (leaf, conv)
    assert (ours.d_max == dmax) or (np.isnan(ours.d_max) and np.isnan(dmax))


def test_max_range_and_bbox_bit_identical(B, ref):
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(5000, 3)) * 17.0
    assert B.max_range(pts) == ref.max_range(pts)
    (lo, hi) = B.bounding_box(pts)
    assert lo == tuple(pts.min(axis=0)) and hi == tuple(pts.max(axis=0))


def test_gen_scans_bit_identical(ref):
    """C4 harness helper: harness/libbbs_scene.so's gen_scans equals
    oracle/_ref's ref_gen_scans (the reference's own scene internals)."""
    kw = dict(size_x=40.0, size_y=40.0, size_z=10.0, num_boxes=5, min_box_side=3.0,
              max_box_side=8.0, min_box_height=3.0, map_spacing=0.3, scan_spacing=0.45,
              scan_range=20.0, min_scan_points=300)
    a, pa = H.gen_scans(H.SceneSpec.default(**kw), 3, 1000, 4)
    spec = ref.default_spec()
    for k, v in kw.items():
        setattr(spec, k, v)
    b, pb = ref.gen_scans(spec, 3, 1000, 4)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    assert [p.as_tuple() for p in pa] == pb


def test_cut_scan_python_equals_native():
    rng = np.random.default_rng(3)
    pts = rng.normal(size=(5000, 3))
    for k in (0, 1, 777, 5000):
        np.testing.assert_array_equal(H.cut_scan(pts, k, 7), H.cut_scan_py(pts, k, 7))
