"""Device map build (K1-K3) parity: every level's occupied set equals the
reference's occupied_voxels() (golden digests + C restatement), membership
probes agree with a set model, both device layouts, edge cases, and the
reference's voxel_map_test.cpp known answers."""
import hashlib

import numpy as np
import pytest

from conftest import golden_json, load_case

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


LAYOUTS = ["AUTO", "BITMAP", "HASH"]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", ["tiny", "small", "room", "campus"])
def test_levels_match_golden(B, golden_scenes, name, layout):
    if name not in golden_scenes:
        pytest.skip("golden case not generated")
    m, s, _, sc = load_case(B, golden_scenes, name)
    vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"], layout=B.Layout[layout])
    for lv in golden_json(f"{name}_levels.json"):
        occ = vm.level(lv["level"]).occupied_voxels()
        assert occ.shape[0] == lv["count"], (name, lv["level"])
        assert digest(occ) == lv["digest"], (name, lv["level"])
        assert vm.level(lv["level"]).occupied_count() == lv["count"]


def test_bbox_and_resolutions(B):
    # voxel_map_test.cpp:180-195 (MultiRes.ResolutionsDouble / PaperDefaults)
    c = [[0.5, 0.5, 0.5], [3.5, 2.5, 1.5]]
    vm = B.MultiResVoxelMap.build(c, 1.0, 2)
    assert len(vm.levels()) == 3
    assert [vm.level(i).resolution() for i in range(3)] == [1.0, 2.0, 4.0]
    vm6 = B.MultiResVoxelMap.build([[0.5, 0.5, 0.5], [10, 20, 5]], 1.0, 6)
    assert len(vm6.levels()) == 7 and vm6.level(6).resolution() == 64.0
    assert vm.bbox() == ((0.5, 0.5, 0.5), (3.5, 2.5, 1.5))


@pytest.mark.parametrize("layout", ["BITMAP", "HASH"])
def test_single_point_inflates_to_eight(B, layout):
    # voxel_map_test.cpp:78-87
    vm = B.MultiResVoxelMap.build([[0.5, 0.5, 0.5]], 1.0, 1, layout=B.Layout[layout])
    lv = vm.level(0)
    assert lv.occupied_count() == 8
    for x in (-1, 0):
        for y in (-1, 0):
            for z in (-1, 0):
                assert lv.contains((x, y, z))
    assert not lv.contains((1, 0, 0)) and not lv.contains((-2, 0, 0))


def test_duplicate_points_set_semantics(B):
    a = B.MultiResVoxelMap.build([[0.5, 0.5, 0.5]], 1.0, 1)
    b = B.MultiResVoxelMap.build([[0.5, 0.5, 0.5], [0.4, 0.6, 0.5]], 1.0, 1)
    np.testing.assert_array_equal(a.level(0).occupied_voxels(), b.level(0).occupied_voxels())


@pytest.mark.parametrize("layout", ["BITMAP", "HASH"])
def test_membership_vs_set_model_100k(B, orc, layout):
    # voxel_map_test.cpp:119-140 (LookupMatchesReferenceSetOn100kProbes)
    rng = np.random.default_rng(31)
    pts = rng.uniform(-30, 30, size=(10000, 3))
    vm = B.MultiResVoxelMap.build(pts, 1.0, 1, layout=B.Layout[layout])
    om = orc.map_build(pts, 1.0, 1)
    ref_set = {tuple(v) for v in om.occupied(0)}
    near = rng.uniform(-31, 31, size=(50000, 3))
    far = rng.uniform(-500, 500, size=(50000, 3))
    probes = np.floor(np.concatenate([near, far])).astype(np.int32)
    got = vm.level(0).contains_many(probes)
    want = np.array([tuple(p) in ref_set for p in probes])
    np.testing.assert_array_equal(got, want)
    assert want.sum() > 1000 and (~want).sum() > 1000


def test_hierarchical_cover(B):
    # voxel_map_test.cpp:194-208: every leaf voxel centre is occupied at all levels
    rng = np.random.default_rng(43)
    pts = rng.uniform(-15, 15, size=(2000, 3))
    r = 0.7
    vm = B.MultiResVoxelMap.build(pts, r, 4)
    leaves = vm.level(0).occupied_voxels()
    centres = r * (leaves.astype(np.float64) + 0.5)
    for lv in range(5):
        cell = r * 2 ** lv
        vox = np.floor(centres / cell).astype(np.int32)
        assert vm.level(lv).contains_many(vox).all(), lv


def test_memory_cap_throws(B):
    # voxel_map_test.cpp:146-150 (MemoryCapThrows)
    rng = np.random.default_rng(29)
    pts = rng.uniform(-50, 50, size=(5000, 3))
    with pytest.raises(B.CapacityExceededError, match="exceeds memory cap"):
        B.MultiResVoxelMap.build(pts, 1.0, 1, memory_cap_bytes=4096)


def test_empty_set_probe_and_sentinel(B):
    vm = B.MultiResVoxelMap.build([[0.5, 0.5, 0.5]], 1.0, 1)
    i32min = -2147483648
    # contains(kEmpty) is false (voxel_map.hpp:131)
    assert not vm.level(0).contains((i32min, i32min, i32min))
    assert not vm.level(0).contains((i32min, 0, 0))


def test_from_levels_roundtrip(B, orc):
    rng = np.random.default_rng(7)
    pts = rng.uniform(0, 40, size=(3000, 3))
    vm = B.MultiResVoxelMap.build(pts, 0.5, 3)
    per_level = [vm.level(lv).occupied_voxels() for lv in range(4)]
    shuffled = [p[rng.permutation(p.shape[0])] for p in per_level]
    shuffled[1] = np.concatenate([shuffled[1], shuffled[1][:50]])  # duplicates are deduped
    vm2 = B.MultiResVoxelMap.from_levels(shuffled, 0.5, vm.bbox())
    for lv in range(4):
        np.testing.assert_array_equal(vm2.level(lv).occupied_voxels(), per_level[lv])
        assert vm2.level(lv).resolution() == 0.5 * 2 ** lv
    assert vm2.max_level() == 3 and vm2.bbox() == vm.bbox()


def test_from_levels_empty_level(B):
    vm = B.MultiResVoxelMap.from_levels([[[0, 0, 0], [1, 2, 3]], []], 1.0, ((0, 0, 0), (3, 3, 3)))
    assert vm.level(1).occupied_count() == 0
    assert not vm.level(1).contains((0, 0, 0))
    assert vm.level(0).contains((1, 2, 3))


def test_negative_and_boundary_coordinates(B, orc):
    # exact multiples of the cell, negatives (true floor), huge values
    pts = np.array([[0.0, 0.0, 0.0], [-0.2, -0.4, -0.6], [0.6, 0.4, 0.2], [-1e-12, 1e-12, 0.2],
                    [1.2000000000000002, -1.2, 0.5999999999999999]])
    vm = B.MultiResVoxelMap.build(pts, 0.2, 3)
    om = orc.map_build(pts, 0.2, 3)
    for lv in range(4):
        np.testing.assert_array_equal(vm.level(lv).occupied_voxels(), om.occupied(lv))


def test_layout_info(B):
    rng = np.random.default_rng(1)
    pts = rng.uniform(0, 50, size=(20000, 3))
    for layout in ("BITMAP", "HASH"):
        vm = B.MultiResVoxelMap.build(pts, 0.5, 3, layout=B.Layout[layout])
        for lv in range(4):
            L = vm.level(lv)
            assert L.layout().name == layout
            assert 0 < L.load_factor() < 1 and L.device_bytes() > 0
