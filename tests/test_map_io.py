"""load_map / save_map / is_map_file (map_io.hpp:17-126) -> device levels.

CPU: every format error is raised before any device work, with the reference's
status and message, on hand-made and corrupted files (checked against the
reference's own load_map, oracle/_ref).
GPU: files the reference saved load into identical occupied sets; our save is
byte-identical to the reference's save of the same map; a search on a loaded
map equals the search on the built map.
"""
import os
import struct

import numpy as np
import pytest
import harness as H  # noqa: E402  (synthetic inputs)

MAGIC = b"3DBBS\x01"


def _header(r=1.0, max_level=2, version=1, bbox=(0, 0, 0, 1, 1, 1), magic=MAGIC):
    return magic + struct.pack("<IdI6d", version, r, max_level, *bbox)


def _level(l, vox):
    v = np.asarray(vox, np.int32).reshape(-1, 3)
    return struct.pack("<IQ", l, v.shape[0]) + v.tobytes()


def _good_file(max_level=2):
    body = b"".join(_level(l, [[0, 0, 0], [1, 2, 3]]) for l in range(max_level + 1))
    return _header(max_level=max_level) + body


CASES = {
    "bad_magic": lambda: _header(magic=b"XXBBS\x01"),
    "short_magic": lambda: b"3DB",
    "bad_version": lambda: _header(version=2),
    "zero_resolution": lambda: _header(r=0.0),
    "nan_resolution": lambda: _header(r=float("nan")),
    "max_level_0": lambda: _header(max_level=0),
    "max_level_63": lambda: _header(max_level=63),
    "truncated_header": lambda: _header()[:20],
    "truncated_bbox": lambda: _header()[:-4],
    "no_levels": lambda: _header(),
    "levels_out_of_order": lambda: _header() + _level(1, [[0, 0, 0]]),
    "truncated_count": lambda: _header() + struct.pack("<I", 0) + b"\x01\x00",
    "truncated_voxels": lambda: _good_file()[:-6],
    "missing_last_level": lambda: _header() + _level(0, [[0, 0, 0]]) + _level(1, [[0, 0, 0]]),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_format_errors_match_reference(B, ref, tmp_path, case):
    p = tmp_path / f"{case}.vxm"
    p.write_bytes(CASES[case]())
    with pytest.raises(B.Error) as got:
        B.load_map(str(p))
    from pyoracle import OracleError
    with pytest.raises(OracleError) as want:
        ref.load_map(str(p))
    assert type(got.value) is B._ERRORS[want.value.code], (got.value, want.value)
    assert str(got.value) == want.value.message
    assert B.is_map_file(str(p)) == ref.is_map_file(str(p))


def test_huge_count_is_a_format_error(B, ref, tmp_path):
    """A level count beyond the file's remaining bytes: the reference's
    voxels.resize(count) (map_io.hpp:106) throws std::length_error (a generic
    Error here); the device loader checks the count against the file size and
    reports the truncation instead, before allocating anything."""
    p = tmp_path / "huge.vxm"
    p.write_bytes(_header() + struct.pack("<IQ", 0, 1 << 60))
    with pytest.raises(B.FormatError, match="truncated map file"):
        B.load_map(str(p))
    from pyoracle import OracleError
    with pytest.raises(OracleError):
        ref.load_map(str(p))


def test_missing_file_and_is_map_file(B, ref, tmp_path):
    p = str(tmp_path / "missing.vxm")
    with pytest.raises(B.FileNotFoundError_) as e:
        B.load_map(p)
    assert str(e.value) == f"file not found: {p}"
    assert not B.is_map_file(p) and not ref.is_map_file(p)
    good = tmp_path / "good.vxm"
    good.write_bytes(_good_file())
    assert B.is_map_file(str(good)) and ref.is_map_file(str(good))
    txt = tmp_path / "c.xyz"
    txt.write_text("1 2 3\n")
    assert not B.is_map_file(str(txt))


def _scene(B):
    spec = H.SceneSpec.default(size_x=24, size_y=24, size_z=10, num_boxes=4, min_box_side=2.5,
                               max_box_side=6.0, min_box_height=3.0, map_spacing=0.3,
                               scan_spacing=0.45, scan_range=14.0, min_scan_points=300)
    return H.gen_scene(spec, 42)


@pytest.mark.gpu
def test_save_is_byte_identical_to_reference(B, ref, tmp_path):
    m, _, _ = _scene(B)
    ours, theirs = tmp_path / "ours.vxm", tmp_path / "ref.vxm"
    B.MultiResVoxelMap.build(m, 0.5, 3).save(str(ours))
    ref.map_build(m, 0.5, 3, 0.3).save(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_load_reference_file_and_round_trip(B, ref, tmp_path):
    m, s, _ = _scene(B)
    theirs = tmp_path / "ref.vxm"
    ref.map_build(m, 0.5, 3, 0.3).save(str(theirs))
    loaded = B.load_map(str(theirs))
    built = B.MultiResVoxelMap.build(m, 0.5, 3)
    assert loaded.max_level() == 3 and loaded.min_resolution() == 0.5
    assert loaded.bbox() == built.bbox()
    for lv in range(4):
        assert np.array_equal(loaded.level(lv).occupied_voxels(), built.level(lv).occupied_voxels())
    # save of the loaded map reproduces the file
    again = tmp_path / "again.vxm"
    B.save_map(loaded, str(again))
    assert again.read_bytes() == theirs.read_bytes()
    # a search on the loaded map is the search on the built map
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, roll_pitch_half_range=0.02,
                         batch_size=500, collect_trace=True)
    a, b = B.search(loaded, s, cfg), B.search(built, s, cfg)
    assert (a.best_score, a.best_pose.as_tuple(), a.stats.nodes_generated, a.best_score_trace) == \
        (b.best_score, b.best_pose.as_tuple(), b.stats.nodes_generated, b.best_score_trace)


@pytest.mark.gpu
def test_load_map_empty_levels_and_duplicates(B, tmp_path):
    """Empty level blocks load as empty levels; duplicate voxels collapse
    (LevelMap::from_voxels keeps the set)."""
    p = tmp_path / "dup.vxm"
    p.write_bytes(_header(max_level=2) + _level(0, [[1, 1, 1], [1, 1, 1], [-5, 7, 2]]) +
                  _level(1, []) + _level(2, [[0, 0, 0]]))
    vm = B.load_map(str(p))
    assert vm.level(0).occupied_voxels().tolist() == [[-5, 7, 2], [1, 1, 1]]
    assert vm.level(1).occupied_voxels().shape[0] == 0
    assert vm.level(2).occupied_voxels().tolist() == [[0, 0, 0]]
