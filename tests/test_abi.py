"""C-ABI surface (CPU): the library loads, exports every symbol declared in
include/bbs.h, struct layouts match the ctypes mirror, host-only entry points
map reference exceptions to status codes, and compute entry points fail
loudly (no CPU fallback) when no GPU is visible."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bbs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s+(bbs_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("bbs_map_build", "bbs_batch_evaluate", "bbs_search", "bbs_localize_scan",
                 "bbs_level_score", "bbs_search_sharded", "bbs_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(B):
    lib = C.CDLL(os.path.join(ROOT, "paper_2310_10023_b200", "libbbs_b200.so"))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_dynamic_symbol_table_matches_header():
    so = os.path.join(ROOT, "paper_2310_10023_b200", "libbbs_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T bbs_" in ln}
    assert set(declared_functions()) <= exported


def test_python_binding_covers_header(B):
    from paper_2310_10023_b200 import _lib
    assert set(declared_functions()) <= set(_lib.exported_symbols())


def test_struct_sizes(B):
    from paper_2310_10023_b200 import _abi
    assert C.sizeof(_abi.Node) == 32           # bnbloc::Node, nodes.hpp:18-29
    assert C.sizeof(_abi.Pose6) == 48
    assert C.sizeof(_abi.Aabb) == 48
    assert C.sizeof(_abi.StatsC) == 64
    # the library writes the config defaults into our mirror: a layout
    # mismatch would scramble these fields
    c = _abi.SearchConfigC()
    B.lib.bbs_search_config_default(C.byref(c))
    assert (c.min_resolution, c.max_level, c.roll_pitch_half_range, c.batch_size,
            c.strategy, c.branch_mode, c.workers) == (1.0, 6, 0.02, 10000, 1, 1, 1)
    assert c.score_threshold_fraction == 0.95 and c.yaw_max == _abi.TWO_PI


def test_abi_version(B):
    from paper_2310_10023_b200 import _lib
    assert B.lib.bbs_abi_version() == _lib.ABI_VERSION == 5


def test_search_config_defaults_match_reference(B):
    cfg = B.SearchConfig()  # search_config.hpp:24-52
    assert (cfg.min_resolution, cfg.max_level, cfg.roll_pitch_half_range,
            cfg.score_threshold_fraction, cfg.batch_size) == (1.0, 6, 0.02, 0.95, 10000)
    assert cfg.strategy == B.Strategy.BFS and cfg.branch_mode == B.BranchMode.ROTO_TRANS


def test_host_errors_map_to_reference_exceptions(B):
    cfg = B.SearchConfig(min_resolution=1.0, max_level=3)
    with pytest.raises(B.DegenerateScanError, match="angular_step: d_max must be > 0"):
        B.AngularGrid(cfg, 0.0)
    bad = B.SearchConfig(yaw_min=1.0, yaw_max=1.0)
    with pytest.raises(B.ConfigError, match="yaw range must have positive width"):
        B.AngularGrid(bad, 10.0)
    with pytest.raises(B.ConfigError, match="roll/pitch range must be >= 0"):
        B.AngularGrid(B.SearchConfig(roll_pitch_half_range=-0.1), 10.0)
    with pytest.raises(B.EmptyCloudError, match="max_range: empty cloud"):
        B.max_range([])
    with pytest.raises(B.EmptyCloudError, match="bounding_box: empty cloud"):
        B.bounding_box([])


def test_no_gpu_means_loud_failure(B):
    if B.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(B.CudaError, match="no CPU fallback"):
        B.MultiResVoxelMap.build([[0.5, 0.5, 0.5]], 1.0, 2)


def test_map_build_validation_order_without_gpu(B):
    # validation happens on the host before any device work (voxel_map.hpp:230-233)
    with pytest.raises(B.EmptyCloudError, match="MultiResVoxelMap: empty map"):
        B.MultiResVoxelMap.build([], 1.0, 3)
    with pytest.raises(B.ConfigError, match="max_level must be >= 1"):
        B.MultiResVoxelMap.build([[0, 0, 0]], 1.0, 0)
    with pytest.raises(B.ConfigError, match="min_resolution must be > 0"):
        B.MultiResVoxelMap.build([[0, 0, 0]], -1.0, 3)


def test_from_levels_requires_two_levels(B):
    with pytest.raises(B.FormatError, match="at least 2 levels"):
        B.MultiResVoxelMap.from_levels([[[0, 0, 0]]], 1.0, ((0, 0, 0), (1, 1, 1)))
