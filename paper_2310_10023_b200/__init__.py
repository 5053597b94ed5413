"""B200-native batched branch-and-bound scan matcher (3D-BBS hot path).

A Python mirror of the reference's localizer API (``bnbloc``,
/root/reference/proj/include/bnbloc) over the C-ABI of include/bbs.h: the
same names, argument meanings and exception types, so code and tests written
against ``bnbloc`` read the same here.  All compute runs on the GPU through
libbbs_b200.so; there is no CPU fallback.

    MultiResVoxelMap.build   voxel_map.hpp:226      (device map build, K1-K3)
    LevelMap.score           voxel_map.hpp:142      (K4 score)
    batch_evaluate           search.hpp:23          (K4 over node batches)
    search                   search.hpp:72          (device frontier, K5-K6)
    localize_scan            pipeline.hpp:45
    AngularGrid              angular_grid.hpp:65
"""
import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from ._abi import Aabb, AxisGridC, LevelInfo, MapOptions, Node, SearchConfigC, SearchResultC, Shard
from ._lib import lib

__all__ = [
    "Error", "FileNotFoundError_", "ParseError", "EmptyCloudError", "CapacityExceededError",
    "IoError", "FormatError", "DegenerateScanError", "EmptySearchSpaceError", "TooLargeError",
    "InfeasiblePoseError", "ConfigError", "CudaError", "InvalidArgumentError",
    "Strategy", "BranchMode", "Layout", "SearchConfig", "Stats", "SearchResult", "Pose6",
    "AxisGrid", "AngularGrid", "LevelMap", "MultiResVoxelMap", "DeviceScan", "NODE_DTYPE",
    "batch_evaluate", "search", "search_scan_dump", "search_sharded", "search_scans", "Comm", "nccl_version",
    "save_map", "load_map", "is_map_file", "localize_scan", "prepare_source", "prepare_source_device",
    "max_range", "bounding_box", "pose_to_transform", "node_pose", "initial_node_count",
    "device_count",
]

KTWO_PI = _abi.TWO_PI


# ---- errors (errors.hpp:11-98) ---------------------------------------------
class Error(RuntimeError):
    """bnbloc::Error."""


class FileNotFoundError_(Error):
    pass


class ParseError(Error):
    pass


class EmptyCloudError(Error):
    pass


class CapacityExceededError(Error):
    pass


class IoError(Error):
    pass


class FormatError(Error):
    pass


class DegenerateScanError(Error):
    pass


class EmptySearchSpaceError(Error):
    pass


class TooLargeError(Error):
    pass


class InfeasiblePoseError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    """Device failure (no reference counterpart)."""


class InvalidArgumentError(Error):
    """Null handle / bad buffer (no reference counterpart)."""


_ERRORS = {
    1: Error, 2: FileNotFoundError_, 3: ParseError, 4: EmptyCloudError,
    5: CapacityExceededError, 6: IoError, 7: FormatError, 8: DegenerateScanError,
    9: EmptySearchSpaceError, 10: TooLargeError, 11: InfeasiblePoseError, 12: ConfigError,
    13: CudaError, 14: InvalidArgumentError,
}


def _check(status, msg_fn=None):
    if status != 0:
        msg = (msg_fn or lib.bbs_last_error)()
        raise _ERRORS.get(status, Error)(msg.decode() if isinstance(msg, bytes) else str(msg))


def device_count():
    return lib.bbs_device_count()


# ---- config / results (search_config.hpp) ----------------------------------
class Strategy(enum.IntEnum):
    DFS = 0  # kDfs
    BFS = 1  # kBfs


class BranchMode(enum.IntEnum):
    TRANS_ONLY = 0  # kTransOnly
    ROTO_TRANS = 1  # kRotoTrans


class Layout(enum.IntEnum):
    AUTO = 0
    BITMAP = 1
    HASH = 2


@dataclass
class Pose6:
    """geometry.hpp:46-60."""
    x: float = 0.0
    y: float = 0.0
    z: float = 0.0
    roll: float = 0.0
    pitch: float = 0.0
    yaw: float = 0.0

    def normalized(self):
        return Pose6(self.x, self.y, self.z, self.roll, self.pitch, normalize_angle(self.yaw))

    def as_tuple(self):
        return (self.x, self.y, self.z, self.roll, self.pitch, self.yaw)


@dataclass
class SearchConfig:
    """search_config.hpp:24-52 (same fields and defaults)."""
    min_resolution: float = 1.0
    max_level: int = 6
    translation_range: Optional[tuple] = None  # ((minx, miny, minz), (maxx, maxy, maxz))
    roll_pitch_half_range: float = 0.02
    yaw_min: float = 0.0
    yaw_max: float = KTWO_PI
    score_threshold_fraction: float = 0.95
    batch_size: int = 10000
    strategy: Strategy = Strategy.BFS
    branch_mode: BranchMode = BranchMode.ROTO_TRANS
    workers: int = 1
    d_max: Optional[float] = None
    collect_trace: bool = False

    def to_c(self) -> SearchConfigC:
        c = SearchConfigC()
        lib.bbs_search_config_default(C.byref(c))
        c.min_resolution = float(self.min_resolution)
        c.max_level = int(self.max_level)
        if self.translation_range is not None:
            c.has_translation_range = 1
            (a, b) = self.translation_range
            c.translation_range.min.x, c.translation_range.min.y, c.translation_range.min.z = a
            c.translation_range.max.x, c.translation_range.max.y, c.translation_range.max.z = b
        c.roll_pitch_half_range = float(self.roll_pitch_half_range)
        c.yaw_min = float(self.yaw_min)
        c.yaw_max = float(self.yaw_max)
        c.score_threshold_fraction = float(self.score_threshold_fraction)
        c.batch_size = int(self.batch_size)
        c.strategy = int(self.strategy)
        c.branch_mode = int(self.branch_mode)
        c.workers = int(self.workers)
        if self.d_max is not None:
            c.has_d_max = 1
            c.d_max = float(self.d_max)
        c.collect_trace = 1 if self.collect_trace else 0
        return c


@dataclass
class Stats:
    """search_config.hpp:55-69."""
    nodes_generated: int = 0
    nodes_pruned: int = 0
    batches_flushed: int = 0
    create_voxel_maps_ms: float = 0.0
    set_source_ms: float = 0.0
    initial_nodes_ms: float = 0.0
    find_best_score_ms: float = 0.0
    pop_remaining_queue_ms: float = 0.0

    def preprocessing_total_ms(self):
        return self.create_voxel_maps_ms + self.set_source_ms

    def localization_total_ms(self):
        return self.initial_nodes_ms + self.find_best_score_ms + self.pop_remaining_queue_ms


@dataclass
class SearchResult:
    """search_config.hpp:71-80, plus device extensions."""
    best_pose: Pose6 = field(default_factory=Pose6)
    best_score: int = 0
    score_threshold: int = 0
    scan_points: int = 0
    matched: bool = False
    stats: Stats = field(default_factory=Stats)
    best_score_trace: List[int] = field(default_factory=list)
    best_node: tuple = ()
    epochs: int = 0
    lookups: int = 0
    device_ms: float = 0.0
    root_score_ms: float = 0.0
    epoch_score_ms: float = 0.0
    root_nodes: int = 0
    queue_peak: int = 0
    root_probes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    evals_per_level: tuple = ()
    root_words: int = 0
    root_col_ms: float = 0.0
    group_checks: int = 0


def _result_from_c(r: SearchResultC, trace_buf=None) -> SearchResult:
    s = r.stats
    out = SearchResult(
        best_pose=Pose6(*r.best_pose.as_tuple()), best_score=r.best_score,
        score_threshold=r.score_threshold, scan_points=r.scan_points, matched=bool(r.matched),
        stats=Stats(s.nodes_generated, s.nodes_pruned, s.batches_flushed, s.create_voxel_maps_ms,
                    s.set_source_ms, s.initial_nodes_ms, s.find_best_score_ms,
                    s.pop_remaining_queue_ms),
        best_node=tuple(getattr(r.best_node, f) for f in _abi.NODE_DTYPE_FIELDS),
        epochs=r.epochs, lookups=r.lookups, device_ms=r.device_ms, root_score_ms=r.root_score_ms,
        epoch_score_ms=r.epoch_score_ms, root_nodes=r.root_nodes, queue_peak=r.queue_peak,
        root_probes=r.root_probes, h2d_bytes=r.h2d_bytes, d2h_bytes=r.d2h_bytes,
        kernel_launches=r.kernel_launches, evals_per_level=tuple(r.evals_per_level),
        root_words=r.root_words, root_col_ms=r.root_col_ms, group_checks=r.group_checks)
    if trace_buf is not None:
        out.best_score_trace = list(trace_buf[: min(r.trace_length, len(trace_buf))])
    return out


def _new_result(trace_cap):
    res = SearchResultC()
    buf = None
    if trace_cap:
        buf = (C.c_int32 * trace_cap)()
        res.best_score_trace = C.cast(buf, C.POINTER(C.c_int32))
        res.trace_capacity = trace_cap
    return res, buf


# ---- geometry helpers (geometry.hpp) ----------------------------------------
def normalize_angle(a):
    """geometry.hpp:36-43."""
    r = math.fmod(a, KTWO_PI)
    if r < 0.0:
        r += KTWO_PI
    if r >= KTWO_PI:
        r = 0.0
    return r


def pose_to_transform(p: Pose6):
    """geometry.hpp:102-112 -> (rotation row-major list of 9, translation)."""
    ca, sa = math.cos(p.roll), math.sin(p.roll)
    cb, sb = math.cos(p.pitch), math.sin(p.pitch)
    cg, sg = math.cos(p.yaw), math.sin(p.yaw)
    R = [cg * cb, cg * sb * sa - sg * ca, cg * sb * ca + sg * sa,
         sg * cb, sg * sb * sa + cg * ca, sg * sb * ca - cg * sa,
         -sb, cb * sa, cb * ca]
    return R, [p.x, p.y, p.z]


def _xyz(points):
    a = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    return a


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def max_range(points):
    """point_cloud.hpp:58-63."""
    a = _xyz(points)
    out = C.c_double()
    _check(lib.bbs_max_range(_dptr(a), a.shape[0], C.byref(out)))
    return out.value


def bounding_box(points):
    """point_cloud.hpp:42-54 -> ((min), (max))."""
    a = _xyz(points)
    b = Aabb()
    _check(lib.bbs_bounding_box(_dptr(a), a.shape[0], C.byref(b)))
    return (b.min.x, b.min.y, b.min.z), (b.max.x, b.max.y, b.max.z)


@dataclass
class SourcePrep:
    """pipeline.hpp:14-20."""
    scan: np.ndarray
    leaf: float
    leaf_converged: bool
    d_max: float


def prepare_source(raw_scan, target_points):
    """pipeline.hpp:25-41 (host C++ in libbbs_b200)."""
    a = _xyz(raw_scan)
    cnt = C.c_uint64()
    leaf, dm = C.c_double(), C.c_double()
    conv = C.c_int32()
    _check(lib.bbs_prepare_source(_dptr(a), a.shape[0], int(target_points), None, 0,
                                  C.byref(cnt), None, None, None))
    out = np.zeros((cnt.value, 3))
    _check(lib.bbs_prepare_source(_dptr(a), a.shape[0], int(target_points), _dptr(out), cnt.value,
                                  C.byref(cnt), C.byref(leaf), C.byref(conv), C.byref(dm)))
    return SourcePrep(out, leaf.value, bool(conv.value), dm.value)


def prepare_source_device(raw_scan, target_points, device=0):
    """pipeline.hpp:25-41 on the device (bbs_prepare_source_device): exact
    leaf / convergence / voxel set; centroid sums in input order."""
    a = _xyz(raw_scan)
    cnt = C.c_uint64()
    leaf, dm = C.c_double(), C.c_double()
    conv = C.c_int32()
    out = np.zeros((max(a.shape[0], 1), 3))
    _check(lib.bbs_prepare_source_device(int(device), _dptr(a), a.shape[0], int(target_points), _dptr(out),
                                         out.shape[0], C.byref(cnt), C.byref(leaf), C.byref(conv),
                                         C.byref(dm)))
    return SourcePrep(out[: cnt.value].copy(), leaf.value, bool(conv.value), dm.value)


# ---- angular grid (angular_grid.hpp) ----------------------------------------
@dataclass
class AxisGrid:
    """angular_grid.hpp:45-58."""
    w_min: float
    w_max: float
    step: float
    segments: int
    periodic: bool

    def max_index(self):
        if self.segments == 0:
            return 0
        return self.segments - 1 if self.periodic else self.segments

    def index_count(self):
        return self.max_index() + 1

    def angle(self, index):
        return self.w_min + self.step * float(index)


class AngularGrid:
    """angular_grid.hpp:65-125: AngularGrid(cfg, d_max)."""

    def __init__(self, cfg: SearchConfig, d_max: float):
        self.cfg = cfg
        self.d_max = float(d_max)
        n = 3 * (cfg.max_level + 1)
        out = (AxisGridC * n)()
        c = cfg.to_c()
        _check(lib.bbs_angular_grid(C.byref(c), self.d_max, out, n))
        self._axes = [AxisGrid(g.w_min, g.w_max, g.step, g.segments, bool(g.periodic)) for g in out]
        self._max_level = cfg.max_level

    def max_level(self):
        return self._max_level

    def axis(self, axis, level):
        return self._axes[axis * (self._max_level + 1) + level]

    def divisions(self, axis, level):
        parent, child = self.axis(axis, level), self.axis(axis, level - 1)
        if child.segments <= 1:
            return 1
        return (child.segments + parent.segments - 1) // parent.segments


NODE_DTYPE = np.dtype([(f, np.int32) for f in _abi.NODE_DTYPE_FIELDS])


def node_pose(node, grids: AngularGrid, min_resolution):
    """nodes.hpp:33-43."""
    ix, iy, iz, ir, ip, iw, level = (int(v) for v in list(node)[:7])
    cell = math.ldexp(min_resolution, level)
    return Pose6(cell * float(ix), cell * float(iy), cell * float(iz),
                 grids.axis(0, level).angle(ir), grids.axis(1, level).angle(ip),
                 grids.axis(2, level).angle(iw))


def initial_node_count(cfg: SearchConfig, d_max, rng):
    """len(initial_nodes(...)), nodes.hpp:60-85."""
    c = cfg.to_c()
    b = Aabb()
    (b.min.x, b.min.y, b.min.z), (b.max.x, b.max.y, b.max.z) = rng
    out = C.c_uint64()
    _check(lib.bbs_initial_node_count(C.byref(c), float(d_max), C.byref(b), C.byref(out)))
    return out.value


def _nodes_array(nodes):
    a = np.asarray(nodes)
    if a.dtype == NODE_DTYPE:
        a = a.view(np.int32).reshape(-1, 8)
    return np.ascontiguousarray(a.astype(np.int32, copy=False).reshape(-1, 8))


# ---- voxel map (voxel_map.hpp) ----------------------------------------------
class LevelMap:
    """One level of a device map (voxel_map.hpp:57-180)."""

    def __init__(self, parent, level):
        self._m = parent
        self._level = level
        info = LevelInfo()
        _check(lib.bbs_map_level_info(parent._h, level, C.byref(info)))
        self._info = info

    def level(self):
        return self._level

    def resolution(self):
        return self._info.resolution

    def occupied_count(self):
        return self._info.occupied_count

    def bucket_count(self):
        return self._info.bucket_count

    def collision_rate(self):
        return self._info.collision_rate

    def load_factor(self):
        return self._info.load_factor

    def layout(self):
        return Layout(self._info.layout)

    def device_bytes(self):
        return self._info.bytes

    def occupied_voxels(self):
        """Ascending (x, y, z), voxel_map.hpp:158-165 -> (n, 3) int32."""
        n = C.c_uint64()
        _check(lib.bbs_level_occupied(self._m._h, self._level, None, 0, C.byref(n)))
        out = np.zeros((n.value, 3), np.int32)
        if n.value:
            _check(lib.bbs_level_occupied(self._m._h, self._level,
                                          out.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                          C.byref(n)))
        return out

    def contains_many(self, voxels):
        v = np.ascontiguousarray(np.asarray(voxels, np.int32).reshape(-1, 3))
        out = np.zeros(v.shape[0], np.uint8)
        if v.shape[0]:
            _check(lib.bbs_level_contains(self._m._h, self._level,
                                          v.ctypes.data_as(C.POINTER(C.c_int32)), v.shape[0],
                                          out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.astype(bool)

    def contains(self, v):
        """voxel_map.hpp:127-135."""
        return bool(self.contains_many([v])[0])

    def score(self, transform, scan):
        """voxel_map.hpp:142-154; transform = (rotation[9] row-major, translation[3])."""
        R, t = transform
        Ra = np.ascontiguousarray(np.asarray(R, np.float64).ravel())
        ta = np.ascontiguousarray(np.asarray(t, np.float64).ravel())
        s = _xyz(scan)
        out = C.c_int32()
        _check(lib.bbs_level_score(self._m._h, self._level, _dptr(Ra), _dptr(ta), _dptr(s),
                                   s.shape[0], C.byref(out)))
        return out.value


class MultiResVoxelMap:
    """voxel_map.hpp:220-274, device-resident."""

    kDefaultCollisionTarget = 0.001
    kDefaultMemoryCapBytes = 2 << 30

    def __init__(self, handle):
        self._h = handle
        r, ml = C.c_double(), C.c_int32()
        _check(lib.bbs_map_min_resolution(self._h, C.byref(r)))
        _check(lib.bbs_map_max_level(self._h, C.byref(ml)))
        self._r, self._max_level = r.value, ml.value
        self._levels = [LevelMap(self, l) for l in range(self._max_level + 1)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.bbs_map_free(h)
            self._h = None

    @staticmethod
    def build(map_points, min_resolution, max_level, collision_target=0.001,
              memory_cap_bytes=2 << 30, layout=Layout.AUTO, device=0):
        """voxel_map.hpp:226-244."""
        a = _xyz(map_points)
        h = C.c_void_p()
        opts = MapOptions(int(device), int(layout))
        _check(lib.bbs_map_build(_dptr(a), a.shape[0], float(min_resolution), int(max_level),
                                 float(collision_target), int(memory_cap_bytes), C.byref(opts),
                                 C.byref(h)))
        return MultiResVoxelMap(h)

    @staticmethod
    def from_levels(per_level, min_resolution, bbox, collision_target=0.001,
                    memory_cap_bytes=2 << 30, layout=Layout.AUTO, device=0):
        """voxel_map.hpp:247-261; bbox = ((min), (max))."""
        arrs = [np.ascontiguousarray(np.asarray(v, np.int32).reshape(-1, 3)) for v in per_level]
        n = len(arrs)
        ptrs = (C.POINTER(C.c_int32) * max(n, 1))(
            *[a.ctypes.data_as(C.POINTER(C.c_int32)) for a in arrs])
        counts = (C.c_uint64 * max(n, 1))(*[a.shape[0] for a in arrs])
        b = Aabb()
        (b.min.x, b.min.y, b.min.z), (b.max.x, b.max.y, b.max.z) = bbox
        h = C.c_void_p()
        opts = MapOptions(int(device), int(layout))
        _check(lib.bbs_map_from_levels(ptrs, counts, n, float(min_resolution), C.byref(b),
                                       float(collision_target), int(memory_cap_bytes),
                                       C.byref(opts), C.byref(h)))
        return MultiResVoxelMap(h)

    def save(self, path):
        """save_map, map_io.hpp:44-65."""
        _check(lib.bbs_map_save(self._h, os.fsencode(path)))

    def min_resolution(self):
        return self._r

    def max_level(self):
        return self._max_level

    def bbox(self):
        b = Aabb()
        _check(lib.bbs_map_bbox(self._h, C.byref(b)))
        return (b.min.x, b.min.y, b.min.z), (b.max.x, b.max.y, b.max.z)

    def level(self, l):
        return self._levels[l]

    def levels(self):
        return list(self._levels)

    def set_stream(self, stream_ptr):
        """Run later work on an external cudaStream_t (int pointer, 0 = own)."""
        _check(lib.bbs_map_set_stream(self._h, C.c_void_p(int(stream_ptr) or None)))

    def build_ms(self):
        out = C.c_double()
        _check(lib.bbs_map_build_ms(self._h, C.byref(out)))
        return out.value


def save_map(vmap: MultiResVoxelMap, path):
    """save_map, map_io.hpp:44-65 (byte-identical to the reference's file)."""
    vmap.save(path)


def load_map(path, collision_target=0.001, memory_cap_bytes=2 << 30, layout=Layout.AUTO, device=0):
    """load_map, map_io.hpp:67-115: the reference's map file straight into
    device levels (format errors are raised before any device work)."""
    h = C.c_void_p()
    opts = MapOptions(int(device), int(layout))
    _check(lib.bbs_map_load(os.fsencode(path), float(collision_target), int(memory_cap_bytes),
                            C.byref(opts), C.byref(h)))
    return MultiResVoxelMap(h)


def is_map_file(path) -> bool:
    """is_map_file, map_io.hpp:119-126."""
    return bool(lib.bbs_is_map_file(os.fsencode(path)))


class DeviceScan:
    """A scan uploaded once to the map's GPU (SoA doubles in HBM)."""

    def __init__(self, vmap: MultiResVoxelMap, scan):
        a = _xyz(scan)
        self._map = vmap
        self.k = a.shape[0]
        self._h = C.c_void_p()
        _check(lib.bbs_scan_upload(vmap._h, _dptr(a), a.shape[0], C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.bbs_scan_free(h)
            self._h = None


# ---- search (search.hpp, pipeline.hpp) --------------------------------------
def batch_evaluate(nodes, vmap: MultiResVoxelMap, scan, grids: AngularGrid, workers=1):
    """search.hpp:23-34.  Returns the nodes (n, 8) int32 with scores filled;
    a writable contiguous int32 (n, 8) input is also updated in place."""
    arr = _nodes_array(nodes)
    s = _xyz(scan)
    c = grids.cfg.to_c()
    if arr.shape[0]:
        _check(lib.bbs_batch_evaluate(vmap._h, _dptr(s), s.shape[0], C.byref(c), grids.d_max,
                                      arr.ctypes.data_as(C.POINTER(Node)), arr.shape[0]))
    if isinstance(nodes, np.ndarray) and nodes.dtype == np.int32 and nodes.flags.c_contiguous \
            and nodes.shape == arr.shape and nodes is not arr:
        nodes[...] = arr
    return arr


def search(vmap: MultiResVoxelMap, scan, cfg: SearchConfig, trace_capacity=1 << 16):
    """search.hpp:72-186 (host scan buffer in, result out)."""
    s = _xyz(scan)
    res, buf = _new_result(trace_capacity if cfg.collect_trace else 0)
    c = cfg.to_c()
    _check(lib.bbs_search(vmap._h, _dptr(s), s.shape[0], C.byref(c), C.byref(res)))
    return _result_from_c(res, buf)


ORACLE_MAX_LEAVES = 100_000_000  # kOracleMaxLeaves, oracle.hpp:25


@dataclass
class OracleResult:
    """oracle.hpp:17-21 (plus the argmax leaves as (n, 8) int32 nodes)."""
    best_score: int
    argmax_poses: list
    leaf_count: int
    argmax_nodes: np.ndarray


def oracle_search(vmap: MultiResVoxelMap, scan, cfg: SearchConfig, argmax_capacity=None):
    """oracle.hpp:29-95: every level-0 leaf under the root index ranges x the
    level-0 rotation grid, enumerated and scored on the device (no pruning),
    in one pass (bbs_oracle_search_all); argmax_capacity (optional) takes the
    capped bbs_oracle_search entry point instead."""
    s = _xyz(scan)
    c = cfg.to_c()
    best, cnt, leaves = C.c_int32(), C.c_uint64(), C.c_uint64()
    if argmax_capacity is not None:
        cap = max(int(argmax_capacity), 1)
        buf = np.zeros((cap, 8), np.int32)
        _check(lib.bbs_oracle_search(vmap._h, _dptr(s), s.shape[0], C.byref(c), C.byref(best),
                                     buf.ctypes.data_as(C.POINTER(Node)), cap, C.byref(cnt),
                                     C.byref(leaves)))
        nodes = buf[:min(cnt.value, cap)].copy()
    else:
        p = C.POINTER(Node)()
        _check(lib.bbs_oracle_search_all(vmap._h, _dptr(s), s.shape[0], C.byref(c), C.byref(best),
                                         C.byref(p), C.byref(cnt), C.byref(leaves)))
        try:
            nodes = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int32)),
                                          shape=(max(cnt.value, 1), 8))[:cnt.value].copy()
        finally:
            lib.bbs_free(C.cast(p, C.c_void_p))
    d_max = cfg.d_max if cfg.d_max is not None else max_range(s)
    grids = AngularGrid(cfg, d_max)
    poses = [node_pose(n, grids, cfg.min_resolution).normalized() for n in nodes]
    return OracleResult(int(best.value), poses, int(leaves.value), nodes)


class DeviceStream:
    """A non-blocking CUDA stream owned by the library (concurrent searches)."""

    def __init__(self, device=0):
        self._h = C.c_void_p()
        _check(lib.bbs_stream_create(int(device), C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.bbs_stream_destroy(h)
            self._h = None


def search_scan(vmap: MultiResVoxelMap, dscan: DeviceScan, cfg: SearchConfig,
                trace_capacity=1 << 16, stream=None):
    """search() on a device-resident scan (no host copy inside the call).
    `stream`: a DeviceStream or a raw cudaStream_t (int); searches on
    different streams run concurrently."""
    res, buf = _new_result(trace_capacity if cfg.collect_trace else 0)
    c = cfg.to_c()
    if stream is None:
        _check(lib.bbs_search_scan(vmap._h, dscan._h, C.byref(c), C.byref(res)))
    else:
        sp = stream._h if isinstance(stream, DeviceStream) else C.c_void_p(int(stream))
        _check(lib.bbs_search_scan_on(vmap._h, dscan._h, C.byref(c), sp, C.byref(res)))
    return _result_from_c(res, buf)


@dataclass
class SearchDumpResult:
    """What the device scored inside one search (bbs_search_scan_dump)."""
    result: "SearchResult"
    root_scores: np.ndarray       # int32, initial_nodes() order
    flush_nodes: np.ndarray       # (n, 8) int32, every dumped flush batch
    flush_scores: np.ndarray      # int32 device scores of flush_nodes
    epoch_offsets: np.ndarray     # batch i = [off[i], off[i+1])
    epoch_ids: np.ndarray         # flush index of batch i


def search_scan_dump(vmap: MultiResVoxelMap, dscan: DeviceScan, cfg: SearchConfig, exact_roots=False,
                     epoch_stride=1, root_capacity=1 << 24, flush_capacity=1 << 22,
                     epoch_capacity=1 << 16, trace_capacity=1 << 16) -> SearchDumpResult:
    """search() with the root batch and flushed batches copied out
    (parity instrumentation; one epoch per host check, no graphs)."""
    res, buf = _new_result(trace_capacity if cfg.collect_trace else 0)
    c = cfg.to_c()
    roots = np.zeros(root_capacity, np.int32)
    fn = np.zeros((flush_capacity, 8), np.int32)
    fs = np.zeros(flush_capacity, np.int32)
    off = np.zeros(epoch_capacity + 1, np.uint64)
    ids = np.zeros(epoch_capacity, np.uint32)
    d = _abi.SearchDump()
    d.exact_roots = 1 if exact_roots else 0
    d.epoch_stride = int(epoch_stride)
    d.root_scores = roots.ctypes.data_as(C.POINTER(C.c_int32))
    d.root_capacity = root_capacity
    d.flush_nodes = fn.ctypes.data_as(C.POINTER(Node))
    d.flush_scores = fs.ctypes.data_as(C.POINTER(C.c_int32))
    d.flush_capacity = flush_capacity
    d.epoch_offsets = off.ctypes.data_as(C.POINTER(C.c_uint64))
    d.epoch_ids = ids.ctypes.data_as(C.POINTER(C.c_uint32))
    d.epoch_capacity = epoch_capacity
    _check(lib.bbs_search_scan_dump(vmap._h, dscan._h, C.byref(c), C.byref(d), C.byref(res)))
    if d.root_count > root_capacity or d.flush_count > flush_capacity or d.epoch_count > epoch_capacity:
        raise InvalidArgumentError(f"search_scan_dump: capacity exceeded (roots {d.root_count}, "
                                   f"flush {d.flush_count}, epochs {d.epoch_count})")
    ne = int(d.epoch_count)
    return SearchDumpResult(_result_from_c(res, buf), roots[:d.root_count].copy(),
                            fn[:d.flush_count].copy(), fs[:d.flush_count].copy(),
                            off[:ne + 1].astype(np.int64), ids[:ne].copy())


def search_scans(vmap: MultiResVoxelMap, dscans, cfg: SearchConfig, concurrency=16, trace_capacity=0):
    """Throughput mode (bbs_search_scans): search() for every device scan,
    `concurrency` searches in flight on native threads / streams."""
    n = len(dscans)
    arr = (SearchResultC * max(n, 1))()
    bufs = []
    for i in range(n):
        if cfg.collect_trace and trace_capacity:
            b = (C.c_int32 * trace_capacity)()
            arr[i].best_score_trace = C.cast(b, C.POINTER(C.c_int32))
            arr[i].trace_capacity = trace_capacity
            bufs.append(b)
        else:
            bufs.append(None)
    handles = (C.c_void_p * max(n, 1))(*[d._h for d in dscans])
    c = cfg.to_c()
    _check(lib.bbs_search_scans(vmap._h, handles, n, C.byref(c), int(concurrency), arr))
    return [_result_from_c(arr[i], bufs[i]) for i in range(n)]


class Comm:
    """NCCL communicator for the device-side exchanges of a sharded search
    (bbs_comm_t).  Rank 0 draws ``Comm.unique_id()``; every rank builds
    ``Comm(device, rank, world, uid)`` collectively."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib.bbs_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, device: int, rank: int, world: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self._h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib.bbs_comm_init(int(device), int(rank), int(world), buf, C.byref(self._h)))
        self.rank, self.world = int(rank), int(world)

    def close(self):
        if self._h:
            lib.bbs_comm_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def nccl_version() -> int:
    """Version of the NCCL the library loads (0 when none can be loaded)."""
    return int(lib.bbs_nccl_version())


def search_sharded(vmap: MultiResVoxelMap, dscan: DeviceScan, cfg: SearchConfig, rank, world,
                   allreduce_max=None, trace_capacity=1 << 16, mode="roots",
                   comm: Optional[Comm] = None):
    """Sharded search (include/bbs.h bbs_search_sharded).

    mode "roots": each rank runs its own BnB over its root share, the
    incumbent is max-all-reduced every epoch and the winner elected.
    mode "exact": batch-split replay of the single-queue schedule; every rank
    returns the unsharded search() result.
    Exchanges go through ``comm`` (NCCL on the device) when given, else
    through ``allreduce_max(list_of_int64) -> element-wise max over ranks``
    (e.g. torch.distributed all_reduce MAX on the host)."""
    if mode not in ("roots", "exact"):
        raise ValueError(f"unknown shard mode {mode!r}")
    cb = _abi.ALLREDUCE_MAX_FN()
    if allreduce_max is not None:
        def _cb(values, count, _user):
            try:
                vals = [values[i] for i in range(count)]
                out = allreduce_max(vals)
                for i in range(count):
                    values[i] = int(out[i])
                return 0
            except Exception:  # noqa: BLE001 - reported through the status code
                return 1
        cb = _abi.ALLREDUCE_MAX_FN(_cb)
    shard = Shard(int(rank), int(world), cb, None,
                  _abi.SHARD_EXACT if mode == "exact" else _abi.SHARD_ROOTS, 0,
                  comm._h if comm is not None else None)
    res, buf = _new_result(trace_capacity if cfg.collect_trace else 0)
    c = cfg.to_c()
    _check(lib.bbs_search_sharded(vmap._h, dscan._h, C.byref(c), C.byref(shard), C.byref(res)))
    return _result_from_c(res, buf)


def localize_scan(vmap: MultiResVoxelMap, raw_scan, cfg: SearchConfig, downsample_target,
                  trace_capacity=1 << 16, prepare="exact"):
    """pipeline.hpp:45-51.  prepare="exact" (default): centroids in the
    reference's summation order, bit-identical to the reference;
    "device": centroids summed on the device (faster, last-bit differences
    possible for voxels of >= 3 points)."""
    if prepare not in ("exact", "device"):
        raise ValueError(f"unknown prepare mode {prepare!r}")
    s = _xyz(raw_scan)
    res, buf = _new_result(trace_capacity if cfg.collect_trace else 0)
    c = cfg.to_c()
    _check(lib.bbs_localize_scan_ex(vmap._h, _dptr(s), s.shape[0], C.byref(c), int(downsample_target),
                                    0 if prepare == "exact" else 1, C.byref(res)))
    return _result_from_c(res, buf)


