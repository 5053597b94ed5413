"""ctypes mirror of include/bbs.h (the C-ABI boundary).

Struct layouts here must match include/bbs.h byte for byte;
tests/test_abi.py checks the sizes against the compiled library.
"""
import ctypes as C

BBS_OK = 0
STATUS_NAMES = {
    1: "Error", 2: "FileNotFoundError", 3: "ParseError", 4: "EmptyCloudError",
    5: "CapacityExceededError", 6: "IoError", 7: "FormatError",
    8: "DegenerateScanError", 9: "EmptySearchSpaceError", 10: "TooLargeError",
    11: "InfeasiblePoseError", 12: "ConfigError", 13: "CudaError",
    14: "InvalidArgumentError",
}

STRATEGY_DFS, STRATEGY_BFS = 0, 1
BRANCH_TRANS_ONLY, BRANCH_ROTO_TRANS = 0, 1
LAYOUT_AUTO, LAYOUT_BITMAP, LAYOUT_HASH = 0, 1, 2
TWO_PI = 6.283185307179586476925286766559


class Point3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class Pose6(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("x", "y", "z", "roll", "pitch", "yaw")]

    def as_tuple(self):
        return (self.x, self.y, self.z, self.roll, self.pitch, self.yaw)


class Aabb(C.Structure):
    _fields_ = [("min", Point3), ("max", Point3)]


class Node(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("ix", "iy", "iz", "iroll", "ipitch", "iyaw", "level", "score")]


class SearchConfigC(C.Structure):
    _fields_ = [
        ("min_resolution", C.c_double),
        ("max_level", C.c_int32),
        ("has_translation_range", C.c_int32),
        ("translation_range", Aabb),
        ("roll_pitch_half_range", C.c_double),
        ("yaw_min", C.c_double),
        ("yaw_max", C.c_double),
        ("score_threshold_fraction", C.c_double),
        ("batch_size", C.c_uint64),
        ("strategy", C.c_int32),
        ("branch_mode", C.c_int32),
        ("workers", C.c_int32),
        ("has_d_max", C.c_int32),
        ("d_max", C.c_double),
        ("collect_trace", C.c_int32),
    ]


class StatsC(C.Structure):
    _fields_ = [
        ("nodes_generated", C.c_uint64),
        ("nodes_pruned", C.c_uint64),
        ("batches_flushed", C.c_uint64),
        ("create_voxel_maps_ms", C.c_double),
        ("set_source_ms", C.c_double),
        ("initial_nodes_ms", C.c_double),
        ("find_best_score_ms", C.c_double),
        ("pop_remaining_queue_ms", C.c_double),
    ]


class SearchResultC(C.Structure):
    _fields_ = [
        ("best_pose", Pose6),
        ("best_score", C.c_int32),
        ("score_threshold", C.c_int32),
        ("scan_points", C.c_uint64),
        ("matched", C.c_int32),
        ("stats", StatsC),
        ("best_score_trace", C.POINTER(C.c_int32)),
        ("trace_capacity", C.c_uint64),
        ("trace_length", C.c_uint64),
        ("best_node", Node),
        ("epochs", C.c_uint64),
        ("lookups", C.c_uint64),
        ("device_ms", C.c_double),
        ("root_score_ms", C.c_double),
        ("epoch_score_ms", C.c_double),
        ("root_nodes", C.c_uint64),
        ("queue_peak", C.c_uint64),
        ("root_probes", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("evals_per_level", C.c_uint64 * 16),
        ("root_words", C.c_uint64),
        ("root_col_ms", C.c_double),
        ("group_checks", C.c_uint64),
    ]


class AxisGridC(C.Structure):
    _fields_ = [
        ("w_min", C.c_double), ("w_max", C.c_double), ("step", C.c_double),
        ("segments", C.c_int32), ("periodic", C.c_int32),
    ]


class MapOptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("layout", C.c_int32)]


class LevelInfo(C.Structure):
    _fields_ = [
        ("level", C.c_int32),
        ("layout", C.c_int32),
        ("resolution", C.c_double),
        ("occupied_count", C.c_uint64),
        ("bucket_count", C.c_uint64),
        ("collision_rate", C.c_double),
        ("load_factor", C.c_double),
        ("bytes", C.c_uint64),
        ("box_min", C.c_int32 * 3),
        ("box_max", C.c_int32 * 3),
    ]


ALLREDUCE_MAX_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_int64), C.c_int32, C.c_void_p)


class Shard(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("world_size", C.c_int32),
        ("allreduce_max", ALLREDUCE_MAX_FN),
        ("user", C.c_void_p),
        ("mode", C.c_int32),
        ("reserved", C.c_int32),
        ("comm", C.c_void_p),
    ]


class SearchDump(C.Structure):
    """bbs_search_dump (parity instrumentation)."""
    _fields_ = [
        ("exact_roots", C.c_int32),
        ("epoch_stride", C.c_uint32),
        ("root_scores", C.POINTER(C.c_int32)),
        ("root_capacity", C.c_uint64),
        ("root_count", C.c_uint64),
        ("flush_nodes", C.POINTER(Node)),
        ("flush_scores", C.POINTER(C.c_int32)),
        ("flush_capacity", C.c_uint64),
        ("flush_count", C.c_uint64),
        ("epoch_offsets", C.POINTER(C.c_uint64)),
        ("epoch_ids", C.POINTER(C.c_uint32)),
        ("epoch_capacity", C.c_uint64),
        ("epoch_count", C.c_uint64),
    ]


SHARD_ROOTS = 0  # BBS_SHARD_ROOTS: own BnB per rank over its root share
SHARD_EXACT = 1  # BBS_SHARD_EXACT: batch-split replay of the single-queue schedule


NODE_DTYPE_FIELDS = ("ix", "iy", "iz", "iroll", "ipitch", "iyaw", "level", "score")
