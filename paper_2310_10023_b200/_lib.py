"""Loads libbbs_b200.so (the C-ABI of include/bbs.h) and declares signatures.

The library is built in-tree by ``make -C paper_2310_10023_b200/csrc``
(``__graft_entry__.build()``).  There is no fallback: importing the package
without the library raises, and every compute entry point fails loudly
(BBS_ERR_CUDA) when no GPU is present.
"""
import ctypes as C
import os

from ._abi import (
    Aabb, AxisGridC, LevelInfo, MapOptions, Node, SearchConfigC, SearchDump, SearchResultC,
    Shard,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbbs_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {HERE}/csrc` "
        "(or __graft_entry__.build()); the B200 path has no Python/CPU fallback")

lib = C.CDLL(LIB_PATH)

_d = C.c_double
_u64 = C.c_uint64
_i32 = C.c_int32
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)

SIGNATURES = {
    # name: (restype, argtypes)
    "bbs_last_error": (C.c_char_p, []),
    "bbs_abi_version": (C.c_int, []),
    "bbs_device_count": (C.c_int, []),
    "bbs_search_config_default": (None, [C.POINTER(SearchConfigC)]),
    "bbs_angular_grid": (C.c_int, [C.POINTER(SearchConfigC), _d, C.POINTER(AxisGridC), _u64]),
    "bbs_angular_divisions": (C.c_int, [C.POINTER(SearchConfigC), _d, _i32, _i32, _ip]),
    "bbs_max_range": (C.c_int, [_dp, _u64, _dp]),
    "bbs_bounding_box": (C.c_int, [_dp, _u64, C.POINTER(Aabb)]),
    "bbs_prepare_source": (C.c_int, [_dp, _u64, _u64, _dp, _u64, C.POINTER(_u64), _dp, _ip, _dp]),
    "bbs_prepare_source_device": (C.c_int, [_i32, _dp, _u64, _u64, _dp, _u64, C.POINTER(_u64), _dp, _ip,
                                            _dp]),
    "bbs_initial_node_count": (C.c_int, [C.POINTER(SearchConfigC), _d, C.POINTER(Aabb),
                                         C.POINTER(_u64)]),
    "bbs_map_build": (C.c_int, [_dp, _u64, _d, _i32, _d, _u64, C.POINTER(MapOptions),
                                C.POINTER(_vp)]),
    "bbs_map_from_levels": (C.c_int, [C.POINTER(_ip), C.POINTER(_u64), _i32, _d, C.POINTER(Aabb),
                                      _d, _u64, C.POINTER(MapOptions), C.POINTER(_vp)]),
    "bbs_map_free": (C.c_int, [_vp]),
    "bbs_map_load": (C.c_int, [C.c_char_p, _d, _u64, C.POINTER(MapOptions), C.POINTER(_vp)]),
    "bbs_map_save": (C.c_int, [_vp, C.c_char_p]),
    "bbs_is_map_file": (C.c_int, [C.c_char_p]),
    "bbs_map_min_resolution": (C.c_int, [_vp, _dp]),
    "bbs_map_max_level": (C.c_int, [_vp, _ip]),
    "bbs_map_bbox": (C.c_int, [_vp, C.POINTER(Aabb)]),
    "bbs_map_build_ms": (C.c_int, [_vp, _dp]),
    "bbs_map_set_stream": (C.c_int, [_vp, _vp]),
    "bbs_map_level_info": (C.c_int, [_vp, _i32, C.POINTER(LevelInfo)]),
    "bbs_level_occupied": (C.c_int, [_vp, _i32, _ip, _u64, C.POINTER(_u64)]),
    "bbs_level_contains": (C.c_int, [_vp, _i32, _ip, _u64, C.POINTER(C.c_uint8)]),
    "bbs_level_score": (C.c_int, [_vp, _i32, _dp, _dp, _dp, _u64, _ip]),
    "bbs_batch_evaluate": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), _d,
                                     C.POINTER(Node), _u64]),
    "bbs_search": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), C.POINTER(SearchResultC)]),
    "bbs_oracle_search": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), _ip,
                                    C.POINTER(Node), _u64, C.POINTER(_u64), C.POINTER(_u64)]),
    "bbs_oracle_search_all": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), _ip,
                                        C.POINTER(C.POINTER(Node)), C.POINTER(_u64), C.POINTER(_u64)]),
    "bbs_free": (None, [_vp]),
    "bbs_localize_scan_ex": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), _u64, _i32,
                                       C.POINTER(SearchResultC)]),
    "bbs_localize_scan": (C.c_int, [_vp, _dp, _u64, C.POINTER(SearchConfigC), _u64,
                                    C.POINTER(SearchResultC)]),
    "bbs_scan_upload": (C.c_int, [_vp, _dp, _u64, C.POINTER(_vp)]),
    "bbs_scan_free": (C.c_int, [_vp]),
    "bbs_search_scan": (C.c_int, [_vp, _vp, C.POINTER(SearchConfigC), C.POINTER(SearchResultC)]),
    "bbs_search_scan_dump": (C.c_int, [_vp, _vp, C.POINTER(SearchConfigC), C.POINTER(SearchDump),
                                       C.POINTER(SearchResultC)]),
    "bbs_batch_evaluate_device": (C.c_int, [_vp, _vp, C.POINTER(SearchConfigC), _d, _vp, _u64,
                                            _vp]),
    "bbs_search_scan_on": (C.c_int, [_vp, _vp, C.POINTER(SearchConfigC), _vp,
                                     C.POINTER(SearchResultC)]),
    "bbs_search_scans": (C.c_int, [_vp, C.POINTER(_vp), _u64, C.POINTER(SearchConfigC), _i32,
                                   C.POINTER(SearchResultC)]),
    "bbs_stream_create": (C.c_int, [_i32, C.POINTER(_vp)]),
    "bbs_stream_destroy": (C.c_int, [_vp]),
    "bbs_search_sharded": (C.c_int, [_vp, _vp, C.POINTER(SearchConfigC), C.POINTER(Shard),
                                     C.POINTER(SearchResultC)]),
    "bbs_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "bbs_comm_init": (C.c_int, [_i32, _i32, _i32, C.POINTER(C.c_uint8), C.POINTER(_vp)]),
    "bbs_comm_free": (C.c_int, [_vp]),
    "bbs_nccl_version": (C.c_int, []),
    "bbs_gather_bench": (C.c_int, [_i32, _u64, _dp]),
    "bbs_smem_bench": (C.c_int, [_i32, _dp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

ABI_VERSION = 5  # include/bbs.h BBS_ABI_VERSION this mirror was written for
if lib.bbs_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI version {lib.bbs_abi_version()}, "
                      f"the Python mirror expects {ABI_VERSION}: rebuild the library")


def exported_symbols():
    return sorted(SIGNATURES)
