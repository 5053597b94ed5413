"""Synthetic-input harness (NOT the product, NOT the oracle).

ctypes wrapper of harness/libbbs_scene.so: a bit-identical restatement of the
reference's box-world generator gen_scene (scene.hpp:156-220), the C4 helper
that renders extra scans of one map, and the seeded Fisher-Yates cut to K
points.  Used by bench.py's B200 arm and the tests to build the
same doubles the reference consumes; tests/test_host.py pins it to the
reference's own gen_scene (oracle/_ref).
"""
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbbs_scene.so")

_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64


class SceneSpec(C.Structure):
    """SceneSpec, scene.hpp:21-38 (defaults from hs_scene_spec_default)."""
    _fields_ = [
        ("size_x", C.c_double), ("size_y", C.c_double), ("size_z", C.c_double),
        ("num_boxes", C.c_int32),
        ("min_box_side", C.c_double), ("max_box_side", C.c_double),
        ("min_box_height", C.c_double),
        ("map_spacing", C.c_double), ("scan_spacing", C.c_double),
        ("scan_range", C.c_double), ("point_jitter", C.c_double),
        ("tilt_noise", C.c_int32),
        ("gt_yaw_min", C.c_double), ("gt_yaw_max", C.c_double),
        ("min_scan_points", C.c_uint64),
        ("feasibility_resolution", C.c_double),
    ]

    @staticmethod
    def default(**kw):
        s = SceneSpec()
        _lib().hs_scene_spec_default(C.byref(s))
        for k, v in kw.items():
            setattr(s, k, v)
        return s


@dataclass
class Pose:
    """Ground-truth pose (Pose6, geometry.hpp:46)."""
    x: float
    y: float
    z: float
    roll: float
    pitch: float
    yaw: float

    def as_tuple(self):
        return (self.x, self.y, self.z, self.roll, self.pitch, self.yaw)


class SceneError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C harness)")
        L = C.CDLL(LIB_PATH)
        L.hs_scene_spec_default.argtypes = [C.c_void_p]
        L.hs_scene_spec_default.restype = None
        L.hs_gen_scene.argtypes = [C.c_void_p, _u64, C.POINTER(_dp), C.POINTER(_u64), C.POINTER(_dp),
                                   C.POINTER(_u64), _dp]
        L.hs_gen_scans.argtypes = [C.c_void_p, _u64, _u64, C.c_int32, C.POINTER(_dp),
                                   C.POINTER(_u64), _dp]
        L.hs_cut_scan.argtypes = [_dp, _u64, _u64, _u64, _dp]
        L.hs_last_error.restype = C.c_char_p
        L.hs_free.argtypes = [C.c_void_p]
        L.hs_free.restype = None
        _LIB = L
    return _LIB


def _check(st):
    if st != 0:
        raise SceneError(st, _lib().hs_last_error().decode())


def gen_scene(spec: SceneSpec, seed):
    """scene.hpp:156-220 -> (map (n,3), scan (k,3), gt Pose)."""
    L = _lib()
    mp, sp = _dp(), _dp()
    nm, ns = C.c_uint64(), C.c_uint64()
    gt = (C.c_double * 6)()
    _check(L.hs_gen_scene(C.byref(spec), int(seed), C.byref(mp), C.byref(nm), C.byref(sp),
                          C.byref(ns), gt))
    m = np.ctypeslib.as_array(mp, shape=(nm.value, 3)).copy()
    s = np.ctypeslib.as_array(sp, shape=(ns.value, 3)).copy()
    L.hs_free(C.cast(mp, C.c_void_p))
    L.hs_free(C.cast(sp, C.c_void_p))
    return m, s, Pose(*gt)


def gen_scans(spec: SceneSpec, seed, pose_seed_base, n_scans):
    """Extra scans of seed's map (C4 helper) -> (list of (k,3), list of Pose)."""
    L = _lib()
    sp = _dp()
    offs = (C.c_uint64 * (n_scans + 1))()
    gt = (C.c_double * (6 * max(n_scans, 1)))()
    _check(L.hs_gen_scans(C.byref(spec), int(seed), int(pose_seed_base), int(n_scans),
                          C.byref(sp), offs, gt))
    allp = np.ctypeslib.as_array(sp, shape=(max(offs[n_scans], 1), 3)).copy()
    L.hs_free(C.cast(sp, C.c_void_p))
    scans = [allp[offs[j]:offs[j + 1]].copy() for j in range(n_scans)]
    return scans, [Pose(*gt[6 * j:6 * j + 6]) for j in range(n_scans)]


def cut_scan(scan, k, seed):
    """First k points of a Fisher-Yates shuffle driven by Rng(seed)."""
    a = np.ascontiguousarray(np.asarray(scan, dtype=np.float64).reshape(-1, 3))
    k = int(k)
    out = np.zeros((k, 3))
    _check(_lib().hs_cut_scan(a.ctypes.data_as(_dp), a.shape[0], k, int(seed), out.ctypes.data_as(_dp)))
    return out


def cut_scan_py(scan, k, seed):
    """Pure-Python cut_scan (same splitmix64 Fisher-Yates): for the reference
    arm of bench.py, which must not load any library of this repo."""
    mask = (1 << 64) - 1
    state = seed & mask
    n = scan.shape[0]
    idx = list(range(n))
    for i in range(k):
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z ^= z >> 31
        j = i + z % (n - i)
        idx[i], idx[j] = idx[j], idx[i]
    return scan[idx[:k]].copy()
