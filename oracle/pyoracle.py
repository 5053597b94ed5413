"""TEST INFRASTRUCTURE ONLY — Python bindings for the CPU checkers.

* ``Restated``: oracle/liboracle.so, the plain-C restatement of the
  reference path (oracle/bbs_oracle.c).
* ``Reference``: oracle/_ref/libbnbloc_ref.so, the UNMODIFIED reference
  headers (/root/reference/proj/include/bnbloc) behind a C shim
  (oracle/ref_shim.cpp), built here by oracle/Makefile and shipped prebuilt
  to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs may import this module, and only as the checker or the
timed CPU baseline — never as the product path.
"""
import ctypes as C
import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _load_abi_structs():
    """The C-ABI struct layouts (paper_2310_10023_b200/_abi.py: ctypes only),
    loaded by file path so that importing the checker never imports the
    product package (which would load libbbs_b200.so into the process)."""
    path = os.path.join(os.path.dirname(HERE), "paper_2310_10023_b200", "_abi.py")
    spec = importlib.util.spec_from_file_location("bbs_abi_structs", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


_abi = _load_abi_structs()
Aabb, AxisGridC, Node, SearchConfigC = _abi.Aabb, _abi.AxisGridC, _abi.Node, _abi.SearchConfigC
SearchResultC, Shard, STATUS_NAMES = _abi.SearchResultC, _abi.Shard, _abi.STATUS_NAMES

RESTATED_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libbnbloc_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.message = msg
        self.kind = STATUS_NAMES.get(code, str(code))


def _dptr(a):
    return a.ctypes.data_as(_dp)


def _xyz(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
    return a


class SceneSpec(C.Structure):
    """SceneSpec, scene.hpp:21-38."""
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


def nodes_to_array(nodes):
    """list/ndarray of 8-int rows -> contiguous (n, 8) int32."""
    return np.ascontiguousarray(np.asarray(nodes, dtype=np.int32).reshape(-1, 8))


class Reference:
    """The reference itself (oracle/_ref)."""

    def __init__(self, path=REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_map_build.argtypes = [_dp, C.c_uint64, C.c_double, C.c_int32, C.c_double,
                                    C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_map_free.argtypes = [C.c_void_p]
        L.ref_map_free.restype = None
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_free.restype = None
        L.ref_save_map.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_load_map.argtypes = [C.c_char_p, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_is_map_file.argtypes = [C.c_char_p]
        L.ref_map_max_level.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def default_spec(self):
        s = SceneSpec()
        self.lib.ref_scene_spec_default(C.byref(s))
        return s

    def gen_scene(self, spec, seed):
        mp, sp = _dp(), _dp()
        nm, ns = C.c_uint64(), C.c_uint64()
        gt = (C.c_double * 6)()
        self._check(self.lib.ref_gen_scene(C.byref(spec), C.c_uint64(seed), C.byref(mp),
                                           C.byref(nm), C.byref(sp), C.byref(ns), gt))
        m = np.ctypeslib.as_array(mp, shape=(nm.value, 3)).copy()
        s = np.ctypeslib.as_array(sp, shape=(ns.value, 3)).copy()
        self.lib.ref_free(mp)
        self.lib.ref_free(sp)
        return m, s, tuple(gt)

    def gen_scans(self, spec, seed, pose_seed_base, n_scans):
        """C4 harness helper (ref_gen_scans): seed's map layout, n_scans scans
        with poses from Rng(pose_seed_base + j).  Returns (list of (n,3)
        scans, list of gt 6-tuples)."""
        sp = _dp()
        offs = (C.c_uint64 * (n_scans + 1))()
        gt = (C.c_double * (6 * max(n_scans, 1)))()
        self._check(self.lib.ref_gen_scans(C.byref(spec), C.c_uint64(seed),
                                           C.c_uint64(pose_seed_base), C.c_int32(n_scans),
                                           C.byref(sp), offs, gt))
        allp = np.ctypeslib.as_array(sp, shape=(max(offs[n_scans], 1), 3)).copy()
        self.lib.ref_free(sp)
        scans = [allp[offs[j]:offs[j + 1]].copy() for j in range(n_scans)]
        return scans, [tuple(gt[6 * j:6 * j + 6]) for j in range(n_scans)]

    def map_build(self, pts, r, max_level, collision_target=0.001, cap=2 << 30):
        pts = _xyz(pts)
        h = C.c_void_p()
        self._check(self.lib.ref_map_build(_dptr(pts), pts.shape[0], r, max_level,
                                           collision_target, cap, C.byref(h)))
        return RefMap(self, h, max_level)

    def load_map(self, path, collision_target=0.001, cap=2 << 30):
        """load_map, map_io.hpp:67-115 (raises OracleError(status, message))."""
        h = C.c_void_p()
        self._check(self.lib.ref_load_map(os.fsencode(path), C.c_double(collision_target),
                                          C.c_uint64(cap), C.byref(h)))
        m = RefMap(self, h, 0)
        m.max_level = m.max_level_from_levels()
        return m

    def is_map_file(self, path):
        return bool(self.lib.ref_is_map_file(os.fsencode(path)))

    def map_from_levels(self, levels, r, bbox, collision_target=0.001, cap=2 << 30):
        arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int32).reshape(-1, 3)) for v in levels]
        ptrs = (C.POINTER(C.c_int32) * len(arrs))(*[a.ctypes.data_as(_ip) for a in arrs])
        counts = (C.c_uint64 * len(arrs))(*[a.shape[0] for a in arrs])
        h = C.c_void_p()
        self._check(self.lib.ref_map_from_levels(ptrs, counts, len(arrs), C.c_double(r),
                                                 C.byref(bbox), C.c_double(collision_target),
                                                 C.c_uint64(cap), C.byref(h)))
        return RefMap(self, h, len(arrs) - 1)

    def angular_grid(self, cfg, d_max):
        out = (AxisGridC * (3 * (cfg.max_level + 1)))()
        self._check(self.lib.ref_angular_grid(C.byref(cfg), C.c_double(d_max), out))
        return out

    def divisions(self, cfg, d_max, axis, level):
        o = C.c_int32()
        self._check(self.lib.ref_angular_divisions(C.byref(cfg), C.c_double(d_max), axis,
                                                   level, C.byref(o)))
        return o.value

    def node_pose(self, cfg, d_max, node):
        n = Node(*[int(v) for v in node])
        p = (C.c_double * 6)()
        self._check(self.lib.ref_node_pose(C.byref(cfg), C.c_double(d_max), C.byref(n), p))
        return tuple(p)

    def pose_to_transform(self, pose6):
        p = (C.c_double * 6)(*pose6)
        R = (C.c_double * 9)()
        t = (C.c_double * 3)()
        self.lib.ref_pose_to_transform(p, R, t)
        return np.array(R[:]), np.array(t[:])

    def initial_nodes(self, cfg, d_max, rng_aabb, cap=1 << 22):
        cnt = C.c_uint64()
        self._check(self.lib.ref_initial_nodes(C.byref(cfg), C.c_double(d_max),
                                               C.byref(rng_aabb), None, C.c_uint64(0),
                                               C.byref(cnt)))
        n = cnt.value
        out = np.zeros((n, 8), np.int32)
        self._check(self.lib.ref_initial_nodes(C.byref(cfg), C.c_double(d_max),
                                               C.byref(rng_aabb), out.ctypes.data_as(_ip),
                                               C.c_uint64(n), C.byref(cnt)))
        return out

    def branch(self, cfg, d_max, parent):
        p = Node(*[int(v) for v in parent])
        out = np.zeros((4096, 8), np.int32)
        cnt = C.c_uint64()
        self._check(self.lib.ref_branch(C.byref(cfg), C.c_double(d_max), C.byref(p),
                                        out.ctypes.data_as(_ip), C.c_uint64(4096),
                                        C.byref(cnt)))
        return out[: cnt.value].copy()

    def max_range(self, pts):
        pts = _xyz(pts)
        o = C.c_double()
        self._check(self.lib.ref_max_range(_dptr(pts), pts.shape[0], C.byref(o)))
        return o.value

    def prepare_source(self, raw, target):
        raw = _xyz(raw)
        op = _dp()
        cnt = C.c_uint64()
        leaf = C.c_double()
        conv = C.c_int32()
        dm = C.c_double()
        self._check(self.lib.ref_prepare_source(_dptr(raw), raw.shape[0], C.c_uint64(target),
                                                C.byref(op), C.byref(cnt), C.byref(leaf),
                                                C.byref(conv), C.byref(dm)))
        out = np.ctypeslib.as_array(op, shape=(cnt.value, 3)).copy() if cnt.value else \
            np.zeros((0, 3))
        self.lib.ref_free(op)
        return out, leaf.value, bool(conv.value), dm.value


class RefMap:
    def __init__(self, ref, handle, max_level):
        self.ref, self.h, self.max_level = ref, handle, max_level

    def save(self, path):
        """save_map, map_io.hpp:44-65."""
        self.ref._check(self.ref.lib.ref_save_map(self.h, os.fsencode(path)))

    def max_level_from_levels(self):
        lvl = C.c_int32()
        self.ref._check(self.ref.lib.ref_map_max_level(self.h, C.byref(lvl)))
        return lvl.value

    def __del__(self):
        try:
            if self.h:
                self.ref.lib.ref_map_free(self.h)
                self.h = None
        except Exception:
            pass

    def bbox(self):
        b = Aabb()
        self.ref.lib.ref_map_bbox(self.h, C.byref(b))
        return b

    def level_info(self, level):
        occ, buckets, cr = C.c_uint64(), C.c_uint64(), C.c_double()
        self.ref.lib.ref_level_info(self.h, level, C.byref(occ), C.byref(buckets), C.byref(cr))
        return occ.value, buckets.value, cr.value

    def occupied(self, level):
        n = C.c_uint64()
        self.ref._check(self.ref.lib.ref_level_occupied(self.h, level, None, C.c_uint64(0),
                                                        C.byref(n)))
        out = np.zeros((n.value, 3), np.int32)
        self.ref._check(self.ref.lib.ref_level_occupied(self.h, level, out.ctypes.data_as(_ip),
                                                        C.c_uint64(n.value), C.byref(n)))
        return out

    def contains(self, level, vox):
        vox = np.ascontiguousarray(np.asarray(vox, np.int32).reshape(-1, 3))
        out = np.zeros(vox.shape[0], np.uint8)
        self.ref.lib.ref_level_contains(self.h, level, vox.ctypes.data_as(_ip),
                                        C.c_uint64(vox.shape[0]),
                                        out.ctypes.data_as(C.POINTER(C.c_uint8)))
        return out

    def level_score(self, level, R, t, scan):
        scan = _xyz(scan)
        Ra = (C.c_double * 9)(*[float(v) for v in np.asarray(R).ravel()])
        ta = (C.c_double * 3)(*[float(v) for v in np.asarray(t).ravel()])
        o = C.c_int32()
        self.ref._check(self.ref.lib.ref_level_score(self.h, level, Ra, ta, _dptr(scan),
                                                     C.c_uint64(scan.shape[0]), C.byref(o)))
        return o.value

    def batch_evaluate(self, scan, cfg, nodes, d_max=0.0, workers=1):
        scan = _xyz(scan)
        nodes = nodes_to_array(nodes).copy()
        self.ref._check(self.ref.lib.ref_batch_evaluate(
            self.h, _dptr(scan), C.c_uint64(scan.shape[0]), C.byref(cfg), C.c_double(d_max),
            nodes.ctypes.data_as(_ip), C.c_uint64(nodes.shape[0]), C.c_int32(workers)))
        return nodes

    def search(self, scan, cfg, trace_cap=4096):
        scan = _xyz(scan)
        res = SearchResultC()
        tr = (C.c_int32 * trace_cap)()
        res.best_score_trace = C.cast(tr, C.POINTER(C.c_int32))
        res.trace_capacity = trace_cap
        self.ref._check(self.ref.lib.ref_search(self.h, _dptr(scan), C.c_uint64(scan.shape[0]),
                                                C.byref(cfg), C.byref(res)))
        trace = list(tr[: min(res.trace_length, trace_cap)])
        return res, trace

    def localize_scan(self, raw, cfg, target):
        raw = _xyz(raw)
        res = SearchResultC()
        self.ref._check(self.ref.lib.ref_localize_scan(self.h, _dptr(raw),
                                                       C.c_uint64(raw.shape[0]), C.byref(cfg),
                                                       C.c_uint64(target), C.byref(res)))
        return res

    def oracle_search(self, scan, cfg, cap=1 << 16):
        scan = _xyz(scan)
        best, leaves, n = C.c_int32(), C.c_uint64(), C.c_uint64()
        poses = np.zeros((cap, 6))
        self.ref._check(self.ref.lib.ref_oracle_search(
            self.h, _dptr(scan), C.c_uint64(scan.shape[0]), C.byref(cfg), C.byref(best),
            C.byref(leaves), _dptr(poses), C.c_uint64(cap), C.byref(n)))
        return best.value, leaves.value, poses[: min(n.value, cap)]


class Restated:
    """The plain-C restatement (oracle/liboracle.so)."""

    def __init__(self, path=RESTATED_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.orc_voxel_index.restype = C.c_int32
        L.orc_voxel_index.argtypes = [C.c_double, C.c_double]
        L.orc_map_build.argtypes = [_dp, C.c_uint64, C.c_double, C.c_int32,
                                    C.POINTER(C.c_void_p)]
        L.orc_map_free.argtypes = [C.c_void_p]
        L.orc_map_free.restype = None
        L.orc_level_count.restype = C.c_uint64
        L.orc_level_count.argtypes = [C.c_void_p, C.c_int32]
        L.orc_level_voxels.restype = _ip
        L.orc_level_voxels.argtypes = [C.c_void_p, C.c_int32]
        L.orc_level_contains.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.orc_level_score.restype = C.c_int32
        L.orc_level_score.argtypes = [C.c_void_p, C.c_int32, _dp, _dp, _dp, C.c_uint64]
        L.orc_max_range.restype = C.c_double
        L.orc_max_range.argtypes = [_dp, C.c_uint64]
        L.orc_batch_evaluate.argtypes = [C.c_void_p, _dp, C.c_uint64, C.c_void_p, C.c_double,
                                         _ip, C.c_uint64]
        L.orc_search.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_uint64, C.c_void_p,
                                 C.c_void_p]
        L.orc_search_sharded.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_uint64, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        L.orc_exhaustive.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_uint64, C.c_void_p,
                                     C.POINTER(C.c_int32), _u64p, _u64p]
        L.orc_angular_grid.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
        L.orc_divisions.restype = C.c_int32
        L.orc_divisions.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]
        L.orc_node_pose.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_void_p, _dp]
        L.orc_node_pose.restype = None
        L.orc_pose_to_transform.argtypes = [_dp, _dp, _dp]
        L.orc_pose_to_transform.restype = None

    def _check(self, st):
        if st != 0:
            raise OracleError(st, "oracle restatement")

    def voxel_index(self, c, cell):
        return self.lib.orc_voxel_index(c, cell)

    def map_build(self, pts, r, max_level):
        pts = _xyz(pts)
        h = C.c_void_p()
        self._check(self.lib.orc_map_build(_dptr(pts), pts.shape[0], r, max_level, C.byref(h)))
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        bbox = Aabb()
        bbox.min.x, bbox.min.y, bbox.min.z = (float(v) for v in lo)
        bbox.max.x, bbox.max.y, bbox.max.z = (float(v) for v in hi)
        return OrcMap(self, h, max_level, r, bbox)

    def angular_grid(self, cfg, d_max):
        out = (AxisGridC * (3 * (cfg.max_level + 1)))()
        self._check(self.lib.orc_angular_grid(C.byref(cfg), C.c_double(d_max), out))
        return out

    def pose_to_transform(self, pose6):
        p = (C.c_double * 6)(*pose6)
        R = (C.c_double * 9)()
        t = (C.c_double * 3)()
        self.lib.orc_pose_to_transform(p, R, t)
        return np.array(R[:]), np.array(t[:])

    def max_range(self, pts):
        pts = _xyz(pts)
        return self.lib.orc_max_range(_dptr(pts), pts.shape[0])


class OrcMap:
    def __init__(self, orc, handle, max_level, r, bbox):
        self.orc, self.h, self.max_level, self.r, self.bbox = orc, handle, max_level, r, bbox

    def __del__(self):
        try:
            if self.h:
                self.orc.lib.orc_map_free(self.h)
                self.h = None
        except Exception:
            pass

    def occupied(self, level):
        n = self.orc.lib.orc_level_count(self.h, level)
        p = self.orc.lib.orc_level_voxels(self.h, level)
        return np.ctypeslib.as_array(p, shape=(n, 3)).copy() if n else np.zeros((0, 3), np.int32)

    def contains(self, level, x, y, z):
        return self.orc.lib.orc_level_contains(self.h, level, x, y, z)

    def level_score(self, level, R, t, scan):
        scan = _xyz(scan)
        Ra = np.ascontiguousarray(R, np.float64)
        ta = np.ascontiguousarray(t, np.float64)
        return self.orc.lib.orc_level_score(self.h, level, _dptr(Ra), _dptr(ta), _dptr(scan),
                                            scan.shape[0])

    def batch_evaluate(self, scan, cfg, nodes, d_max=0.0):
        scan = _xyz(scan)
        nodes = nodes_to_array(nodes).copy()
        self.orc._check(self.orc.lib.orc_batch_evaluate(
            self.h, _dptr(scan), scan.shape[0], C.byref(cfg), d_max, nodes.ctypes.data_as(_ip),
            nodes.shape[0]))
        return nodes

    def search(self, scan, cfg, trace_cap=4096, shard=None):
        scan = _xyz(scan)
        res = SearchResultC()
        tr = (C.c_int32 * trace_cap)()
        res.best_score_trace = C.cast(tr, C.POINTER(C.c_int32))
        res.trace_capacity = trace_cap
        if shard is None:
            st = self.orc.lib.orc_search(self.h, C.byref(self.bbox), _dptr(scan), scan.shape[0],
                                         C.byref(cfg), C.byref(res))
        else:
            st = self.orc.lib.orc_search_sharded(self.h, C.byref(self.bbox), _dptr(scan),
                                                 scan.shape[0], C.byref(cfg), C.byref(shard),
                                                 C.byref(res))
        self.orc._check(st)
        return res, list(tr[: min(res.trace_length, trace_cap)])

    def exhaustive(self, scan, cfg):
        scan = _xyz(scan)
        b, n, leaves = C.c_int32(), C.c_uint64(), C.c_uint64()
        self.orc._check(self.orc.lib.orc_exhaustive(self.h, C.byref(self.bbox), _dptr(scan),
                                                    scan.shape[0], C.byref(cfg), C.byref(b),
                                                    C.byref(n), C.byref(leaves)))
        return b.value, n.value, leaves.value


def default_config(**kw):
    """SearchConfig defaults, search_config.hpp:24-52."""
    c = SearchConfigC()
    c.min_resolution = 1.0
    c.max_level = 6
    c.has_translation_range = 0
    c.roll_pitch_half_range = 0.02
    c.yaw_min = 0.0
    c.yaw_max = 6.283185307179586476925286766559
    c.score_threshold_fraction = 0.95
    c.batch_size = 10000
    c.strategy = 1
    c.branch_mode = 1
    c.workers = 1
    c.has_d_max = 0
    c.d_max = 0.0
    c.collect_trace = 0
    for k, v in kw.items():
        if k == "translation_range":
            c.has_translation_range = 1
            c.translation_range = v
        elif k == "d_max":
            c.has_d_max = 1
            c.d_max = v
        else:
            setattr(c, k, v)
    return c
