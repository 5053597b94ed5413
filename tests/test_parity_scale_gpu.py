"""Per-candidate parity of the kernels that do the search's work, and parity
on every BASELINE config (C1-C5), against goldens made by running the
UNMODIFIED reference (tests/golden/make_scale_goldens.py, oracle/_ref).

* root batch (search.hpp:111-124): the device root kernels' survivor set
  (score >= threshold, initial_nodes order) and scores equal the reference's
  batch_evaluate on every root; with the survivor-bound early exit disabled
  (bbs_search_dump.exact_roots) every root score equals the reference's
  (sha256 over all 3.97M C2 root scores);
* flush batches (search.hpp:132-143): every node the device flushed is
  re-scored by the reference's batch_evaluate (oracle/_ref) and must be equal
  — these are the scores of the flush cache (cache_build/cache_probe), the
  cube kernel and the general kernel, whichever scored them;
* C3 (city, 7 levels, +-5 deg), C4 (64 scans of the C2 map), C5 (1M
  candidates x K 1k-100k per level): search() and batch_evaluate results
  equal the reference's goldens."""
import hashlib
import math
import os
import sys

import numpy as np
import pytest

import harness as H  # noqa: E402  (synthetic inputs)
from conftest import GOLDEN, golden_json, golden_npz, load_case

sys.path.insert(0, GOLDEN)
from make_scale_goldens import C1, C2, C3, C4_PICK, C5_KS, c5_nodes, max_index  # noqa: E402

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def has(name):
    return os.path.exists(os.path.join(GOLDEN, name))


CASES = {"room": ("c1", C1), "campus": ("c2", C2)}


@pytest.fixture(scope="module")
def scenes(B, golden_scenes):
    out = {}

    def get(name):
        if name not in out:
            m, s, gt, sc = load_case(B, golden_scenes, name)
            vm = B.MultiResVoxelMap.build(m, sc["r"], sc["max_level"])
            out[name] = (vm, B.DeviceScan(vm, s), s, sc)
        return out[name]
    return get


def search_cfg(B, case, **ov):
    kw = dict(min_resolution=case["r"], max_level=case["max_level"],
              roll_pitch_half_range=case["rp"], collect_trace=True, batch_size=10000)
    kw.update(ov)
    return B.SearchConfig(**kw)


def assert_same_search(res, want, label):
    assert res.best_score == want["best_score"], label
    assert res.matched == want["matched"], label
    assert list(res.best_pose.as_tuple()) == want["best_pose"], label
    assert (res.stats.nodes_generated, res.stats.nodes_pruned, res.stats.batches_flushed) == \
        (want["nodes_generated"], want["nodes_pruned"], want["batches_flushed"]), label
    assert res.best_score_trace == want["trace"], label


@pytest.mark.parametrize("name", ["room", "campus"])
def test_root_batch_survivors_match_reference(B, scenes, name):
    """The production root kernels (early exit ON): the set of roots with
    score >= threshold and their scores equal the reference's; every other
    root is below the threshold (a partial count of an early-exited column
    can never reach it)."""
    tag, case = CASES[name]
    g = golden_npz(f"{tag}_roots.npz")
    vm, ds, s, sc = scenes(name)
    d = B.search_scan_dump(vm, ds, search_cfg(B, case))
    assert d.root_scores.shape[0] == int(g["n_roots"])
    thr = int(g["threshold"])
    surv = np.nonzero(d.root_scores >= thr)[0]
    np.testing.assert_array_equal(surv, g["index"])
    np.testing.assert_array_equal(d.root_scores[surv], g["score"])
    assert_same_search(d.result, golden_json(f"{name}_search.json")["bfs_roto_b10000"], name)


@pytest.mark.parametrize("name", ["room", "campus"])
def test_root_batch_every_score_exact(B, scenes, name):
    """Early exit OFF (bbs_search_dump.exact_roots): every root score of the
    root column kernel equals the reference's batch_evaluate (digest over all
    roots in initial_nodes order + the score histogram)."""
    tag, case = CASES[name]
    g = golden_npz(f"{tag}_roots.npz")
    vm, ds, s, sc = scenes(name)
    d = B.search_scan_dump(vm, ds, search_cfg(B, case), exact_roots=True)
    hist = np.bincount(d.root_scores, minlength=s.shape[0] + 1)
    np.testing.assert_array_equal(hist, g["hist"])
    assert digest(d.root_scores.astype(np.int32)) == str(g["scores_digest"])
    # results do not depend on the early exit
    assert_same_search(d.result, golden_json(f"{name}_search.json")["bfs_roto_b10000"], name)


@pytest.mark.parametrize("name", ["room", "campus"])
def test_flush_batches_rescored_by_reference(B, ref, scenes, name):
    """Every flushed batch of the search, re-scored by the reference's own
    batch_evaluate (search.hpp:23-34), node by node."""
    tag, case = CASES[name]
    vm, ds, s, sc = scenes(name)
    cfg = search_cfg(B, case)
    d = B.search_scan_dump(vm, ds, cfg)
    want = golden_json(f"{name}_search.json")["bfs_roto_b10000"]
    assert_same_search(d.result, want, name)
    # the dumped batches are all of the search's non-root evaluations
    assert d.root_scores.shape[0] + d.flush_nodes.shape[0] == want["nodes_generated"]
    assert len(d.epoch_ids) == want["batches_flushed"] - 1
    from pyoracle import default_config
    rmap = ref.map_build(*_ref_inputs(ref, name, case))
    rc = default_config(min_resolution=case["r"], max_level=case["max_level"],
                        roll_pitch_half_range=case["rp"])
    got = rmap.batch_evaluate(s, rc, d.flush_nodes, workers=os.cpu_count())
    bad = np.nonzero(got[:, 7] != d.flush_scores)[0]
    assert bad.size == 0, f"{bad.size} of {d.flush_nodes.shape[0]} flush scores differ, e.g. " \
                          f"{d.flush_nodes[bad[:3]].tolist()} dev {d.flush_scores[bad[:3]].tolist()} " \
                          f"ref {got[bad[:3], 7].tolist()}"
    # the flush scores span the levels the search visited
    assert set(np.unique(d.flush_nodes[:, 6])) <= set(range(case["max_level"]))


def _ref_inputs(ref, name, case):
    spec = ref.default_spec()
    for k, v in case["spec"].items():
        setattr(spec, k, v)
    m, _, _ = ref.gen_scene(spec, case["seed"])
    return m, case["r"], case["max_level"], 0.3, 8 << 30


@pytest.mark.parametrize("level", range(6))
def test_c5_sweep_matches_reference(B, level):
    """C5 (BASELINE configs[4]): 1M candidates of one level x K in 1k-100k
    (prefixes of the raw C2 scan), scored by the device batch_evaluate: all
    1M scores equal the reference's for K <= 10k (sha256), every 64th
    candidate for K > 10k."""
    if not has("c5.npz"):
        pytest.skip("c5 golden not generated")
    g = golden_npz("c5.npz")
    m, raw, _ = H.gen_scene(H.SceneSpec.default(**C2["spec"]), C2["seed"])
    full = H.cut_scan(raw, min(max(C5_KS), raw.shape[0]), 7)
    assert digest(full) == str(g["scan_digest"])
    vm = _c2_map(B, m)
    cfg = search_cfg(B, C2)
    grids = B.AngularGrid(cfg, float(g["d_max"]))
    lo, hi = vm.bbox()
    mi = [grids.axis(a, level).max_index() for a in range(3)]
    nodes = c5_nodes(lo, hi, C2["r"], level, mi)
    assert digest(nodes) == str(g[f"nodes_digest_l{level}"])
    for k in C5_KS:
        if k > full.shape[0]:
            continue
        sc = B.batch_evaluate(nodes, vm, full[:k], grids)[:, 7].astype(np.int32)
        if k <= 10000:
            assert digest(sc) == str(g[f"digest_l{level}_k{k}"]), (level, k)
        else:
            np.testing.assert_array_equal(sc[::64], g[f"every64_l{level}_k{k}"], err_msg=f"{level} {k}")


_C2_MAP = {}


def _c2_map(B, m):
    if "vm" not in _C2_MAP:
        _C2_MAP["vm"] = B.MultiResVoxelMap.build(m, C2["r"], C2["max_level"])
    return _C2_MAP["vm"]


def test_c4_scans_match_reference(B, monkeypatch):
    """C4 (BASELINE configs[3]): 64 scans of the C2 map; the device search of
    scans 0, 8, ..., 56 equals the reference's search(), alone and inside the
    throughput path (bbs_search_scans, 16 in flight: per-search graphs on
    their own streams, and co-batched flushes)."""
    if not has("c4_search.json"):
        pytest.skip("c4 golden not generated")
    g = golden_json("c4_search.json")
    spec = H.SceneSpec.default(**C2["spec"])
    m, _, _ = H.gen_scene(spec, C2["seed"])
    scans, poses = H.gen_scans(spec, C2["seed"], g["pose_seed_base"], 64)
    scans = [H.cut_scan(s, min(g["K"], s.shape[0]), g["cut_seed"]) for s in scans]
    assert [digest(s) for s in scans] == g["scan_digests"]
    vm = _c2_map(B, m)
    cfg = search_cfg(B, C2)
    ds = [B.DeviceScan(vm, s) for s in scans]
    for j in C4_PICK:
        assert_same_search(B.search_scan(vm, ds[j], cfg), g["searches"][str(j)], f"c4 scan {j}")
    for cobatch in ("0", "1"):
        monkeypatch.setenv("BBS_COBATCH", cobatch)
        many = B.search_scans(vm, ds, cfg, concurrency=16, trace_capacity=1 << 16)
        for j in C4_PICK:
            assert_same_search(many[j], g["searches"][str(j)], f"c4 scan {j} (search_scans, co-batched {cobatch})")
        assert (sum(r.group_checks for r in many) > 0) == (cobatch == "1")


@pytest.fixture(scope="module")
def c3(B):
    if not has("c3_search.json"):
        pytest.skip("c3 golden not generated")
    m, s, gt = H.gen_scene(H.SceneSpec.default(**C3["spec"]), C3["seed"])
    s = H.cut_scan(s, min(C3["K"], s.shape[0]), 7)
    vm = B.MultiResVoxelMap.build(m, C3["r"], C3["max_level"])
    return vm, s


@pytest.mark.parametrize("direct", ["1", "0", "1-tiled"])
def test_c3_search_matches_reference(B, c3, direct, monkeypatch):
    """C3 city (BASELINE configs[2]): 30M map points, K = 30k, 7 levels,
    +-5 deg roll/pitch: search() equals the reference's (score, pose, Stats,
    trace) -- with the speculative rounds' direct runs scored in the probe
    kernel (default) and by the cube kernel after it; "tiled": the merge
    kernel's two-phase survivor sort forced from 257 survivors (72 rounds of
    up to 16 flushes)."""
    direct, _, tiled = direct.partition("-")
    monkeypatch.setenv("BBS_DIRECT_RUNS", direct)
    if tiled:
        monkeypatch.setenv("BBS_TILE_RANK_MIN", "256")
    vm, s = c3
    want = golden_json("c3_search.json")["bfs_roto_b10000"]
    assert digest(s) == want["scan_digest"]
    res = B.search(vm, s, search_cfg(B, C3))
    assert_same_search(res, want, f"c3 (direct runs {direct})")


def test_c3_batches_match_reference(B, c3):
    """C3: 512 random candidates per level (7 levels) at K = 30k scored by the
    device batch_evaluate equal the reference's."""
    if not has("c3_batch.npz"):
        pytest.skip("c3 batch golden not generated")
    vm, s = c3
    g = golden_npz("c3_batch.npz")
    cfg = search_cfg(B, C3)
    grids = B.AngularGrid(cfg, B.max_range(s))
    got = B.batch_evaluate(g["nodes"], vm, s, grids)[:, 7]
    np.testing.assert_array_equal(got, g["scores"])


def test_c2_localize_scan_raw_scan_matches_reference(B):
    """localize_scan (pipeline.hpp:45-51), the public entry point, on the RAW
    C2 scan (~236k points, downsample target 10k): the default exact prepare
    (device auto_leaf counts + the reference's centroid summation order) and
    the search equal the reference's localize_scan: score, pose, Stats."""
    if not has("c2_localize.json"):
        pytest.skip("c2 localize golden not generated")
    want = golden_json("c2_localize.json")
    m, raw, _ = H.gen_scene(H.SceneSpec.default(**C2["spec"]), C2["seed"])
    assert digest(raw) == want["raw_digest"]
    prep = B.prepare_source(raw, want["target"])  # host restatement, same order
    assert digest(prep.scan) == want["prepared_digest"]
    vm = _c2_map(B, m)
    cfg = search_cfg(B, C2, collect_trace=False)
    res = B.localize_scan(vm, raw, cfg, want["target"])
    assert res.scan_points == want["scan_points"]
    assert res.best_score == want["best_score"]
    assert list(res.best_pose.as_tuple()) == want["best_pose"]
    assert (res.stats.nodes_generated, res.stats.nodes_pruned, res.stats.batches_flushed) == \
        (want["nodes_generated"], want["nodes_pruned"], want["batches_flushed"])
