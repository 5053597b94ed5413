"""Multi-GPU path: root sharding + per-epoch incumbent
max-all-reduce + winner election.

* CPU (gloo, world_size 2, two processes): the C restatement runs the SAME
  protocol as the device path (oracle/bbs_oracle.c orc_search_sharded,
  csrc/search.cu run_search); checks the partition of the root set, that
  every rank returns the same winner, and that TransOnly results equal the
  unsharded search and the exhaustive oracle (admissible bound).
* GPU (one device, two host threads): bbs_search_sharded per rank with a
  thread-barrier all-reduce; each rank's result and Stats equal the CPU
  restatement of the protocol exactly.  The ranks' kernels never wait on one
  another (the exchange is on the host), so running them on one GPU is safe.
"""
import ctypes as C
import os
import threading

import numpy as np
import pytest
import harness as H  # noqa: E402  (synthetic inputs)
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

SPEC = dict(size_x=24.0, size_y=24.0, size_z=10.0, num_boxes=4, min_box_side=2.5,
            max_box_side=6.0, min_box_height=3.0, map_spacing=0.3, scan_spacing=0.45,
            scan_range=14.0, min_scan_points=300)


def _scene():
    import paper_2310_10023_b200 as B
    m, s, gt = H.gen_scene(H.SceneSpec.default(**SPEC), 42)
    return m, s, gt


def _cfg(mode, **kw):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import default_config
    c = dict(min_resolution=0.5, max_level=3, branch_mode=mode, batch_size=400,
             roll_pitch_half_range=0.0 if mode == 0 else 0.02, collect_trace=1)
    c.update(kw)
    return default_config(**c)


def _gloo_worker(rank, world, port, mode, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    from pyoracle import Restated
    from paper_2310_10023_b200._abi import ALLREDUCE_MAX_FN, Shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Restated()
    m, s, _ = _scene()
    om = orc.map_build(m, 0.5, 3)

    def allreduce(values, count, _user):
        t = torch.tensor([values[i] for i in range(count)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for i in range(count):
            values[i] = int(t[i])
        return 0

    cb = ALLREDUCE_MAX_FN(allreduce)
    res, trace = om.search(s, _cfg(mode), shard=Shard(rank, world, cb, None))
    out_q.put((rank, res.best_score, bool(res.matched), res.best_pose.as_tuple(),
               res.root_nodes, res.stats.nodes_generated))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
def test_gloo_world2_protocol(mode, orc):
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = dict((r[0], r[1:]) for r in (q.get(timeout=10) for _ in range(2)))
    # every rank reports the same elected winner
    assert got[0][:3] == got[1][:3]
    m, s, _ = _scene()
    om = orc.map_build(m, 0.5, 3)
    single, _ = om.search(s, _cfg(mode))
    # the root set is partitioned exactly
    assert got[0][3] + got[1][3] == single.root_nodes
    assert got[0][3] > 0 and got[1][3] > 0
    if mode == 0:  # TransOnly: admissible bound -> same best score as unsharded
        assert got[0][0] == single.best_score
        assert got[0][1] == bool(single.matched)


def test_world1_shard_equals_unsharded(orc):
    from paper_2310_10023_b200._abi import ALLREDUCE_MAX_FN, Shard
    m, s, _ = _scene()
    om = orc.map_build(m, 0.5, 3)
    cb = ALLREDUCE_MAX_FN(lambda v, n, u: 0)
    for mode in (0, 1):
        a, ta = om.search(s, _cfg(mode))
        b, tb = om.search(s, _cfg(mode), shard=Shard(0, 1, cb, None))
        assert (a.best_score, a.best_pose.as_tuple(), a.stats.nodes_generated,
                a.stats.nodes_pruned, a.stats.batches_flushed, ta) == \
            (b.best_score, b.best_pose.as_tuple(), b.stats.nodes_generated,
             b.stats.nodes_pruned, b.stats.batches_flushed, tb)


class ThreadAllReduce:
    """Element-wise MAX across `n` host threads (stand-in for NCCL)."""

    def __init__(self, n):
        self.n = n
        self.barrier = threading.Barrier(n)
        self.lock = threading.Lock()
        self.buf = {}

    def __call__(self, rank, vals):
        with self.lock:
            self.buf[rank] = list(vals)
        self.barrier.wait()
        out = [max(self.buf[r][i] for r in range(self.n)) for i in range(len(vals))]
        self.barrier.wait()
        return out


def _run_threads(world, fn):
    results, errors = {}, []

    def body(rank):
        try:
            results[rank] = fn(rank)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    return results


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_device_sharded_equals_restated_protocol(B, orc, world, mode):
    from paper_2310_10023_b200._abi import ALLREDUCE_MAX_FN, Shard
    m, s, _ = _scene()
    vm = B.MultiResVoxelMap.build(m, 0.5, 3)
    ds = B.DeviceScan(vm, s)
    cfgc = _cfg(mode)
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, branch_mode=mode, batch_size=400,
                         roll_pitch_half_range=0.0 if mode == 0 else 0.02, collect_trace=True)
    ar_dev, ar_orc = ThreadAllReduce(world), ThreadAllReduce(world)
    dev = _run_threads(world, lambda r: B.search_sharded(vm, ds, cfg, r, world,
                                                         lambda v: ar_dev(r, v)))
    om = orc.map_build(m, 0.5, 3)

    def orc_rank(r):
        def cb(values, count, _u):
            out = ar_orc(r, [values[i] for i in range(count)])
            for i in range(count):
                values[i] = out[i]
            return 0
        keep = ALLREDUCE_MAX_FN(cb)
        res, trace = om.search(s, cfgc, shard=Shard(r, world, keep, None))
        return res, trace

    want = _run_threads(world, orc_rank)
    for r in range(world):
        d, (w, wt) = dev[r], want[r]
        assert d.best_score == w.best_score and d.matched == bool(w.matched), r
        assert d.best_pose.as_tuple() == w.best_pose.as_tuple(), r
        assert (d.stats.nodes_generated, d.stats.nodes_pruned, d.stats.batches_flushed) == \
            (w.stats.nodes_generated, w.stats.nodes_pruned, w.stats.batches_flushed), r
        assert d.root_nodes == w.root_nodes
        assert d.best_score_trace == wt
    assert sum(dev[r].root_nodes for r in range(world)) == \
        B.search(vm, s, cfg).root_nodes


# ---- batch-split exact mode (SURVEY §8e "parity caveat" mitigation) --------

def _gloo_exact_worker(rank, world, port, mode, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    from pyoracle import Restated
    from paper_2310_10023_b200._abi import ALLREDUCE_MAX_FN, SHARD_EXACT, Shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Restated()
    m, s, _ = _scene()
    om = orc.map_build(m, 0.5, 3)
    calls = [0]

    def allreduce(values, count, _user):
        calls[0] += 1
        t = torch.tensor([values[i] for i in range(count)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for i in range(count):
            values[i] = int(t[i])
        return 0

    cb = ALLREDUCE_MAX_FN(allreduce)
    res, trace = om.search(s, _cfg(mode), shard=Shard(rank, world, cb, None, SHARD_EXACT, 0, None))
    out_q.put((rank, res.best_score, bool(res.matched), res.best_pose.as_tuple(), res.root_nodes,
               res.stats.nodes_generated, res.stats.nodes_pruned, res.stats.batches_flushed,
               tuple(trace), calls[0]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
def test_gloo_world2_exact_equals_unsharded(mode, orc):
    """Exact mode over gloo: each rank scores half of every batch, yet both
    return the single-queue search() result, RotoTrans included."""
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_gloo_exact_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = dict((r[0], r[1:]) for r in (q.get(timeout=10) for _ in range(2)))
    m, s, _ = _scene()
    om = orc.map_build(m, 0.5, 3)
    single, strace = om.search(s, _cfg(mode))
    want = (single.best_score, bool(single.matched), single.best_pose.as_tuple())
    for r in (0, 1):
        assert got[r][:3] == want, r
        assert got[r][4:7] == (single.stats.nodes_generated, single.stats.nodes_pruned,
                               single.stats.batches_flushed), r
        assert list(got[r][7]) == list(strace), r
        assert got[r][8] == single.stats.batches_flushed  # one score exchange per batch
    assert got[0][3] + got[1][3] == single.root_nodes and min(got[0][3], got[1][3]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_device_exact_threads_equal_unsharded(B, world, mode):
    """Exact mode on the device (host exchange, one host thread per rank):
    every rank equals the unsharded device search exactly."""
    m, s, _ = _scene()
    vm = B.MultiResVoxelMap.build(m, 0.5, 3)
    ds = B.DeviceScan(vm, s)
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, branch_mode=mode, batch_size=400,
                         roll_pitch_half_range=0.0 if mode == 0 else 0.02, collect_trace=True)
    single = B.search_scan(vm, ds, cfg)
    with pytest.raises(B.ConfigError):  # exact mode with world > 1 needs an exchange
        B.search_sharded(vm, ds, cfg, 0, world, mode="exact")
    ar = ThreadAllReduce(world)
    dev = _run_threads(world, lambda r: B.search_sharded(vm, ds, cfg, r, world,
                                                         lambda v: ar(r, v), mode="exact"))
    for r in range(world):
        d = dev[r]
        assert (d.best_score, d.matched, d.best_pose.as_tuple()) == \
            (single.best_score, single.matched, single.best_pose.as_tuple()), r
        assert (d.stats.nodes_generated, d.stats.nodes_pruned, d.stats.batches_flushed) == \
            (single.stats.nodes_generated, single.stats.nodes_pruned, single.stats.batches_flushed), r
        assert d.best_score_trace == single.best_score_trace, r
        assert d.epochs == single.epochs
    assert sum(dev[r].root_nodes for r in range(world)) == single.root_nodes


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_nccl_world1_equals_unsharded(B, mode):
    """The device-side NCCL exchange path (bbs_comm_t, world 1): roots and
    exact modes reproduce the unsharded search, Stats and trace included."""
    m, s, _ = _scene()
    vm = B.MultiResVoxelMap.build(m, 0.5, 3)
    ds = B.DeviceScan(vm, s)
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, branch_mode=mode, batch_size=400,
                         roll_pitch_half_range=0.0 if mode == 0 else 0.02, collect_trace=True)
    single = B.search_scan(vm, ds, cfg)
    comm = B.Comm(0, 0, 1, B.Comm.unique_id())
    try:
        for smode in ("roots", "exact"):
            d = B.search_sharded(vm, ds, cfg, 0, 1, comm=comm, mode=smode)
            assert (d.best_score, d.matched, d.best_pose.as_tuple()) == \
                (single.best_score, single.matched, single.best_pose.as_tuple()), smode
            assert (d.stats.nodes_generated, d.stats.nodes_pruned, d.stats.batches_flushed) == \
                (single.stats.nodes_generated, single.stats.nodes_pruned,
                 single.stats.batches_flushed), smode
            assert d.best_score_trace == single.best_score_trace, smode
    finally:
        comm.close()


def _nccl_worker(rank, world, port, mode, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_2310_10023_b200 as B
    m, s, _ = _scene()
    vm = B.MultiResVoxelMap.build(m, 0.5, 3, device=rank)
    ds = B.DeviceScan(vm, s)
    cfg = B.SearchConfig(min_resolution=0.5, max_level=3, branch_mode=1, batch_size=400,
                         roll_pitch_half_range=0.02, collect_trace=True)
    uid = [B.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = B.Comm(rank, rank, world, uid[0])
    try:
        d = B.search_sharded(vm, ds, cfg, rank, world, comm=comm, mode=mode)
        single = B.search_scan(vm, ds, cfg)
        out_q.put((rank, d.best_score, d.best_pose.as_tuple(),
                   (d.stats.nodes_generated, d.stats.nodes_pruned, d.stats.batches_flushed),
                   d.best_score_trace, single.best_score, single.best_pose.as_tuple(),
                   (single.stats.nodes_generated, single.stats.nodes_pruned, single.stats.batches_flushed),
                   single.best_score_trace))
    finally:
        comm.close()
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["exact", "roots"])
def test_nccl_world2_processes(mode):
    """Two processes, one GPU each, NCCL communicator (the bench's --gpus 2
    path): EXACT equals the unsharded search on every rank (Stats and trace
    included); ROOTS gives every rank the same winner.  Needs >= 2 GPUs
    (ranks that wait on one another must not share a GPU)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    winners = {(r[1], r[2]) for r in res}
    assert len(winners) == 1
    if mode == "exact":
        for r in res:
            assert (r[1], r[2], r[3], r[4]) == (r[5], r[6], r[7], r[8])
