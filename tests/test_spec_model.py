"""CPU check of the speculative-round ALGORITHM (DESIGN §3 K6s) against the
reference's own search() (oracle/_ref): a plain-Python model forms up to k
epochs from the queue as if no flush had survivors, scores them with the
reference's batch_evaluate, keeps the prefix of epochs no survivor overtakes
and commits exactly; best score, Stats and trace must equal the reference's.
The CUDA kernels (frontier_spec_kernel, survivors_spec_kernel) implement this
model; tests/test_search_gpu.py checks them on the device."""
import math

import numpy as np
import pytest

from conftest import golden_json

KS = 1 << 20


def bfs_key(score, level, seq):
    return ((KS - 1 - score) << 44) | ((15 - level) << 40) | seq


def spec_search(ref, rm, scan, cfg, k_spec):
    d_max = ref.max_range(scan)

    def score(nodes):
        return rm.batch_evaluate(scan, cfg, np.array(nodes, np.int32), d_max=d_max) if len(nodes) else nodes

    thr = math.floor(cfg.score_threshold_fraction * scan.shape[0])
    roots = score(ref.initial_nodes(cfg, d_max, rm.bbox()))
    st = dict(gen=len(roots), pruned=0, flushed=1)
    q, seq = [], 0
    for n in roots:
        if n[7] < thr:
            st["pruned"] += 1
        else:
            q.append((bfs_key(int(n[7]), int(n[6]), seq), tuple(int(x) for x in n)))
            seq += 1
    q.sort()
    best, trace, b = thr, [], cfg.batch_size
    while q:
        eps, i, B, cur, prn, trl = [], 0, best, [], 0, []
        while i < len(q) and len(eps) < k_spec:
            kk, n = q[i]
            if n[7] < B:
                prn += 1
            elif n[6] == 0:
                B = n[7]
                trl.append(B)
            else:
                cur += [tuple(int(x) for x in c) for c in ref.branch(cfg, d_max, n)]
                if len(cur) > b:  # search.hpp:166
                    eps.append(dict(ch=cur, cons=i + 1, last=kk, B=B, pr=prn, tr=list(trl), drain=False))
                    cur = []
            i += 1
        if len(eps) < k_spec and i == len(q):
            if cur:  # drain flush, search.hpp:146-148
                eps.append(dict(ch=cur, cons=i, last=None, B=B, pr=prn, tr=list(trl), drain=True))
            elif not eps:
                st["pruned"] += prn
                best = B
                trace += trl
                break
        for e in eps:
            e["sc"] = score(e["ch"])
            e["sv"] = [c for c in e["sc"] if c[7] >= e["B"]]
            e["mk"] = min([bfs_key(int(c[7]), int(c[6]), (1 << 40) - 1) for c in e["sv"]], default=None)
        A, mk, anys = 1, eps[0]["mk"], bool(eps[0]["sv"])
        for e in eps[1:]:
            if not ((not anys) if e["drain"] else (mk is None or mk > e["last"])):
                break
            A += 1
            if e["mk"] is not None:
                mk = e["mk"] if mk is None else min(mk, e["mk"])
            anys = anys or bool(e["sv"])
        last = eps[A - 1]
        st["pruned"] += last["pr"]
        best = last["B"]
        trace += last["tr"]
        nq = q[last["cons"]:]
        for e in eps[:A]:
            st["gen"] += len(e["ch"])
            st["flushed"] += 1
            for c in e["sc"]:
                if c[7] >= e["B"]:
                    nq.append((bfs_key(int(c[7]), int(c[6]), seq), tuple(int(x) for x in c)))
                    seq += 1
                else:
                    st["pruned"] += 1
        kept = [x for x in nq if x[1][7] >= best]  # the incumbent trim
        st["pruned"] += len(nq) - len(kept)
        q = sorted(kept)
    return best, st, trace


@pytest.mark.parametrize("name,batch,k_spec", [("tiny", 10000, 1), ("tiny", 40, 3), ("tiny", 40, 8),
                                               ("small", 300, 8)])
def test_speculative_rounds_model_equals_reference(ref, golden_scenes, name, batch, k_spec):
    from pyoracle import default_config
    sc = golden_scenes[name]
    spec = ref.default_spec()
    for a, v in sc["spec"].items():
        setattr(spec, a, v)
    m, scan, _ = ref.gen_scene(spec, sc["seed"])
    rm = ref.map_build(m, sc["r"], sc["max_level"], 0.3, 8 << 30)
    cfg = default_config(min_resolution=sc["r"], max_level=sc["max_level"], roll_pitch_half_range=0.02,
                         batch_size=batch, score_threshold_fraction=0.9, collect_trace=1)
    want, trace = rm.search(scan, cfg, trace_cap=1 << 16)
    best, st, tr = spec_search(ref, rm, scan, cfg, k_spec)
    assert best == want.best_score
    assert (st["gen"], st["pruned"], st["flushed"]) == \
        (want.stats.nodes_generated, want.stats.nodes_pruned, want.stats.batches_flushed)
    assert tr == trace
