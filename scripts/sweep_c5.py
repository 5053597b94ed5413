"""C5 (BASELINE configs[4]): score-kernel sweep on the C2 campus
map: per level, 1M random candidates (translation uniform over the root
translation range at that level's cell, rotation indices uniform) x scan size
K in {1k..100k} (seeded prefixes of the raw C2 scan), scored with the device
batch_evaluate (rotation grouping + runs kernel).  Device time from CUDA
events on the call's stream; lookups/s and the SURVEY §8d gather model
(32 B per lookup) against the measured random-gather ceilings.

    python scripts/sweep_c5.py [--n 1000000] [--levels 0,1,2,3,4,5] > profiles/.../c5.json
Parity of these kernels on random candidates is pinned by
tests/test_score_gpu.py (golden batches from the reference incl. campus).
"""
import argparse
import ctypes as C
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import harness as H  # noqa: E402  (synthetic inputs)
import bench  # noqa: E402
import paper_2310_10023_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--levels", default="0,1,2,3,4,5")
    ap.add_argument("--ks", default="1000,2000,5000,10000,20000,50000,100000")
    args = ap.parse_args()
    cfgd = bench.CONFIGS["c2"]
    spec = H.SceneSpec.default(**cfgd["spec"])
    m, raw, _ = H.gen_scene(spec, cfgd["seed"])
    kmax = min(max(int(k) for k in args.ks.split(",")), raw.shape[0])
    full = H.cut_scan(raw, kmax, 7)
    vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    vm.set_stream(stream.cuda_stream)
    cfg = bench.search_config(B, cfgd)
    (lo, hi) = vm.bbox()
    gather = {}
    for label, nbytes in (("l2_64MiB", 64 << 20), ("hbm_4GiB", 4 << 30)):
        out = C.c_double()
        if B.lib.bbs_gather_bench(0, nbytes, C.byref(out)) == 0:
            gather[label] = out.value
    rows = []
    for lv in (int(x) for x in args.levels.split(",")):
        rng = np.random.default_rng(5000 + lv)
        cell = cfgd["r"] * 2 ** lv
        grids = B.AngularGrid(cfg, B.max_range(full))
        n = args.n
        nodes = np.zeros((n, 8), np.int32)
        for a, (l0, h0) in enumerate(zip(lo, hi)):
            nodes[:, a] = rng.integers(math.floor(l0 / cell), math.ceil(h0 / cell) + 1, n)
        for a in range(3):
            nodes[:, 3 + a] = rng.integers(0, grids.axis(a, lv).max_index() + 1, n)
        nodes[:, 6] = lv
        nodes[:, 7] = -1
        d_nodes = torch.from_numpy(nodes).cuda()
        for k in (int(x) for x in args.ks.split(",")):
            if k > full.shape[0]:
                continue
            ds = B.DeviceScan(vm, full[:k])
            c = cfg.to_c()

            def run():
                st = B.lib.bbs_batch_evaluate_device(vm._h, ds._h, C.byref(c), grids.d_max,
                                                     C.c_void_p(d_nodes.data_ptr()), n,
                                                     C.c_void_p(stream.cuda_stream))
                assert st == 0, B.lib.bbs_last_error()

            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record(stream)
            for _ in range(reps):
                run()
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            lookups = n * k
            gbs = lookups * 32 / (ms * 1e-3) / 1e9
            row = dict(level=lv, K=k, candidates=n, ms=ms, evals_per_s=n / (ms * 1e-3),
                       lookups_per_s=lookups / (ms * 1e-3), gather_model_gbs=gbs,
                       frac_of_l2_gather=gbs / gather.get("l2_64MiB", float("nan")),
                       level_bytes=vm.level(lv).device_bytes())
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
            del ds
    print(json.dumps({"config": "C5 sweep on the C2 campus map", "gather_peaks_gbs": gather,
                      "rows": rows}))


if __name__ == "__main__":
    main()
