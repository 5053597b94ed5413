"""Time prepare_source: device vs the host restatement vs the reference (C2 raw scan)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import harness as H  # noqa: E402  (synthetic inputs)
import numpy as np
import bench
import paper_2310_10023_b200 as B
from pyoracle import Reference
cfgd = bench.CONFIGS["c2"]
spec = H.SceneSpec.default(**cfgd["spec"])
_, raw, _ = H.gen_scene(spec, 1)
ref = Reference()
for target in (10000, 2000):
    B.prepare_source_device(raw, target)  # warm
    t = time.perf_counter(); d = B.prepare_source_device(raw, target); td = time.perf_counter() - t
    t = time.perf_counter(); h = B.prepare_source(raw, target); th = time.perf_counter() - t
    t = time.perf_counter(); r = ref.prepare_source(raw, target); tr = time.perf_counter() - t
    same = float(np.mean(np.all(d.scan == r[0], axis=1)))
    print(f"raw {raw.shape[0]} target {target}: device {1e3*td:.1f} ms, host restatement {1e3*th:.1f} ms, "
          f"reference {1e3*tr:.1f} ms; leaf equal {d.leaf == r[1]}, count {d.scan.shape[0]} == {r[0].shape[0]}, "
          f"bit-identical centroids {same:.3f}, max |diff| {np.abs(d.scan - r[0]).max():.3g}")
