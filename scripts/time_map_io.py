"""Time load_map / save_map on the C2 campus map: device loader vs the
reference's load_map (oracle/_ref, collision_target 0.3)."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import harness as H  # noqa: E402  (synthetic inputs)
import numpy as np
import bench
import paper_2310_10023_b200 as B
from pyoracle import Reference
cfgd = bench.CONFIGS["c2"]
m, _, _ = H.gen_scene(H.SceneSpec.default(**cfgd["spec"]), cfgd["seed"])
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
d = tempfile.mkdtemp()
path = os.path.join(d, "c2.vxm")
t = time.perf_counter(); vm.save(path); ts = time.perf_counter() - t
size = os.path.getsize(path)
B.load_map(path)  # warm
t = time.perf_counter(); lm = B.load_map(path); tl = time.perf_counter() - t
same = all(np.array_equal(lm.level(l).occupied_voxels(), vm.level(l).occupied_voxels()) for l in range(cfgd["max_level"] + 1))
ref = Reference()
t = time.perf_counter(); rm = ref.load_map(path, 0.3, 8 << 30); tr = time.perf_counter() - t
print(f"C2 map file {size / 1e6:.1f} MB: save {1e3 * ts:.0f} ms, device load_map {1e3 * tl:.0f} ms "
      f"(identical sets: {same}), reference load_map (ct 0.3) {1e3 * tr:.0f} ms")
