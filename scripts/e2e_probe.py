"""Host-side breakdown of the public bbs_search() call on the bench workload
(BBS_DEBUG_HOST prints per-phase host timestamps to stderr)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS[os.environ.get("CFG", "c2")]
m, s, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
cfg = bench.search_config(B, cfgd)
s = np.ascontiguousarray(s, dtype=np.float64)
for i in range(8):
    t = time.perf_counter()
    r = B.search(vm, s, cfg)
    print(f"search {i}: wall {1e3 * (time.perf_counter() - t):.3f} ms device {r.device_ms:.3f} ms", flush=True)
