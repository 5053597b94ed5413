"""Dev probe: search_scan wall/device time under different timing setups."""
import os, sys, time, subprocess, statistics
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2310_10023_b200 as B
cfgd = bench.CONFIGS["c2"]
m, scan, gt = bench.build_inputs(cfgd)
cfg = bench.search_config(B, cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
ds = B.DeviceScan(vm, scan)
def run(tag, n=5):
    w, d, rs = [], [], []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = B.search_scan(vm, ds, cfg)
        w.append(1e3 * (time.perf_counter() - t)); d.append(r.device_ms); rs.append(r.root_score_ms)
    print(f"{tag:40s} wall {statistics.median(w):8.2f} ms  device {statistics.median(d):8.2f}  root {statistics.median(rs):7.2f}  init {r.stats.initial_nodes_ms:7.2f}", flush=True)
for _ in range(3): B.search_scan(vm, ds, cfg)
run("own stream, no sampler")
for ms in (100, 200, 1000):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv,noheader", "-lms", str(ms)], stdout=subprocess.DEVNULL)
    time.sleep(0.5); run(f"own stream, nvidia-smi -lms {ms}"); p.terminate(); p.wait()
run("own stream, no sampler (again)")
s = torch.cuda.Stream(); torch.cuda.set_stream(s); vm.set_stream(s.cuda_stream)
run("torch side stream")
