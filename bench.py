#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 batched BnB scan matcher.

Workload (BASELINE.json configs[1], SURVEY §8d "C2 campus"): one global
localization of a K=10,000-point scan against a ~5M-point synthetic campus map
(gen_scene 300x300x30 m, 60 boxes; r = 0.2 m, l_max = 5 (6 levels), full yaw,
roll/pitch +-0.02 rad, BFS, RotoTrans, b = 10,000, threshold 0.95).  A "step"
is one search() (root batch + every flush epoch until the queue drains).

  value   candidate score evals/s = W / max-rank device time of the K timed
          steps (CUDA events on the search stream, scan and map resident in
          HBM; L2 flushed before every step).  W = the single-queue search's
          nodes_generated (= the reference's, checked against the golden), so
          at N > 1 the work is held at the N = 1 amount (strong scaling)
  e2e     same metric through the public host API bbs_search(): the scan is
          copied from pinned host memory and the result read back every step
          (host wall clock around each call)
  parity  the result against the reference's search() golden
          (tests/golden): exact at N = 1 and in the exact shard mode; the
          best score plus the pose within one finest voxel / angular step in
          the roots shard mode (north_star's tolerance)
  cpu_baseline / --impl reference
          the UNMODIFIED reference (oracle/_ref, bnbloc::batch_evaluate) on a
          bounded uniform sample of the same root batch, all host threads and
          one thread: evals/s; a full search's time is extrapolated from it

--gpus N without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL); the root set is sharded.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import harness as H  # noqa: E402  (synthetic inputs; not the product)

GOLDENS = {"c1": "room_search.json", "c2": "campus_search.json", "c3": "c3_search.json"}

CONFIGS = {
    # name: scene spec, seed, search params, K
    "c2": dict(workload="C2 campus: 300x300x30 m box world (~5M map pts), 10k-pt scan, "
                        "r=0.2 m, 6 levels, 360 deg yaw, +-0.02 rad roll/pitch, BFS RotoTrans b=10000",
               spec=dict(size_x=300.0, size_y=300.0, size_z=30.0, num_boxes=60, min_box_side=6.0,
                         max_box_side=30.0, min_box_height=8.0, map_spacing=0.19, scan_spacing=0.3,
                         scan_range=60.0, min_scan_points=400),
               seed=1, r=0.2, max_level=5, rp=0.02, K=10000),
    "c3": dict(workload="C3 city: 640x640x60 m box world (~30M map pts), 30k-pt scan, r=0.2 m, "
                        "7 levels, 360 deg yaw, +-5 deg roll/pitch, BFS RotoTrans b=10000",
               spec=dict(size_x=640.0, size_y=640.0, size_z=60.0, num_boxes=300, min_box_side=8.0,
                         max_box_side=40.0, min_box_height=10.0, map_spacing=0.225,
                         scan_spacing=0.3, scan_range=80.0, min_scan_points=400),
               seed=1, r=0.2, max_level=6, rp=0.0873, K=30000),
    "c4": dict(workload="C4 throughput: 64 independent 10k-pt scans against the C2 campus map "
                        "(~5M pts), bbs_search_scans with 16 searches in flight, BFS RotoTrans b=10000",
               spec=dict(size_x=300.0, size_y=300.0, size_z=30.0, num_boxes=60, min_box_side=6.0,
                         max_box_side=30.0, min_box_height=8.0, map_spacing=0.19, scan_spacing=0.3,
                         scan_range=60.0, min_scan_points=400),
               seed=1, r=0.2, max_level=5, rp=0.02, K=10000, n_scans=64, streams=16),
    "c1": dict(workload="C1 room: 20x20x4 m (~200k map pts), 2k-pt scan, r=0.1 m, 6 levels, "
                        "360 deg yaw, +-5 deg roll/pitch, BFS RotoTrans b=10000",
               spec=dict(size_x=20.0, size_y=20.0, size_z=4.0, num_boxes=8, min_box_side=1.0,
                         max_box_side=4.0, min_box_height=1.0, map_spacing=0.058, scan_spacing=0.1,
                         scan_range=10.0, min_scan_points=400),
               seed=1, r=0.1, max_level=5, rp=0.0873, K=2000),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    polling thread (~1 ms period, so even a few-ms region gets samples);
    nvidia-smi -lms 100 when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, sm_max_mhz, reason bits)
        self.proc = None
        self.lines = []
        self.thread = None
        self.stop_flag = threading.Event()
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # the NVML handle of THIS CUDA device (NVML indexes by PCI order)
                import torch
                pr = torch.cuda.get_device_properties(self.device)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:  # noqa: BLE001
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, smax, rs))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.001)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.nvml = None
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            sm = [x[0] for x in self.samples]
            bits = [(n, getattr(self.nvml, a)) for n, a in self.REASONS]
            reasons = sorted({n for _, _, rs in self.samples for n, bit in bits if rs & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self.samples[0][1] if self.samples else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def build_inputs(cfgd):
    """The workload's map and K-point scan from the harness's gen_scene
    restatement (bit-identical to the reference's, tests/test_host.py)."""
    spec = H.SceneSpec.default(**cfgd["spec"])
    t = time.time()
    map_pts, raw_scan, gt = H.gen_scene(spec, cfgd["seed"])
    scan = H.cut_scan(raw_scan, min(cfgd["K"], raw_scan.shape[0]), 7)
    log(f"scene: {map_pts.shape[0]} map pts, raw scan {raw_scan.shape[0]}, K={scan.shape[0]} "
        f"({time.time() - t:.1f}s)")
    return map_pts, scan, gt


def config_dict(cfgd, K, map_points):
    """The `config` object of BOTH arms (identical keys and values)."""
    return {"workload": cfgd["workload"], "K": int(K), "map_points": int(map_points),
            "r": cfgd["r"], "levels": cfgd["max_level"] + 1, "roll_pitch_half_range": cfgd["rp"],
            "strategy": "BFS", "branch_mode": "RotoTrans", "batch_size": 10000,
            "l2": "flushed (256 MiB write) before every timed step; the reference arm runs on "
                  "host cores"}


def search_config(B, cfgd):
    return B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                          roll_pitch_half_range=cfgd["rp"], strategy=B.Strategy.BFS,
                          branch_mode=B.BranchMode.ROTO_TRANS, batch_size=10000)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def golden_search(config):
    """The reference's search() result for this workload (tests/golden, made
    by running oracle/_ref: tests/golden/make_golden.py, make_scale_goldens.py)."""
    name = GOLDENS.get(config)
    if not name:
        return None
    try:
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)["bfs_roto_b10000"]
    except (OSError, KeyError, ValueError):
        return None


class RefSampler:
    """The UNMODIFIED reference (oracle/_ref) on bounded uniform samples of
    the workload's root batch (search.hpp:111-124 scores every root with
    batch_evaluate; ~98% of a C2 search's evaluations are roots)."""

    def __init__(self, map_pts, scan, cfgd, log_prefix=""):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from pyoracle import Reference, default_config  # noqa: E402  (reference / cpu_baseline legs only)
        self.ref = Reference()
        t = time.time()
        self.rmap = self.ref.map_build(map_pts, cfgd["r"], cfgd["max_level"], 0.3, 16 << 30)
        log(f"{log_prefix}reference map build (collision_target 0.3): {time.time() - t:.1f}s")
        self.cfg = default_config(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                                  roll_pitch_half_range=cfgd["rp"])
        self.scan = scan
        self.d_max = self.ref.max_range(scan)
        self.roots = self.ref.initial_nodes(self.cfg, self.d_max, self.rmap.bbox(), cap=1 << 25)
        self.rng = np.random.default_rng(11)

    def time_sample(self, n, workers):
        sample = self.roots[self.rng.choice(self.roots.shape[0], size=min(n, self.roots.shape[0]),
                                            replace=False)]
        t = time.time()
        self.rmap.batch_evaluate(self.scan, self.cfg, sample, d_max=self.d_max, workers=workers)
        return sample.shape[0], time.time() - t

    def size_for(self, target_s, workers):
        """Sample size whose batch_evaluate takes ~target_s seconds."""
        n = 256
        while True:
            m, dt = self.time_sample(n, workers)
            if dt >= 0.25 * target_s or m >= self.roots.shape[0]:
                return max(1, min(self.roots.shape[0], int(m * target_s / max(dt, 1e-6))))
            n = int(min(self.roots.shape[0], n * max(2.0, 0.3 * target_s / max(dt, 1e-3))))

    def baseline(self, target_s, work_evals):
        """cpu_baseline: all host threads and one thread, with the full
        search's time extrapolated from the measured rate."""
        cores = os.cpu_count() or 1
        n = self.size_for(target_s, cores)
        m, dt = self.time_sample(n, cores)
        v_all = m / dt
        n1 = self.size_for(max(1.0, target_s / 4), 1)
        m1, dt1 = self.time_sample(n1, 1)
        v_one = m1 / dt1
        return {
            "value": v_all, "unit": "evals/s", "cores": cores, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": (f"{m} root nodes drawn uniformly from initial_nodes() of the workload "
                       f"(level {self.cfg.max_level}, K={self.scan.shape[0]}), bnbloc::batch_evaluate "
                       f"with workers={cores} (oracle/_ref); {dt:.1f} s"),
            "workers_1": {"value": v_one, "unit": "evals/s", "cores": 1,
                          "sample": f"{m1} root nodes, workers=1; {dt1:.1f} s"},
            "extrapolated_search_s": {
                "all_threads": work_evals / v_all if work_evals else None,
                "one_thread": work_evals / v_one if work_evals else None,
                "note": "EXTRAPOLATION: the search's nodes_generated divided by the sampled "
                        "root-batch rate (roots are ~98% of a C2 search's evaluations); not a "
                        "timed full search"},
        }


def run_reference_arm(args, cfgd):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference by oracle/Makefile) on the box's host
    cores.  Loads NO library of this repo's product: inputs come from the
    reference's own gen_scene (oracle/_ref) and a pure-Python cut."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference  # noqa: E402
    ref = Reference()
    spec = ref.default_spec()
    for k, v in cfgd["spec"].items():
        setattr(spec, k, v)
    t = time.time()
    map_pts, raw, _ = ref.gen_scene(spec, cfgd["seed"])
    scan = H.cut_scan_py(raw, min(cfgd["K"], raw.shape[0]), 7)
    log(f"reference scene: {map_pts.shape[0]} map pts, K={scan.shape[0]} ({time.time() - t:.1f}s)")
    rs = RefSampler(map_pts, scan, cfgd)
    cores = os.cpu_count() or 1
    n = rs.size_for(args.ref_step_seconds, cores)
    vals, t_all, n_all = [], 0.0, 0
    for step in range(args.warmup + args.steps):
        m, dt = rs.time_sample(n, cores)
        if step >= args.warmup:
            vals.append(m / dt)
            t_all += dt
            n_all += m
    value = n_all / t_all
    g = golden_search(args.config)
    work = g["nodes_generated"] if g else None
    sample_desc = (f"{n} root nodes per step drawn uniformly from initial_nodes() of the workload "
                   f"(level {cfgd['max_level']}), bnbloc::batch_evaluate with workers={cores}")
    line = {
        "impl": "reference", "metric": "candidate score evals/sec", "value": value,
        "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's own gen_scene, oracle/_ref)",
        "config": config_dict(cfgd, scan.shape[0], map_pts.shape[0]),
        "parallelism": f"host threads x{cores} (parallel_chunks, parallel.hpp:16-42)",
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": sample_desc},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated_search_s": (work / value) if work else None,
        "extrapolation": "a full search() = the golden's nodes_generated / this rate (EXTRAPOLATION, "
                         "not a timed search)",
    }
    print(json.dumps(line), flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def profile_summary(config):
    """ncu evidence committed under profiles/ (scripts/traffic.py): DRAM
    bytes per launch and speed-of-light percentages per kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(config, {})
    except (OSError, ValueError):
        return {}


def pose_parity(res, want, grids, r, exact):
    """north_star: best score equal; pose equal, or (roots shard mode, where
    the RotoTrans schedule legitimately differs) within one finest-level
    voxel and one finest angular step."""
    got = list(res.best_pose.as_tuple())
    out = {"best_score": res.best_score, "golden_best_score": want["best_score"],
           "score_ok": res.best_score == want["best_score"]}
    if got == want["best_pose"]:
        out["pose"] = "exact"
    elif exact:
        out["pose"] = "DIFFERS"
    else:
        d = [abs(a - b) for a, b in zip(got, want["best_pose"])]
        d[5] = min(d[5], 2 * math.pi - d[5])
        steps = [grids.axis(a, 0).step for a in range(3)]
        ok = all(x <= r * (1 + 1e-9) for x in d[:3]) and all(
            d[3 + a] <= steps[a] * (1 + 1e-9) for a in range(3))
        out["pose"] = "within one finest voxel / angular step" if ok else "OUT OF TOLERANCE"
    if exact:
        out["stats_ok"] = (res.stats.nodes_generated, res.stats.nodes_pruned,
                           res.stats.batches_flushed) == (want["nodes_generated"], want["nodes_pruned"],
                                                          want["batches_flushed"])
    out["ok"] = out["score_ok"] and out["pose"] != "DIFFERS" and out["pose"] != "OUT OF TOLERANCE" \
        and out.get("stats_ok", True)
    return out


def run_b200_arm(args, cfgd):
    import torch
    world, rank, local = dist_env()
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, only {torch.cuda.device_count()} visible "
                         f"(--gpus N needs N GPUs on this node)")
    torch.cuda.set_device(local)
    # BBS_BENCH_SHARDED=1 takes the sharded path at world 1 too (torchrun
    # --nproc-per-node 1): a one-GPU check of the NCCL glue
    sharded = world > 1 or os.environ.get("BBS_BENCH_SHARDED") == "1"
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2310_10023_b200 as B

    map_pts, scan, gt = build_inputs(cfgd)
    cfg = search_config(B, cfgd)
    stream = torch.cuda.current_stream()
    vmap = B.MultiResVoxelMap.build(map_pts, cfgd["r"], cfgd["max_level"],
                                    layout=B.Layout[args.layout.upper()], device=local)
    build_ms = vmap.build_ms()
    vmap.set_stream(stream.cuda_stream)
    layouts = [vmap.level(l).layout().name for l in range(cfgd["max_level"] + 1)]
    level_bytes = [vmap.level(l).device_bytes() for l in range(cfgd["max_level"] + 1)]
    log(f"rank {rank}: map build {build_ms:.1f} ms device, layouts {layouts}, bytes {level_bytes}")
    dscan = B.DeviceScan(vmap, scan)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    K = int(scan.shape[0])

    # the single-queue search (= the reference's schedule): its
    # nodes_generated is the work W of one step at every N
    single = B.search_scan(vmap, dscan, cfg)
    work = int(single.stats.nodes_generated)

    if sharded:
        import torch.distributed as dist
        # the search's own NCCL communicator: incumbent / score exchanges are
        # ncclAllReduce(MAX) calls on the search stream (no host round-trip)
        uid = [B.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = B.Comm(local, rank, world, uid[0])

        def one_search(ds=None):
            return B.search_sharded(vmap, ds or dscan, cfg, rank, world, comm=comm,
                                    mode=args.shard_mode)
    else:
        # on the stream the step's events and the L2 flush are recorded on:
        # the search starts after the flush and the end event follows its
        # last kernel (on the map's own stream it overlapped the flush)
        def one_search():
            return B.search_scan(vmap, dscan, cfg, stream=stream.cuda_stream)

    def barrier():
        if sharded:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        r = one_search()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    results, step_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed iterations (outside the events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = one_search()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        results.append(r)
    barrier()
    clk = clocks.stop()
    t_local = sum(step_ms)
    executed_local = sum(r.stats.nodes_generated for r in results)
    if sharded:
        import torch.distributed as dist
        tt = torch.tensor([t_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ev = torch.tensor([executed_local], dtype=torch.int64, device="cuda")
        # exact mode: every rank reports the whole search's Stats
        dist.all_reduce(ev, op=dist.ReduceOp.MAX if args.shard_mode == "exact" else dist.ReduceOp.SUM)
        t_max, executed = float(tt.item()), int(ev.item())
    else:
        t_max, executed = t_local, executed_local
    value = work * args.steps / (t_max * 1e-3)
    r0 = results[-1]

    # ---- parity against the reference's golden search()
    want = golden_search(args.config)
    grids = B.AngularGrid(cfg, B.max_range(scan))
    exact = (not sharded) or args.shard_mode == "exact"
    if want is not None:
        parity = pose_parity(r0, want, grids, cfgd["r"], exact)
        parity["golden"] = f"tests/golden/{GOLDENS[args.config]} (reference search(), oracle/_ref)"
        parity["work_matches_golden"] = work == want["nodes_generated"]
    else:
        parity = {"golden": None, "note": "no reference golden for this config"}
    if rank == 0 and want is not None and not parity["ok"]:
        log(f"PARITY FAILURE: {parity}")

    # ---- e2e through the public host API (pinned host scan, result read back)
    pinned = torch.empty((K, 3), dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(scan))
    host_scan = pinned.numpy()
    e2e_t, h2d, d2h = 0.0, 0, 0
    if not sharded:
        B.search(vmap, host_scan, cfg)  # warm
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t = time.perf_counter()
            re = B.search(vmap, host_scan, cfg)
            e2e_t += time.perf_counter() - t
            h2d, d2h = re.h2d_bytes, re.d2h_bytes
        e2e = {"value": work * args.steps / e2e_t, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_t / args.steps,
               "timing": "host wall clock around bbs_search() (scan copied in, result read back)"}
    else:
        # sharded e2e: the scan is re-uploaded from pinned memory every step
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            t = time.perf_counter()
            ds = B.DeviceScan(vmap, host_scan)
            re = one_search(ds)
            barrier()
            e2e_t += time.perf_counter() - t
            h2d, d2h = re.h2d_bytes + 24 * K, re.d2h_bytes
        import torch.distributed as dist
        tt = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": work * args.steps / float(tt.item()), "unit": "evals/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * float(tt.item()) / args.steps,
               "timing": "host wall clock (scan upload + sharded search), max over ranks"}

    # ---- roofline of the dominant kernel: the root column kernel
    # (root_colpad_kernel, the largest single launch of a step, profiles/).
    # Algorithmic bytes = the z-column words it actually gathers from its
    # staged shared-memory window (4 B each, counted on the device): one word
    # per (translation column, de-duplicated histogram entry), which answers
    # all nz z-translations of that column at once.  Peak = the measured
    # conflict-free shared-memory read ceiling of this GPU (bbs_smem_bench).
    peaks, peak_kind = measured_peaks()
    col_ms = statistics.mean(r.root_col_ms for r in results)
    words = statistics.mean(r.root_words for r in results)
    smem_gbs = gather_l2 = gather_hbm = None
    if rank == 0 and not args.no_gather_bench:
        import ctypes as C
        out = C.c_double()
        if B.lib.bbs_smem_bench(local, C.byref(out)) == 0:
            smem_gbs = round(out.value, 1)
        for label, nbytes in (("l2", 64 << 20), ("hbm", 4 << 30)):
            if B.lib.bbs_gather_bench(local, nbytes, C.byref(out)) == 0:
                if label == "l2":
                    gather_l2 = round(out.value, 1)
                else:
                    gather_hbm = round(out.value, 1)
    achieved = (words * 4.0 / (col_ms * 1e-3) / 1e9) if col_ms > 0 else None
    prof = profile_summary(args.config)
    col_prof = prof.get("root_colpad_kernel", {})
    traffic = col_prof.get("dram_bytes_per_launch")
    roofline = {
        "bound": "smem", "kernel": "root_colpad_kernel (root batch: batch_evaluate on initial_nodes)",
        "achieved": achieved, "peak": smem_gbs, "unit": "GB/s",
        "frac": (achieved / smem_gbs) if (achieved and smem_gbs) else None,
        "traffic": traffic,
        "algorithmic_bytes_per_launch": words * 4.0,
        "kernel_ms_per_step": col_ms,
        "unit_of_work": "one 4 B z-column word gathered from the staged shared-memory window per "
                        "(translation column, de-duplicated scan-voxel offset); one word answers every "
                        "z-translation of the column",
        "peak_source": "measured in this run: bbs_smem_bench, conflict-free LDS.32 over all 148 SMs "
                       "(MEASURED_PEAKS.json has no shared-memory figure)",
        "ncu": {k: col_prof.get(k) for k in ("sm_throughput_pct", "memory_throughput_pct",
                                             "l1tex_throughput_pct", "ipc_active", "achieved_occupancy_pct",
                                             "source")},
        "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per launch)",
        # the bound that actually limits it: instruction issue (4 schedulers
        # per SM, one instruction each per cycle)
        "issue": {"ipc_active": col_prof.get("ipc_active"), "peak_ipc": 4.0,
                  "frac": (col_prof["ipc_active"] / 4.0) if col_prof.get("ipc_active") else None,
                  "note": "ncu issued IPC per active SM over the 4-wide issue peak: ~8 instructions per "
                          "gathered word (LDS, funnel shift, byte permute, LOP3 + IDP4A per z-translation)"},
        "context": {"hbm_copy_gbs": peaks.get("hbm_gbs"), "hbm_peak_source": f"MEASURED_PEAKS.json ({peak_kind})",
                    "l2_random_sector_gather_gbs": gather_l2, "hbm_random_sector_gather_gbs": gather_hbm,
                    "survey_lookup_model": {
                        "lookups_per_s": r0.lookups / (statistics.mean(step_ms) * 1e-3),
                        "note": "SURVEY §8d's per-(node, scan point) lookup count (nodes_generated x K): "
                                "an effective rate, not a traffic figure; histogram de-duplication and "
                                "column words make the kernels issue far fewer loads"}},
    }

    line = {
        "metric": "candidate score evals/sec", "value": value, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (harness gen_scene restatement, bit-identical to the reference's)",
        "config": config_dict(cfgd, K, map_pts.shape[0]),
        "parallelism": (f"{args.shard_mode}-shard x{world}, NCCL incumbent/score all-reduce on the "
                        "search stream") if sharded else "single GPU",
        "work_evals_per_step": work,
        "executed_evals_per_step": executed / args.steps,
        "latency_ms": {"localization_total": t_max / args.steps,
                       "initial_nodes": statistics.mean(r.stats.initial_nodes_ms for r in results),
                       "find_best_score": statistics.mean(r.stats.find_best_score_ms for r in results),
                       "pop_remaining_queue": statistics.mean(r.stats.pop_remaining_queue_ms
                                                              for r in results),
                       "create_voxel_maps": build_ms,
                       "note": "localization_total = max-rank device time per step (CUDA events)"},
        "search": {"best_score": r0.best_score, "matched": r0.matched,
                   "nodes_generated": r0.stats.nodes_generated, "epochs": r0.epochs,
                   "root_nodes": r0.root_nodes, "root_probes": r0.root_probes,
                   "root_words": r0.root_words, "layouts": layouts,
                   "trans_err_m": math.dist(r0.best_pose.as_tuple()[:3], gt.as_tuple()[:3])},
        "parity": parity,
        "e2e": e2e, "roofline": roofline, "clocks": clk,
        "gpu_launches": int(sum(r.kernel_launches for r in results)),
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            rs = RefSampler(map_pts, scan, cfgd, "cpu_baseline: ")
            line["cpu_baseline"] = rs.baseline(args.cpu_seconds, work)
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "evals/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if sharded:
        torch.cuda.synchronize()
        comm.close()
        torch.distributed.destroy_process_group()
    if want is not None and exact and not parity["ok"]:
        sys.exit(3)  # the single-queue schedule must equal the reference exactly


def run_b200_throughput(args, cfgd):
    """C4: many independent scans against one map.  Each rank (replicas only,
    scans j % world == rank) runs its scans on `streams` concurrent CUDA
    streams (one host thread each; every search leases its own workspace)."""
    import threading

    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2310_10023_b200 as B
    spec = H.SceneSpec.default(**cfgd["spec"])
    t = time.time()
    map_pts, _, _ = H.gen_scene(spec, cfgd["seed"])
    scans, poses = H.gen_scans(spec, cfgd["seed"], 1000, cfgd["n_scans"])
    scans = [H.cut_scan(s, min(cfgd["K"], s.shape[0]), 7) for s in scans]
    log(f"scene + {len(scans)} scans: {time.time() - t:.1f}s")
    mine = [j for j in range(len(scans)) if j % world == rank]
    cfg = search_config(B, cfgd)
    vmap = B.MultiResVoxelMap.build(map_pts, cfgd["r"], cfgd["max_level"], device=local)
    dscans = {j: B.DeviceScan(vmap, scans[j]) for j in mine}
    T = int(os.environ.get("BBS_BENCH_STREAMS", cfgd["streams"]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def batch(host=False):
        if host:  # the public host API, one scan at a time (bbs_search copies in/out)
            return {j: B.search(vmap, scans[j], cfg) for j in mine}
        # throughput mode: bbs_search_scans keeps T searches in flight on
        # native worker threads, one stream each (no Python in the loop)
        res = B.search_scans(vmap, [dscans[j] for j in mine], cfg, concurrency=T)
        return dict(zip(mine, res))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        batch()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms, evals, res = [], 0, {}
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = batch()
        torch.cuda.synchronize()  # all streams done before the end event
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        evals += sum(r.stats.nodes_generated for r in res.values())
    barrier()
    clk = clocks.stop()
    t_local = sum(step_ms)
    # e2e: the throughput-mode public API from pinned host scans -- every scan
    # uploaded (bbs_scan_upload), bbs_search_scans, results read back; the
    # sequential bbs_search() loop is reported beside it
    pinned = {}
    for j in mine:
        p = torch.empty(scans[j].shape, dtype=torch.float64, pin_memory=True)
        p.copy_(torch.from_numpy(scans[j]))
        pinned[j] = p.numpy()
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    up = [B.DeviceScan(vmap, pinned[j]) for j in mine]
    res_h = dict(zip(mine, B.search_scans(vmap, up, cfg, concurrency=T)))
    e2e_s = time.perf_counter() - t0
    del up
    e2e_evals = sum(r.stats.nodes_generated for r in res_h.values())
    t0 = time.perf_counter()
    res_seq = batch(host=True)
    seq_s = time.perf_counter() - t0
    seq_evals = sum(r.stats.nodes_generated for r in res_seq.values())
    if world > 1:
        import torch.distributed as dist
        v = torch.tensor([t_local, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        c = torch.tensor([evals, e2e_evals], dtype=torch.int64, device="cuda")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        t_max, e2e_s = float(v[0]), float(v[1])
        evals, e2e_evals = int(c[0]), int(c[1])
    else:
        t_max = t_local
    ok = 0
    for j, r in res.items():
        g = poses[j]
        if r.matched and math.dist(r.best_pose.as_tuple()[:3], g.as_tuple()[:3]) < 2.0:
            ok += 1
    line = {
        "metric": "candidate score evals/sec", "value": evals / (t_max * 1e-3), "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (harness gen_scene restatement, bit-identical to the reference's)",
        "config": {"workload": cfgd["workload"], "scans": len(scans), "K": cfgd["K"],
                   "parallelism": f"replicas x{world}, {T} concurrent searches per GPU (bbs_search_scans)",
                   "l2": "flushed (256 MiB write) before every timed step"},
        "scans_per_s": len(scans) * args.steps / (t_max * 1e-3),
        "success_within_2m_rank0": f"{ok}/{len(res)}",
        "e2e": {"value": e2e_evals / e2e_s, "unit": "evals/s",
                "h2d_bytes_per_step": int(sum(24 * scans[j].shape[0] for j in mine)),
                "d2h_bytes_per_step": int(sum(r.d2h_bytes for r in res_h.values())),
                "timing": "host wall clock (rank max): pinned host scans uploaded with bbs_scan_upload, "
                          "bbs_search_scans, results read back",
                "sequential_bbs_search": {"value": seq_evals / seq_s, "unit": "evals/s"}},
        "clocks": clk, "gpu_launches": int(sum(r.kernel_launches for r in res.values())) * args.steps,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def spawn_ranks(args):
    """--gpus N outside torchrun: re-launch this script as N ranks, one per
    GPU, under torch.distributed.run (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    log("launching: " + " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--layout", choices=["auto", "bitmap", "hash"], default="auto")
    ap.add_argument("--shard-mode", choices=["roots", "exact"], default="roots",
                    help="N>1: roots = own BnB per rank over its root share + incumbent "
                         "all-reduce; exact = batch-split replay of the single-queue schedule")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="cpu_baseline: seconds of reference work per leg")
    ap.add_argument("--ref-step-seconds", type=float, default=6.0,
                    help="--impl reference: seconds of reference work per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gather-bench", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (contract minimum)")
        args.warmup = 3
    cfgd = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference_arm(args, cfgd)
    elif "n_scans" in cfgd:
        run_b200_throughput(args, cfgd)
    else:
        run_b200_arm(args, cfgd)


if __name__ == "__main__":
    main()
