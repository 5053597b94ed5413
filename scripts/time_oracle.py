"""Time oracle_search (oracle.hpp:29-95) on the C1 room map: the device leaf
grid (bbs_oracle_search) vs the reference's oracle_search (oracle/_ref, all
host threads), same window around the ground-truth pose, results compared.
Prints one JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench
import paper_2310_10023_b200 as B
from pyoracle import Reference

cfgd = bench.CONFIGS["c1"]
m, scan, gt = bench.build_inputs(cfgd)
vm = B.MultiResVoxelMap.build(m, cfgd["r"], cfgd["max_level"])
gx, gy, gz = gt.x, gt.y, gt.z
half = float(os.environ.get("ORACLE_HALF", "1.0"))
workers = os.cpu_count()
out = []
for mode, rp, yaw in (("TRANS_ONLY", 0.0, 0.05), ("ROTO_TRANS", 0.01, 0.02)):
    y = B.normalize_angle(gt.yaw)
    cfg = B.SearchConfig(min_resolution=cfgd["r"], max_level=cfgd["max_level"],
                         roll_pitch_half_range=rp, yaw_min=y - yaw, yaw_max=y + yaw,
                         branch_mode=getattr(B.BranchMode, mode), workers=workers,
                         translation_range=((gx - half, gy - half, gz - 0.5),
                                            (gx + half, gy + half, gz + 0.5)))
    B.oracle_search(vm, scan, cfg)  # warm (LUT, allocator)
    t = time.perf_counter()
    got = B.oracle_search(vm, scan, cfg)
    dev_s = time.perf_counter() - t
    rec = dict(mode=mode, leaves=got.leaf_count, K=int(scan.shape[0]), best=got.best_score,
               n_argmax=len(got.argmax_poses), device_s=dev_s,
               device_lookups_per_s=got.leaf_count * scan.shape[0] / dev_s)
    if os.environ.get("ORACLE_NO_REF") is None:
        ref = Reference()
        rm = ref.map_build(m, cfgd["r"], cfgd["max_level"])
        t = time.perf_counter()
        best, leaves, poses = rm.oracle_search(scan, cfg.to_c())
        ref_s = time.perf_counter() - t
        rec.update(reference_s=ref_s, reference_threads=workers,
                   identical=bool(best == got.best_score and leaves == got.leaf_count and
                                  len(poses) == len(got.argmax_poses) and
                                  all(p.as_tuple() == tuple(q) for p, q in zip(got.argmax_poses, poses))),
                   speedup=ref_s / dev_s)
    out.append(rec)
    print(json.dumps(rec), flush=True)
