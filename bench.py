"""Benchmark: rays/s integrated into a region-chunked voxel map on B200.

Default workload = BASELINE.json configs[1] ("C2"): a synthetic Ouster-128
sequence, 1000 batches x 26,240 rays (26.24 M rays), 0.05 m voxels,
occupancy (+ sub-voxel mean), deterministic sort+segmented update path.
One step = the whole 1000-batch sequence integrated into a freshly cleared
map (region creation included), batch by batch, exactly as 1000
`submit_batch` calls would do it.

  value  inputs resident in HBM (OHMB1 records), timed with CUDA events on
         the map's stream, max over ranks
  e2e    the same through the public API `submit_batch(vmap, records)` with
         pinned HOST records: host->device copy of every batch and the
         device->host stats read inside the timed region

N > 1 (torchrun): ONE region-sharded map over all ranks (sharded.py,
SURVEY.md 8(e)), weak scaling: N copies of the scene in parallel streets,
merged batch by batch; each rank walks 1/N of every batch, owns 1/N of the
regions and receives its regions' miss counts / ordered records over NCCL
all-to-all (`--replicas`: independent per-GPU maps instead).
`--impl reference` times the reference's own native kernel on the host
cores instead (oracle/ref_runner.py).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "rays/s integrated (occupancy & NDT-OM, 0.1 m voxels) at 1/2/4/8 B200 vs CPU"
UNIT = "rays/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("c2", "c2_01", "c1", "c3", "c4", "c5"), default="c2")
    ap.add_argument("--exec", dest="exec_", choices=("det", "cas"), default="det")
    ap.add_argument("--batches", type=int, default=1000, help="C2 batches per step")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-batch", action="store_true",
                    help="one vm_integrate / submit_batch call per batch instead of one "
                         "pipelined vm_integrate_many / submit_batches call per step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="default run: skip the NDT-OM (C3) and C1 blocks and the CPU sweep")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent per-GPU maps instead of the region-sharded map")
    return ap.parse_args()


def workload(name: str, batches: int):
    from paper_2206_06079_b200 import MapConfig, scans
    if name == "c2":
        cfg = MapConfig(voxel_size=0.05)
        scan_list = scans.os128_canyon_batches(batches)
        # replayed in the reference CLI's 0.1 s batches (cli.py:31,70-94)
        data = scans.batch_by_period(np.concatenate(scan_list))
        desc = dict(workload="C2: synthetic OS1-128 street-canyon sequence", scans=len(scan_list),
                    rays_per_scan=int(len(scan_list[0])), batches=len(data),
                    batch_period_s=scans.BATCH_PERIOD, rays_per_batch=int(len(data[0])),
                    voxel_size=0.05, region_dim=32, mode="occupancy")
        mode = "occupancy"
    elif name == "c2_01":
        # the north_star target's case: sustained 0.1 m occupancy integration
        # (C2's OS1-128 sequence and batching, at 0.1 m voxels)
        cfg = MapConfig(voxel_size=0.1)
        scan_list = scans.os128_canyon_batches(batches)
        data = scans.batch_by_period(np.concatenate(scan_list))
        desc = dict(workload="C2 sequence at 0.1 m: synthetic OS1-128 street canyon",
                    scans=len(scan_list), rays_per_scan=int(len(scan_list[0])), batches=len(data),
                    batch_period_s=scans.BATCH_PERIOD, rays_per_batch=int(len(data[0])),
                    voxel_size=0.1, region_dim=32, mode="occupancy")
        mode = "occupancy"
    elif name == "c1":
        cfg = MapConfig(voxel_size=0.1)
        data = [scans.os64_room_scan()]
        desc = dict(workload="C1: one synthetic OS1-64 scan", scans=1, rays_per_batch=131072,
                    voxel_size=0.1, region_dim=32, mode="occupancy")
        mode = "occupancy"
    elif name == "c3":
        cfg = MapConfig(voxel_size=0.1)
        data = scans.os64_tunnel_scans(77)
        desc = dict(workload="C3: synthetic OS1-64 tunnel, NDT-OM", scans=77,
                    rays_per_batch=131072, voxel_size=0.1, region_dim=32, mode="ndt-om")
        mode = "ndt-om"
    elif name == "c4":
        # configs[3]: TSDF + decay at 0.05 m from the UAV; a bounded prefix of
        # the 382-scan flight (the modes alternate per batch on one map)
        cfg = MapConfig(voxel_size=0.05)
        data = scans.uav_lawnmower_scans(min(batches, 40))
        desc = dict(workload="C4: synthetic UAV lawnmower, TSDF then decay per scan",
                    scans=len(data), of_scans=scans.UAV_SCANS, rays_per_batch=131072,
                    voxel_size=0.05, region_dim=32, mode="tsdf+decay")
        mode = "tsdf+decay"
    else:
        # configs[4]: NDT-OM at 0.1 m through the procedural town; a bounded
        # window of the 7,630-scan loop (any window regenerates on its own)
        cfg = MapConfig(voxel_size=0.1)
        data = scans.town_scans(0, min(batches, 77))
        desc = dict(workload="C5: synthetic town loop, NDT-OM", scans=len(data),
                    of_scans=scans.TOWN_SCANS, rays_per_batch=131072, voxel_size=0.1,
                    region_dim=32, mode="ndt-om")
        mode = "ndt-om"
    return cfg, mode, data, desc


def sample_clocks(path: str):
    cmd = ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
           "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
           "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
           "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"]
    try:
        return subprocess.Popen(cmd, stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except FileNotFoundError:
        return None


def parse_clocks(path: str, dev: int):
    sm, mx, reasons = [], 0.0, set()
    names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    try:
        for line in open(path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) != dev:
                continue
            sm.append(float(f[1]))
            mx = max(mx, float(f[2]))
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
    except (OSError, ValueError):
        pass
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
            "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(S, V, H):
    """SURVEY.md 8(d) occupancy: 49 B per segment input + 8 B per miss visit
    (f32 log-odds RMW) + 24 B per hit (log-odds + packed mean + count RMW)."""
    return 49 * S + 8 * (V - H) + 24 * H


def load_peaks():
    try:
        d = json.load(open(ROOT / "MEASURED_PEAKS.json"))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload_name, exec_):
    """dram bytes per walk launch from the committed ncu capture, if any."""
    try:
        d = json.load(open(ROOT / "profiles" / "ncu_summary.json"))
        return d.get(f"{workload_name}_{exec_}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def best_workers(cfg, data):
    """The reference kernel's fastest thread count on this host: one batch
    per W in {1, 2, 4, ..., cores} (its thread scaling is not monotone --
    the sensor voxel's CAS hot spot, SURVEY finding 2)."""
    from oracle import oracle as orc
    from oracle import ref_runner
    cores = orc.host_cores()
    best, best_w = 0.0, cores
    for w in sorted({w for w in (1, 2, 4, 8, 16, 32, 64) if w <= cores} | {cores}):
        t = ref_runner.time_reference(cfg, data[:1], w, budget_s=0.0)
        rate = t["rays"] / t["seconds"] if t["seconds"] else 0.0
        if rate > best:
            best, best_w = rate, w
    return best_w


def cpu_baseline(cfg, data, budget, mode):
    from oracle import ref_runner
    if mode != "occupancy":
        return None
    workers = best_workers(cfg, data)
    r = ref_runner.time_reference(cfg, data, workers, budget_s=budget)
    return {"value": r["rays"] / r["seconds"], "unit": UNIT, "cores": workers,
            "kind": r["kind"],
            "sample": f"first {r['batches']} batches ({r['rays']} rays, {r['visits']} voxel "
                      f"visits) of the same workload; reference _kernels.integrate_occupancy "
                      f"on {workers} threads (the fastest W of a 1..cores probe), kernel-only "
                      f"(clip/segment/prefetch untimed)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, mode, data, desc = workload(args.workload, args.batches)
    from oracle import ref_runner
    workers = best_workers(cfg, data)
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        ref_runner.time_reference(cfg, data[:2], workers, budget_s=budget / 4)
    rays = secs = 0.0
    used = 0
    for _ in range(args.steps):
        r = ref_runner.time_reference(cfg, data, workers, budget_s=budget)
        rays += r["rays"]
        secs += r["seconds"]
        used = r["batches"]
        kind = r["kind"]
    value = rays / secs if secs else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32", "data": "synthetic",
        "config": desc,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
                         "sample": f"each step: first {used} batches of the workload, "
                                   f"reference native kernel, {workers} threads (the fastest "
                                   f"W of a 1..cores probe)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _h_and_u(host, cfg, sizes):
    """H (sample segments: has_sample rays within max range) and U (distinct
    sample voxels, summed over batches) of a record sequence -- the SURVEY
    8(d) byte-model terms the device does not count."""
    o = host["origin"].astype(np.float64)
    e = host["end"].astype(np.float64)
    L = np.sqrt(((e - o) ** 2).sum(1))
    smp = ((host["flags"] & 1) == 1) & (L <= cfg.max_ray_range) & (L > 0)
    H = int(np.sum(smp))
    U = 0
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for b in range(len(sizes)):
        sl = slice(offs[b], offs[b + 1])
        g = np.floor(e[sl][smp[sl]] / cfg.voxel_size).astype(np.int64)
        if len(g):
            U += len(np.unique(g, axis=0))
    return H, U


def ndt_bytes(S, V, H, V3, U):
    """SURVEY.md 8(d) NDT-OM: phase 1 reads count + RMW log-odds per visit
    (12 B), + mean and cov when the voxel holds a Gaussian (40 B); phase 2
    reads each sample (24 B) and RMWs log-odds, mean, count, cov per
    distinct sample voxel (72 B).  Returns (walk bytes, fold bytes)."""
    return 49 * S + 12 * (V - H - V3) + 40 * V3, 24 * H + 72 * U


def run_gpu_workload(name, args, dev, torch, world=1, dist=None, steps=None, e2e_steps=3,
                     det=True):
    """One workload on this GPU: device-resident `value`, host-record `e2e`,
    stage times and the byte model.  A step integrates the workload's whole
    batch sequence into a freshly cleared map."""
    from paper_2206_06079_b200 import (ExecutorOptions, VoxelMap, _native, submit_batch,
                                       submit_batches)
    from paper_2206_06079_b200.layers import MODE_LAYERS

    steps = steps or args.steps
    cfg, mode, data, desc = workload(name, args.batches)
    sizes = [len(b) for b in data]
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    total_rays = int(offsets[-1])
    host = np.concatenate(data)
    d_rec = torch.from_numpy(host.view(np.uint8).copy()).to(f"cuda:{dev}")
    base = d_rec.data_ptr()
    stream = torch.cuda.current_stream()
    # C4 alternates two modes per batch on one map (test_acceptance.py:398-399)
    modes = mode.split("+")
    names = tuple(dict.fromkeys(sum((MODE_LAYERS[x] for x in modes), ())))
    vmap = VoxelMap(cfg, names, device=dev, initial_regions=4096)
    vmap._native.set_stream(stream.cuda_stream)
    keys = ("discover_ms", "walk_ms", "resolve_ms", "sort_ms", "fold_ms", "gpu_ms")

    def step(record=False):
        vmap.clear()
        tot = dict(S=0, V=0, launches=0, batches=0, records=0, rmiss=0, **{k: 0.0 for k in keys})
        rays = [_native.rays_from_records(sizes[b], base + int(offsets[b]) * 40)
                for b in range(len(data))]
        if len(modes) > 1:
            sts = [vmap._native.integrate(r, x, det) for r in rays for x in modes]
        elif args.per_batch:
            sts = [vmap._native.integrate(r, mode, det) for r in rays]
        else:
            sts = vmap._native.integrate_many(rays, mode, det)
        if record:
            for st in sts:
                tot["S"] += st.segments
                tot["V"] += st.voxel_visits
                tot["launches"] += st.launches
                tot["records"] += st.records
                tot["rmiss"] += st.region_misses
                tot["batches"] += 1
                for k in keys:
                    tot[k] += getattr(st, k)
        return tot

    for _ in range(args.warmup):
        step()
    clk_file = tempfile.mktemp(suffix=".csv")
    clk = sample_clocks(clk_file)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs = [step(record=True) for _ in range(steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if clk:
        clk.terminate()
        clk.wait()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    e2e = None
    if e2e_steps:
        pinned = torch.from_numpy(host.view(np.uint8).copy()).pin_memory()
        hv = pinned.numpy().view(host.dtype)
        opts = ExecutorOptions(deterministic=det)
        slices = [hv[offsets[b]:offsets[b + 1]] for b in range(len(data))]

        def run_e2e(batches):
            if len(modes) > 1:
                for x in batches:
                    for md in modes:
                        submit_batch(vmap, x, md, opts)
            elif args.per_batch or len(batches) == 1:
                for x in batches:
                    submit_batch(vmap, x, mode, opts)
            else:
                submit_batches(vmap, batches, mode, opts)

        vmap.clear()
        run_e2e(slices[:50])
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e2e_steps):
            vmap.clear()
            run_e2e(slices)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = max(f0.elapsed_time(f1), (time.perf_counter() - t0) * 1e3)
        if os.environ.get("VOXMAP_B200_E2E_DEBUG"):
            print(f"[e2e] {name}: device {f0.elapsed_time(f1):.2f} ms, wall "
                  f"{(time.perf_counter() - t0) * 1e3:.2f} ms for {e2e_steps} steps", file=sys.stderr)
        if dist:
            t = torch.tensor([ems], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        pageable = None
        if name == "c2" and not args.per_batch:
            # the same through ordinary (pageable) numpy records: the driver
            # stages each copy through its own pinned buffer
            pslices = [host[offsets[b]:offsets[b + 1]] for b in range(len(data))]
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            vmap.clear()
            run_e2e(pslices)
            torch.cuda.synchronize()
            pageable = total_rays / (time.perf_counter() - t1)
        e2e = {"value": total_rays * e2e_steps * world / (ems * 1e-3), "unit": UNIT,
               "pageable_value": pageable,
               "h2d_bytes_per_step": int(host.nbytes),
               "d2h_bytes_per_step": int(len(data) * ctypes_stats_bytes()),
               "steps": e2e_steps,
               "api": ("submit_batch(vmap, pinned OHMB1 records) per batch"
                       if args.per_batch or len(data) == 1 else
                       f"submit_batches(vmap, [pinned OHMB1 records per batch]) ({mode})")}
    H, U = _h_and_u(host, cfg, sizes)
    s0 = recs[-1]
    del d_rec
    return dict(cfg=cfg, mode=mode, desc=desc, total_rays=total_rays, ms=ms, steps=steps,
                value=total_rays * steps * world / (ms * 1e-3), e2e=e2e, s0=s0, H=H, U=U,
                launches=int(sum(r["launches"] for r in recs)), clocks=parse_clocks(clk_file, dev),
                data=data)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        # VM_DIST_BACKEND=gloo lets the sharded protocol run with more ranks
        # than GPUs (exchanges staged through host memory) -- for testing only
        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        dist.init_process_group(os.environ.get("VM_DIST_BACKEND", "nccl"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    if world > 1 and not args.replicas and args.workload in ("c1", "c2", "c3", "c5") and \
            args.exec_ == "det":
        run_sharded(args, world, rank, dev, dist)
        dist.destroy_process_group()
        return

    from paper_2206_06079_b200 import _native

    det = args.exec_ == "det"
    r = run_gpu_workload(args.workload, args, dev, torch, world, dist,
                         e2e_steps=0 if args.no_e2e else max(1, min(args.steps, 3)), det=det)
    cfg, mode, s0 = r["cfg"], r["mode"], r["s0"]
    peak, peak_kind = load_peaks()
    red_peak = _native.probe_red_rate(dev, 64 << 20, 5)
    walk_ms = s0["walk_ms"] / max(1, s0["batches"])
    if mode == "occupancy":
        bytes_launch = algorithmic_bytes(s0["S"], s0["V"], r["H"]) / max(1, s0["batches"])
        kernel = "k_walk_det" if det else "k_walk"
    elif mode == "tsdf+decay":
        # TSDF 49 S_sample + 16 V_band, decay B_occ + 16 V + 8 H (both
        # passes' visits are summed in V; the byte figure is a lower bound)
        bytes_launch = (algorithmic_bytes(s0["S"], s0["V"], r["H"]) + 16 * s0["V"]) / max(1, s0["batches"])
        kernel = "k_walk (tsdf, decay)"
    else:
        wb, _ = ndt_bytes(s0["S"], s0["V"], r["H"], s0["records"] - r["H"], r["U"])
        bytes_launch = wb / max(1, s0["batches"])
        kernel = "k_walk_ndt_det" if det else "k_walk_ndt"
    achieved = bytes_launch / (walk_ms * 1e-3) / 1e9 if walk_ms > 0 else 0.0
    visits_launch = s0["V"] / max(1, s0["batches"])
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
            "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["ms"] / r["steps"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (DDA) / f32 (log-odds)", "data": "synthetic",
            "config": dict(r["desc"], exec="deterministic" if det else "cas",
                           rays_per_step=r["total_rays"], parallelism=f"replicas{world}",
                           l2="inputs and map exceed L2; map cleared each step"),
            "voxel_updates_per_s": s0["V"] * r["steps"] * world / (r["ms"] * 1e-3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(args.workload, args.exec_),
                         "kernel": kernel, "peak_kind": peak_kind,
                         "bytes_per_launch": bytes_launch, "avg_launch_ms": walk_ms},
            # the walk's real ceiling: one atomic update per visit; peak = this
            # GPU's measured RED.ADD rate at L2-resident random addresses
            "roofline_l2_atomic": {"bound": "l2-atomic", "kernel": kernel,
                                   "achieved": visits_launch / (walk_ms * 1e-3) if walk_ms else 0.0,
                                   "peak": red_peak, "unit": "updates/s",
                                   "frac": (visits_launch / (walk_ms * 1e-3) / red_peak)
                                   if walk_ms and red_peak else None,
                                   "peak_kind": "measured (vm_probe_red_rate, 64 MiB footprint)"},
            "e2e": r["e2e"],
            "cpu_baseline": None,
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "stats": {"segments": s0["S"], "visits": s0["V"], "hits": r["H"],
                      "records": s0["records"], "region_misses": s0["rmiss"]},
            "stages_ms_per_step": {k: round(s0[k], 4) for k in (
                "discover_ms", "walk_ms", "resolve_ms", "sort_ms", "fold_ms", "gpu_ms")},
        }
    default_run = args.workload == "c2" and det and world == 1 and not args.per_batch
    if default_run and not args.no_extra:
        # the NDT-OM half of the metric (configs[2], C3) and the 0.1 m
        # occupancy scan (configs[0], C1), measured in the same run
        n = run_gpu_workload("c3", args, dev, torch, steps=min(args.steps, 3), e2e_steps=3)
        ns = n["s0"]
        V3 = ns["records"] - n["H"]
        wb, fb = ndt_bytes(ns["S"], ns["V"], n["H"], V3, n["U"])
        nb = max(1, ns["batches"])
        nwalk = ns["walk_ms"] / nb
        c1 = run_gpu_workload("c1", args, dev, torch, steps=50, e2e_steps=20)
        o1 = run_gpu_workload("c2_01", args, dev, torch, steps=min(args.steps, 5), e2e_steps=3)
        if rank == 0:
            o1s = o1["s0"]
            o1_walk = o1s["walk_ms"] / max(1, o1s["batches"])
            o1_bytes = algorithmic_bytes(o1s["S"], o1s["V"], o1["H"]) / max(1, o1s["batches"])
            line["occ_0p1m"] = {
                "workload": o1["desc"]["workload"], "config": o1["desc"], "value": o1["value"],
                "unit": UNIT, "ms_per_step": o1["ms"] / o1["steps"], "steps": o1["steps"],
                "e2e": o1["e2e"], "clocks": o1["clocks"], "gpu_launches": o1["launches"],
                "target_rays_per_s": 260e6,
                "roofline": {"bound": "hbm", "kernel": "k_walk_det", "unit": "GB/s",
                             "achieved": o1_bytes / (o1_walk * 1e-3) / 1e9 if o1_walk else 0.0,
                             "peak": peak, "peak_kind": peak_kind,
                             "frac": (o1_bytes / (o1_walk * 1e-3) / 1e9) / peak if o1_walk else None,
                             "bytes_per_launch": o1_bytes, "avg_launch_ms": o1_walk},
                "stages_ms_per_step": {k: round(o1s[k], 4) for k in (
                    "discover_ms", "walk_ms", "resolve_ms", "sort_ms", "fold_ms", "gpu_ms")}}
            line["ndt_om"] = {
                "workload": n["desc"]["workload"], "config": n["desc"], "value": n["value"],
                "unit": UNIT, "ms_per_step": n["ms"] / n["steps"], "steps": n["steps"],
                "e2e": n["e2e"], "clocks": n["clocks"], "gpu_launches": n["launches"],
                "roofline": {"bound": "hbm", "kernel": "k_walk_ndt_det", "unit": "GB/s",
                             "achieved": wb / nb / (nwalk * 1e-3) / 1e9 if nwalk else 0.0,
                             "peak": peak, "peak_kind": peak_kind,
                             "frac": (wb / nb / (nwalk * 1e-3) / 1e9) / peak if nwalk else None,
                             "bytes_per_launch": wb / nb, "avg_launch_ms": nwalk,
                             "traffic": load_traffic("c3", "det"),
                             "step_bytes": wb + fb,
                             "step_frac": (wb + fb) / (ns["gpu_ms"] * 1e-3) / 1e9 / peak},
                "stats": {"segments": ns["S"], "visits": ns["V"], "hits": n["H"],
                          "gaussian_visits_V3": V3, "sample_voxels_U": n["U"],
                          "records": ns["records"], "region_misses": ns["rmiss"]},
                "stages_ms_per_step": {k: round(ns[k], 4) for k in (
                    "discover_ms", "walk_ms", "resolve_ms", "sort_ms", "fold_ms", "gpu_ms")},
                "cpu_baseline": None,
            }
            line["c1"] = {"workload": c1["desc"]["workload"], "value": c1["value"], "unit": UNIT,
                          "ms_per_step": c1["ms"] / c1["steps"], "steps": c1["steps"],
                          "e2e": c1["e2e"], "clocks": c1["clocks"],
                          "gpu_ms_per_scan": c1["s0"]["gpu_ms"]}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, r["data"], args.cpu_budget, mode)
        if default_run and not args.no_extra:
            sweep = cpu_sweep(r["data"], line.get("ndt_om"))
            line["cpu_sweep"] = sweep
            if "ndt_om" in line and sweep.get("ndt_om_e2e"):
                best_w, best = max(sweep["ndt_om_e2e"].items(), key=lambda kv: kv[1])
                line["ndt_om"]["cpu_baseline"] = {
                    "value": best, "unit": UNIT, "cores": int(best_w), "kind": "reference",
                    "sample": sweep["ndt_om_sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_sweep(c2_batches, ndt_block):
    """The reference on the host cores, W in {1, 2, 4, ..., cores}:
    kernel-only occupancy (the reference's compiled _kernels.integrate_occupancy,
    best of 3 on one C2 batch) and end-to-end submit_batch (the reference
    package's own engine, Python preprocessing and -- for NDT-OM -- Python
    phase 2 included) for occupancy and NDT-OM."""
    from oracle import oracle as orc
    from oracle import ref_engine, ref_runner
    from paper_2206_06079_b200 import MapConfig, scans
    cores = orc.host_cores()
    ws = sorted({w for w in (1, 2, 4, 8, 16, 32, 64) if w <= cores} | {cores})
    out = {"cores": cores, "workers": ws}
    cfg2 = MapConfig(voxel_size=0.05)
    kern = {}
    for w in ws:
        best = 0.0
        for _ in range(3):
            t = ref_runner.time_reference(cfg2, c2_batches[:1], w, budget_s=0.0)
            best = max(best, t["rays"] / t["seconds"] if t["seconds"] else 0.0)
        kern[str(w)] = best
    out["occupancy_kernel"] = kern
    out["occupancy_kernel_sample"] = ("one C2 batch (262,400 rays, 0.05 m), reference "
                                      "_kernels.integrate_occupancy, best of 3")
    if ref_engine.load_voxmap() is None:
        out["e2e_unavailable"] = "reference package not installed in baseline/_ref"
        return out
    occ = {}
    sub = c2_batches[0][::8].copy()
    for w in sorted({1, min(4, cores), cores}):
        occ[str(w)] = ref_engine.time_submit_batch({"voxel_size": 0.05}, "occupancy", [],
                                                   sub, w)
    out["occupancy_e2e"] = occ
    out["occupancy_e2e_sample"] = ("every 8th ray of the first C2 batch (32,800 rays), "
                                   "reference voxmap.submit_batch, BatchStats.rays_per_second")
    if ndt_block is not None:
        tun = scans.os64_tunnel_scans(3)
        warm = [t[::4].copy() for t in tun[:2]]
        timed = tun[2][::4].copy()
        nd = {}
        for w in sorted({1, min(4, cores), cores}):
            nd[str(w)] = ref_engine.time_submit_batch({"voxel_size": 0.1}, "ndt-om", warm,
                                                      timed, w)
        out["ndt_om_e2e"] = nd
        out["ndt_om_sample"] = ("every 4th ray of C3 tunnel scan 3 (32,768 rays) after scans "
                                "1-2 built the Gaussians; reference voxmap.submit_batch "
                                "(native phase 1 on W threads + Python phase 2)")
    return out


STREET_PITCH = 250.0  # m between the per-GPU copies of the scene (weak scaling)


def run_sharded(args, world, rank, dev, dist):
    """N > 1: ONE region-sharded map over all ranks.  Weak
    scaling: the sequence is N copies of the workload's scene, each in its
    own street STREET_PITCH m apart, merged batch by batch, so every GPU
    walks the same number of rays as the 1-GPU run while every rank owns
    1/N of all regions (hash of 2x2x2 region blocks) and receives the miss
    counts / ordered records of its regions over NCCL all-to-all."""
    import torch

    from paper_2206_06079_b200.sharded import ShardedVoxelMap, submit_batch_sharded

    cfg, mode, data, desc = workload(args.workload, args.batches)
    supers = []
    for b in data:
        parts = []
        for r in range(world):
            c = b.copy()
            c["origin"][:, 0] += np.float32(r * STREET_PITCH)
            c["end"][:, 0] += np.float32(r * STREET_PITCH)
            parts.append(c)
        supers.append(np.concatenate(parts))
    sizes = [len(x) for x in supers]
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    total_rays = int(offsets[-1])
    host = np.concatenate(supers)
    d_all = torch.from_numpy(host.view(np.uint8).copy()).to(f"cuda:{dev}")
    d_batches = [d_all[offsets[i] * 40:offsets[i + 1] * 40] for i in range(len(supers))]
    smap = ShardedVoxelMap(cfg, rank, world, device=dev, initial_regions=4096, mode=mode)
    stream = torch.cuda.current_stream()

    def step(record=False, batches=d_batches):
        smap.vmap.clear()
        tot = dict(S=0, V=0, walk_ms=0.0, batches=0, records=0, rmiss=0, xbytes=0)
        for bt in batches:
            st = submit_batch_sharded(smap, bt)
            if record:
                tot["xbytes"] += st.exchange_bytes
                tot["S"] += st.segments
                tot["V"] += st.voxel_visits
                tot["walk_ms"] += st.walk_time * 1e3
                tot["records"] += st.records
                tot["rmiss"] += st.region_misses
                tot["batches"] += 1
        return tot

    for _ in range(args.warmup):
        step()
    clk_file = tempfile.mktemp(suffix=".csv")
    clk = sample_clocks(clk_file) if rank == 0 else None
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps = [step(record=True) for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    if clk:
        clk.terminate()
        clk.wait()
    t = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = total_rays * args.steps / (ms * 1e-3)
    # e2e: host records through the public sharded API (whole batch H2D per rank)
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(host.view(np.uint8).copy()).pin_memory()
        hv = pinned.numpy().view(host.dtype)
        dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        f0.record(stream)
        smap.vmap.clear()
        for i in range(len(supers)):
            submit_batch_sharded(smap, hv[offsets[i]:offsets[i + 1]])
        f1.record(stream)
        torch.cuda.synchronize()
        ems = max(f0.elapsed_time(f1), (time.perf_counter() - t0) * 1e3)
        t = torch.tensor([ems], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        e2e = {"value": total_rays / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(host.nbytes), "d2h_bytes_per_step": 0, "steps": 1,
               "api": "submit_batch_sharded(smap, pinned OHMB1 records)"}
    if rank == 0:
        s0 = steps[-1]
        o = host["origin"].astype(np.float64)
        e = host["end"].astype(np.float64)
        L = np.sqrt(((e - o) ** 2).sum(1))
        H = int(np.sum(((host["flags"] & 1) == 1) & (L <= cfg.max_ray_range) & (L > 0)))
        if mode == "occupancy":
            bytes_gpu = algorithmic_bytes(s0["S"], s0["V"], H) / world / max(1, s0["batches"])
        else:
            bytes_gpu = ndt_bytes(s0["S"], s0["V"], H, max(0, s0["records"] - H), 0)[0] / world / \
                max(1, s0["batches"])
        walk_ms = s0["walk_ms"] / max(1, s0["batches"])
        peak, peak_kind = load_peaks()
        achieved = bytes_gpu / (walk_ms * 1e-3) / 1e9 if walk_ms > 0 else 0.0
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (DDA) / f32 (log-odds)",
            "data": "synthetic",
            "config": dict(desc, exec="deterministic", rays_per_step=total_rays,
                           copies=world, street_pitch_m=STREET_PITCH,
                           parallelism=f"region-sharded x{world} (NCCL all-to-all of counts/records)",
                           mode=mode),
            "voxel_updates_per_s": s0["V"] * args.steps / (ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_walk_det" if mode == "occupancy" else "k_walk_ndt (sharded)",
                         "peak_kind": peak_kind, "bytes_per_launch": bytes_gpu,
                         "avg_launch_ms": walk_ms},
            "e2e": e2e, "cpu_baseline": None,
            "gpu_launches": None,
            "clocks": parse_clocks(clk_file, dev),
            "stats": {"segments": s0["S"], "visits": s0["V"], "records": s0["records"],
                      "region_misses": s0["rmiss"],
                      "exchange_bytes_per_batch": s0["xbytes"] / max(1, s0["batches"])},
        }
        print(json.dumps(line), flush=True)


def ctypes_stats_bytes():
    import ctypes

    from paper_2206_06079_b200._native import VmStats
    return ctypes.sizeof(VmStats)


if __name__ == "__main__":
    main()
