#!/usr/bin/env python
"""Benchmark: env-camera frames/s of batched 3DGS rendering at 640x480 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[2] = SURVEY C3 — 1024 envs x 1 camera, 640x480, a shared
500k-Gaussian room background + a 10-body robot with 20k attached Gaussians, SH degree 3.
A step = one gsb_render of the whole batch (every hot-path row: K0 RLGK setup, K1 projection,
K2 binning, K3 sort, K4 compositing) on a fresh pose set.  Multi-GPU: one process per GPU,
each rank renders its own contiguous slice of 1024 envs (weak scaling, no collective on the
render path); timing = max over ranks of CUDA-event device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsb|reference] [--config C3]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

FP32_OPS_PER_PAIR = 18      # SURVEY §8(d) d.4 / DESIGN.md §6: compositing ops per evaluated pair
SM_COUNT = 148
LANES_PER_SM = 128


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("GSB_DIST_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    on_gpu = torch.cuda.is_available() and dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------ CPU oracle
def cpu_baseline(cfg, scene, n_pix=4096, seed=0):
    """The oracle (as it stands) on a bounded sample of one frame: full projection + depth
    order over all N Gaussians, then 4096 stratified pixels; extrapolated to whole frames."""
    import oracle
    b = synth.make_batch(cfg, [0])
    prm = oracle.RenderParams(cfg.width, cfg.height)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    proj, zb, valid = oracle.project(scene, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm)
    order = oracle.depth_order(zb, valid)
    t1 = time.perf_counter()
    rng = np.random.default_rng(seed)
    # stratified: one random pixel in each cell of a 64 x 64 grid
    gx, gy = np.meshgrid(np.arange(64), np.arange(64))
    px = np.minimum((gx.reshape(-1) * cfg.width) // 64 + rng.integers(0, cfg.width // 64, gx.size), cfg.width - 1)
    py = np.minimum((gy.reshape(-1) * cfg.height) // 64 + rng.integers(0, max(cfg.height // 64, 1), gy.size),
                    cfg.height - 1)
    px, py = px[:n_pix], py[:n_pix]
    oracle.composite(proj, order, px, py, prm, "box", nthreads=cores)
    t2 = time.perf_counter()
    t_px = (t2 - t1) / px.size
    t_frame = (t1 - t0) + t_px * cfg.width * cfg.height
    return {"value": 1.0 / t_frame, "unit": "env-camera frames/s", "cores": cores, "kind": "oracle",
            "sample": f"1 frame of {cfg.name}: projection+depth order over all {scene.n} Gaussians "
                      f"({t1 - t0:.2f} s) + {px.size} stratified pixels ({t2 - t1:.2f} s), "
                      f"extrapolated to {cfg.width}x{cfg.height}",
            "seconds": t2 - t0}


def run_reference(args, cfg):
    """--impl reference: the oracle as it stands, on this arm's config/metric/unit."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    scene = synth.make_scene(cfg)
    vals = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline(cfg, scene, n_pix=1024, seed=s)
        if s >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    out = {"metric": "env-camera frames/s at 640x480", "value": v, "unit": "env-camera frames/s",
           "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": config_dict(cfg, cfg.n_envs if args.scaling == "weak" else synth.env_slice(cfg.n_envs, 0, world)[1],
                                 world, args),
           "cpu_baseline": {"value": v, "unit": "env-camera frames/s", "cores": vals[0]["cores"], "kind": "oracle",
                            "sample": vals[0]["sample"].replace("4096", "1024")},
           "e2e": {"value": v, "unit": "env-camera frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def config_dict(cfg, B, world, args):
    """The workload named in both arms' JSON lines."""
    C, W, H = cfg.n_cams, cfg.width, cfg.height
    total = B * world if args.scaling == "weak" else cfg.n_envs
    return {"workload": f"{cfg.name}: {B} envs x {C} cam per GPU, {W}x{H}, "
                        f"{cfg.n_bg} static + {cfg.n_rb} robot Gaussians on {cfg.n_bodies} bodies, SH {cfg.sh_degree}",
            "envs_per_gpu": B, "frames_per_step": total * C,
            "l2": "256 MB buffer written between timed steps (outside the events); "
                  "per-step working set (5 GB outputs) >> L2", "parallelism": f"env-slices x{world}"}


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gsb", choices=["gsb", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: cfg.n_envs envs per rank (C3, the headline); strong: cfg.n_envs envs in total, "
                         "contiguous slices per rank (SURVEY §8(e): C5 8192 envs over G GPUs)")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import paper_2604_25459_b200 as gsb

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", local % torch.cuda.device_count() if world > 1 else 0)
    peaks, peaks_kind = load_peaks()

    # weak scaling: every rank renders its own cfg.n_envs envs (global ids rank*B + [0, B));
    # strong scaling: the cfg.n_envs envs are split into contiguous slices (synth.env_slice)
    C, W, H = cfg.n_cams, cfg.width, cfg.height
    if args.scaling == "weak":
        B = cfg.n_envs
        env_ids = np.arange(rank * B, (rank + 1) * B)
    else:
        lo, hi = synth.env_slice(cfg.n_envs, rank, world)
        env_ids = np.arange(lo, hi)
        B = hi - lo
    scene = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(scene, device=dev.index)
    g.reserve(B, C, W, H, chunk_frames=args.chunk, host_io=not args.no_e2e)
    n_pose_sets = min(23, args.steps + args.warmup)
    K_cam, W2C = synth.make_cameras(cfg, env_ids)
    poses = [torch.from_numpy(synth.make_poses(cfg, env_ids, s)).to(dev) for s in range(n_pose_sets)]
    intr = torch.from_numpy(K_cam).to(dev)
    w2c = torch.from_numpy(W2C).to(dev)
    rgb = torch.empty((B, C, 3, H, W), device=dev)
    dep = torch.empty((B, C, H, W), device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)   # 256 MB > L2 (126 MB)
    stream = torch.cuda.current_stream(dev)

    # counters V, K, P in a separate untimed render (STATS)
    g.render(poses[0], intr, w2c, gsb.RenderParams(W, H, stats=True), rgb, dep)
    st = g.stats()

    prm = gsb.RenderParams(W, H, timing=True)
    for s in range(args.warmup):
        g.render(poses[s % n_pose_sets], intr, w2c, prm, rgb, dep)
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(dev.index)
    sampler.start()
    barrier(world)
    torch.cuda.synchronize(dev)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    step_ms, comp_ms, comp_launches, launches, kern = [], [], [], [], []
    for s in range(args.steps):
        flush.fill_(float(s))                       # L2 flush between timed steps (outside the events)
        ev0[s].record(stream)
        g.render(poses[(args.warmup + s) % n_pose_sets], intr, w2c, prm, rgb, dep)
        ev1[s].record(stream)
        tm = g.timings()                            # synchronises with this render
        comp_ms.append(tm["composite_ms"])
        comp_launches.append(tm["composite_launches"])
        launches.append(tm["launches"])
        kern.append(tm)
    torch.cuda.synchronize(dev)
    barrier(world)
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    t_dev = sum(step_ms) / 1e3
    t_max = max_over_ranks(t_dev, world)
    frames_total = (B * world if args.scaling == "weak" else cfg.n_envs) * C * args.steps
    value = frames_total / t_max

    # roofline of the dominant kernel (K4b persistent compositing; the fused K4 when
    # GSB_K4=fused): algorithmic fp32 ops / its event time
    k4_avg_ms = sum(comp_ms) / max(sum(comp_launches), 1)
    pairs_per_launch = st["P"] / max(comp_launches[0], 1)
    achieved = FP32_OPS_PER_PAIR * pairs_per_launch / (k4_avg_ms / 1e3) / 1e12
    peak = SM_COUNT * LANES_PER_SM * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    # whole-path roofline: T_roof = max(B_alg / BW, Ops_alg / R_fp32) per
    # step, from the oracle's work counts (V, K, P of the STATS render), not from our SASS
    F_step = B * C
    n_g = cfg.n_gaussians
    chunk_e = 64
    b_alg = F_step * ((240 if cfg.sh_degree == 3 else 60) * n_g / chunk_e + 8 * n_g) \
        + 108 * st["V"] + 32 * st["K"] + 16 * W * H * F_step
    ops_alg = FP32_OPS_PER_PAIR * st["P"] + 15 * n_g * F_step + (190 if cfg.sh_degree == 3 else 105) * st["V"]
    bw = peaks.get("hbm_gbs", 6546.6) * 1e9
    t_hbm, t_alu = b_alg / bw, ops_alg / (peak * 1e12)
    t_roof = max(t_hbm, t_alu)
    path_roof = {"t_roof_ms_per_step": t_roof * 1e3, "bound": "alu" if t_alu >= t_hbm else "hbm",
                 "t_alu_ms": t_alu * 1e3, "t_hbm_ms": t_hbm * 1e3,
                 "frac": t_roof / (t_max / args.steps) if args.scaling == "weak" or world == 1 else None,
                 "basis": "B_alg = (240|60)N/64 + 8N + 108V + 32K + 16Npx bytes and Ops_alg = 18P + 15N + "
                          "(190|105)V fp32 ops per frame (SURVEY §8(d) d.4); BW = MEASURED_PEAKS hbm_gbs"}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k4_ncu_summary.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass

    # e2e through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        h_poses = [p.cpu().pin_memory() for p in poses[: min(len(poses), args.e2e_steps + 1)]]
        h_intr, h_w2c = intr.cpu().pin_memory(), w2c.cpu().pin_memory()
        h_rgb = torch.empty((B, C, 3, H, W), pin_memory=True)
        h_dep = torch.empty((B, C, H, W), pin_memory=True)
        p0 = gsb.RenderParams(W, H)
        g.render_host(h_poses[0], h_intr, h_w2c, p0, h_rgb, h_dep)  # warm
        barrier(world)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.e2e_steps):
            g.render_host(h_poses[(s + 1) % len(h_poses)], h_intr, h_w2c, p0, h_rgb, h_dep)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3, world)
        h2d = h_poses[0].numel() * 4 + h_intr.numel() * 4 + h_w2c.numel() * 4
        d2h = h_rgb.numel() * 4 + h_dep.numel() * 4
        e2e = {"value": (B * world if args.scaling == "weak" else cfg.n_envs) * C * args.e2e_steps / t_e2e, "unit": "env-camera frames/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, scene)
        cpu.pop("seconds", None)

    if rank == 0:
        tsum = {k: float(np.mean([t[k] for t in kern])) for k in
                ("setup_ms", "project_ms", "scan_ms", "emit_ms", "sort_ms", "composite_ms")}
        out = {
            "metric": "env-camera frames/s at 640x480",
            "value": value,
            "unit": "env-camera frames/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": args.scaling,
            "step_ms": {"median": float(np.median(step_ms)), "min": float(np.min(step_ms)),
                        "max": float(np.max(step_ms))},
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, B, world, args),
            "gpu_launches": int(np.mean(launches)),
            "roofline": {"bound": "alu", "kernel": "K4b blend" if os.environ.get("GSB_K4") != "fused" else "K4 composite", "achieved": achieved, "peak": peak,
                         "unit": "Top/s (fp32 thread-ops)", "frac": achieved / peak, "traffic": traffic,
                         "ops_per_launch": FP32_OPS_PER_PAIR * pairs_per_launch,
                         "avg_launch_ms": k4_avg_ms,
                         "peak_basis": f"148 SM x 128 lanes x {peaks.get('sm_max_mhz', 1965.0)} MHz "
                                       f"(B200_PROFILING.md unit counts; clock from MEASURED_PEAKS.json, {peaks_kind})"},
            "path_roofline": path_roof,
            "stage_ms_per_step": tsum,
            "counters": {"V_per_frame": st["V"] / (B * C), "K_per_frame": st["K"] / (B * C),
                         "P_per_frame": st["P"] / (B * C),
                         # scene statistics reported with every FPS number
                         "V_over_N": st["V"] / (B * C) / cfg.n_gaussians, "K_over_V": st["K"] / max(st["V"], 1),
                         "mean_tile_list": st["K"] / (B * C) / (((W + 15) // 16) * ((H + 15) // 16)),
                         "mean_n_eval_per_pixel": st["P"] / (B * C) / (W * H), "long_lists_per_step": kern[-1]["long_lists"],
                         "max_tile_list": kern[-1]["max_list"], "chunks_per_step": kern[-1]["chunks"]},
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
