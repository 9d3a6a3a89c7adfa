#!/usr/bin/env python
"""Benchmark: env-camera frames/s of batched 3DGS rendering at 640x480 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[2] = SURVEY C3 — 1024 envs x 1 camera, 640x480, a shared
500k-Gaussian room background + a 10-body robot with 20k attached Gaussians, SH degree 3.
A step = one gsb_render of the whole batch (every hot-path row: K0 RLGK setup, K1 projection,
K2 binning, K4a sort, K4b compositing) on a fresh pose set.  Multi-GPU: one
process per GPU, each rank renders its own contiguous env slice (weak scaling: 1024 envs per
rank; --scaling strong: cfg.n_envs split), no collective on the render path; timing = max over
ranks of CUDA-event device time; after the timed region rank 0 re-renders the first envs of
every rank's slice by itself and compares per-env frame hashes (bit-identity to G = 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsb|reference] [--config C3]

--gpus N > 1 without a torchrun environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

FP32_OPS_PER_PAIR = 18      # SURVEY §8(d) d.4 / DESIGN.md §6: compositing ops per evaluated pair
# ... of which 14 are fp32 arithmetic (FMA pipe: dx, dy, quadratic form 5, +log2 o, tT, w, 4
# accumulations), 4 compare/min (ALU pipe) and 1 ex2 (XU).  On sm_100a the FMA pipe runs 128
# lanes/SM/clock for FFMA and packed FFMA2 alike while FFMA2 needs half the issue slots, so the
# pair rate is bounded by the FMA pipe (14 / 128), not by issue (K4b roofline);
# measured pipe rates: scripts/micro/ffma2_rate.cu (profiles/r3_pipe_rates.jsonl)
FMA_OPS_PER_PAIR = 14
SM_COUNT = 148
LANES_PER_SM = 128          # FMA-pipe lanes per SM
HASH_PROBE_ENVS = 4         # envs per rank whose frames are re-rendered by rank 0 alone
# the paper's own number (context, not a target): "up to 2048 scenes at 640x480 with a total
# throughput of up to 10,000 FPS", "~10k" 3DGS render FPS at 640x480 on an RTX 4090 +
# i9-14900K (Table I, note P:150); scene size unstated
PAPER_CONTEXT = {"value": 1.0e4, "unit": "frames/s", "gpu": "NVIDIA RTX 4090", "resolution": "640x480",
                 "cite": "PAPER.md P:139 (Table I), P:150, P:286", "note": "scene size unstated; context only"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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


# ------------------------------------------------------------------------------ launcher
def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_self_launch(args) -> None:
    """--gpus N > 1 outside a torchrun environment: re-run this script as N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1 and exit with its status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    sys.stdout.flush()
    sys.exit(subprocess.call(cmd, env=env))


def dist_setup(args, need_cuda=True):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus not in (1, world):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    import torch
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("GSB_DIST_BACKEND",
                                 "nccl" if (need_cuda and torch.cuda.is_available()) else "gloo")
        if need_cuda and torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend=backend)
    elif need_cuda and torch.cuda.is_available():
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


def gather_objects(obj, world: int):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def rank_envs(cfg, scaling: str, rank: int, world: int) -> np.ndarray:
    """Global env ids of a rank: weak = its own cfg.n_envs envs; strong = a contiguous slice."""
    if scaling == "weak":
        return np.arange(rank * cfg.n_envs, (rank + 1) * cfg.n_envs)
    lo, hi = synth.env_slice(cfg.n_envs, rank, world)
    return np.arange(lo, hi)


def frame_hash(*planes) -> str:
    """Order-sensitive hash of one env's output planes (bit patterns, torch tensors)."""
    import hashlib
    h = hashlib.sha1()
    for p in planes:
        h.update(p.contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


# ------------------------------------------------------------------------------ CPU oracle
def oracle_sample(cfg, scene, env: int, step: int, seed: int, threads: int):
    """The SURVEY §8(d) d.6 protocol, one frame (env, camera 0, pose step): the oracle's full
    projection + depth order over all N Gaussians, then compositing of the d.6 pixel sample (4096
    stratified pixels + 2 full 16x16 tiles, synth.sample_pixels); frames/s extrapolated as
    1 / (t_proj + t_px * Npx).  Returns the timing and the oracle's values on the sample."""
    import oracle
    b = synth.make_batch(cfg, [env], step=step)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    px, py, n_strat = synth.sample_pixels(cfg.width, cfg.height, seed)
    t0 = time.perf_counter()
    proj, zb, valid = oracle.project(scene, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm)
    order = oracle.depth_order(zb, valid)
    t1 = time.perf_counter()
    rgb, dep, alp, term, nev, masked, _, _, tnear, eT = oracle.composite(proj, order, px, py, prm, "box",
                                                                        nthreads=threads)
    t2 = time.perf_counter()
    t_px = (t2 - t1) / px.size
    t_frame = (t1 - t0) + t_px * cfg.width * cfg.height
    return {"value": 1.0 / t_frame, "t_proj_s": t1 - t0, "t_pixels_s": t2 - t1, "n_pixels": int(px.size),
            "n_strat": n_strat, "seconds": t2 - t0, "px": px, "py": py, "rgb": rgb, "depth": dep, "alpha": alp,
            "masked": masked, "term_near": tnear, "terminated": term >= 0}


def oracle_c1_full_frame(threads: int) -> float:
    """C1 (64x48, 1k Gaussians) full frame end to end through the oracle, seconds (d.6)."""
    import oracle
    cfg = synth.CONFIGS["C1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    t0 = time.perf_counter()
    oracle.render_frame(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], oracle.RenderParams(cfg.width, cfg.height),
                        nthreads=threads)
    return time.perf_counter() - t0


def baseline_record(samples, threads, cfg, c1_s):
    s0 = samples[0]
    return {"value": float(np.median([s["value"] for s in samples])), "unit": "env-camera frames/s",
            "cores": threads, "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{len(samples)} frame(s) of {cfg.name} by the d.6 protocol: projection + depth order over all "
                      f"{cfg.n_gaussians} Gaussians ({s0['t_proj_s']:.2f} s) + {s0['n_strat']} stratified pixels + 2 "
                      f"full tiles = {s0['n_pixels']} pixels ({s0['t_pixels_s']:.2f} s), extrapolated to "
                      f"{cfg.width}x{cfg.height} (frames/s = 1 / (t_proj + t_px * W * H))",
            "extrapolated": True, "c1_full_frame_s": c1_s,
            "masked_frac": float(np.mean(np.concatenate([s["masked"] for s in samples]))),
            "term_near_frac": float(np.mean(np.concatenate([s["term_near"] for s in samples]))),
            "terminated_frac": float(np.mean(np.concatenate([s["terminated"] for s in samples])))}


def run_reference(args, cfg):
    """--impl reference: the oracle as it stands, by the d.6 protocol, on this arm's config."""
    world, rank, _ = dist_setup(args, need_cuda=False)
    if rank != 0:
        return
    scene = synth.make_scene(cfg)
    threads = os.cpu_count() or 1
    c1_s = oracle_c1_full_frame(threads)
    envs = rank_envs(cfg, args.scaling, 0, world)
    samples = []
    t_start = time.perf_counter()
    for s in range(args.warmup + args.steps):
        r = oracle_sample(cfg, scene, int(envs[s % len(envs)]), s % 23, seed=s, threads=threads)
        if s >= args.warmup:
            samples.append(r)
    wall = time.perf_counter() - t_start
    base = baseline_record(samples, threads, cfg, c1_s)
    v = base["value"]
    out = {"metric": "env-camera frames/s at 640x480", "value": v, "unit": "env-camera frames/s",
           "impl": "reference", "n_gpus": world if world > 1 else args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 / v * len(envs) * cfg.n_cams,
           "ms_per_step_kind": "extrapolated: one step = the whole batch at the sampled per-frame rate",
           "sample_seconds_per_step": float(np.mean([s["seconds"] for s in samples])), "wall_s": wall,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_dict(cfg, len(envs), max(world, args.gpus), args),
           "cpu_baseline": base, "paper_context": PAPER_CONTEXT,
           "e2e": {"value": v, "unit": "env-camera frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def config_dict(cfg, B, world, args):
    """The workload named in both arms' JSON lines."""
    C, W, H = cfg.n_cams, cfg.width, cfg.height
    total = B * world if args.scaling == "weak" else cfg.n_envs
    return {"workload": f"{cfg.name}: {B} envs x {C} cam per GPU, {W}x{H}, "
                        f"{cfg.n_bg} static + {cfg.n_rb} robot Gaussians on {cfg.n_bodies} bodies, SH {cfg.sh_degree}",
            "envs_per_gpu": B, "frames_per_step": total * C,
            "l2": "256 MB buffer written between timed steps (outside the events); "
                  "per-step working set (5 GB outputs) >> L2", "parallelism": f"env-slices x{world}"}


# ------------------------------------------------------------------------------ launcher self-test
def run_launcher_selftest(args, cfg):
    """Host logic of the multi-GPU bench without a GPU (CPU, gloo): sharding, max over ranks,
    object gather and the per-env hash comparison, on per-env hashes of the synthetic INPUTS
    (poses of the last pose step and cameras).  Prints one JSON line on rank 0."""
    world, rank, _ = dist_setup(args, need_cuda=False)
    import torch
    envs = rank_envs(cfg, args.scaling, rank, world)
    step = (args.warmup + args.steps - 1) % 23
    poses = synth.make_poses(cfg, envs, step)
    K, W2C = synth.make_cameras(cfg, envs)
    hashes = {int(e): frame_hash(torch.from_numpy(poses[k]), torch.from_numpy(K[k]), torch.from_numpy(W2C[k]))
              for k, e in enumerate(envs[:HASH_PROBE_ENVS])}
    t = max_over_ranks(0.001 * (rank + 1), world)
    allh = gather_objects(hashes, world)
    slices = gather_objects([int(envs[0]), int(envs[-1])], world)
    if rank == 0:
        probe = np.array(sorted(e for h in allh for e in h))
        p2, K2, W2 = synth.make_poses(cfg, probe, step), *synth.make_cameras(cfg, probe)
        mism = sum(frame_hash(torch.from_numpy(p2[k]), torch.from_numpy(K2[k]), torch.from_numpy(W2[k]))
                   != next(h[int(e)] for h in allh if int(e) in h) for k, e in enumerate(probe))
        print(json.dumps({"selftest": True, "n_gpus": world, "max_over_ranks": t,
                          "slices": slices,
                          "config": config_dict(cfg, len(envs), world, args),
                          "env_hash_check": {"envs_checked": int(probe.size), "mismatches": int(mism)}}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gsb", choices=["gsb", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hash-check", action="store_true")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--launcher-selftest", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: cfg.n_envs envs per rank (C3, the headline); strong: cfg.n_envs envs in total, "
                         "contiguous slices per rank (SURVEY §8(e): C5 8192 envs over G GPUs)")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    maybe_self_launch(args)
    if args.launcher_selftest:
        return run_launcher_selftest(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import paper_2604_25459_b200 as gsb

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", torch.cuda.current_device())
    peaks, peaks_kind = load_peaks()

    C, W, H = cfg.n_cams, cfg.width, cfg.height
    env_ids = rank_envs(cfg, args.scaling, rank, world)
    B = len(env_ids)
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

    # counters V, K, P and terminated pixels in a separate untimed render (STATS)
    g.render(poses[0], intr, w2c, gsb.RenderParams(W, H, stats=True), rgb, dep)
    st = g.stats_ext()

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
    comp_ms, comp_launches, launches, kern = [], [], [], []
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
    last_step = (args.warmup + args.steps - 1) % n_pose_sets

    # SURVEY §8(e) correctness: per-env frames of every rank == the same envs rendered by rank 0
    # alone (a separate single-GPU call), compared by per-env hashes of the output bits
    hash_check = None
    if not args.no_hash_check:
        k = min(HASH_PROBE_ENVS, B)
        mine = {int(env_ids[j]): frame_hash(rgb[j], dep[j]) for j in range(k)}
        allh = gather_objects(mine, world)
        if rank == 0:
            probe = np.array(sorted(e for h in allh for e in h))
            P = len(probe)
            Kp, Wp = synth.make_cameras(cfg, probe)
            pr = torch.from_numpy(synth.make_poses(cfg, probe, last_step)).to(dev)
            r2 = torch.empty((P, C, 3, H, W), device=dev)
            d2 = torch.empty((P, C, H, W), device=dev)
            g.render(pr, torch.from_numpy(Kp).to(dev), torch.from_numpy(Wp).to(dev), gsb.RenderParams(W, H), r2, d2)
            torch.cuda.synchronize(dev)
            mism = sum(frame_hash(r2[j], d2[j]) != next(h[int(e)] for h in allh if int(e) in h)
                       for j, e in enumerate(probe))
            hash_check = {"envs_checked": int(P), "ranks": world, "mismatches": int(mism),
                          "method": "sha1 of each env's rgb+depth bits vs rank 0 rendering those envs alone"}
        barrier(world)

    # roofline of the dominant kernel (K4b persistent compositing; the fused K4 when
    # GSB_K4=fused): algorithmic fp32 ops / its event time
    k4_avg_ms = sum(comp_ms) / max(sum(comp_launches), 1)
    pairs_per_launch = st["P"] / max(comp_launches[0], 1)
    achieved = FP32_OPS_PER_PAIR * pairs_per_launch / (k4_avg_ms / 1e3) / 1e12
    fma_rate = SM_COUNT * LANES_PER_SM * peaks.get("sm_max_mhz", 1965.0) * 1e6   # fp32 FMA-pipe ops/s
    # the 18-op pair's peak rate: one pair per 14 FMA-pipe lane-cycles (the binding pipe)
    peak = FP32_OPS_PER_PAIR * fma_rate / FMA_OPS_PER_PAIR / 1e12
    # whole-path roofline: T_roof = max(B_alg / BW, Ops_alg / R_fp32) per
    # step, from the oracle's work counts (V, K, P of the STATS render), not from our SASS
    F_step = B * C
    n_g = cfg.n_gaussians
    chunk_e = 64
    b_alg = F_step * ((240 if cfg.sh_degree == 3 else 60) * n_g / chunk_e + 8 * n_g) \
        + 108 * st["V"] + 32 * st["K"] + 16 * W * H * F_step
    ops_alg = FMA_OPS_PER_PAIR * st["P"] + 15 * n_g * F_step + (190 if cfg.sh_degree == 3 else 105) * st["V"]
    bw = peaks.get("hbm_gbs", 6546.6) * 1e9
    t_hbm, t_alu = b_alg / bw, ops_alg / fma_rate
    t_roof = max(t_hbm, t_alu)
    path_roof = {"t_roof_ms_per_step": t_roof * 1e3, "bound": "alu" if t_alu >= t_hbm else "hbm",
                 "t_alu_ms": t_alu * 1e3, "t_hbm_ms": t_hbm * 1e3,
                 "frac": t_roof / (t_max / args.steps),
                 "basis": "B_alg = (240|60)N/64 + 8N + 108V + 32K + 16Npx bytes and Ops_alg = 14P + 15N + "
                          "(190|105)V FMA-pipe fp32 ops per frame (SURVEY §8(d) d.4; 14 of the 18 ops per pair "
                          "are FMA-pipe arithmetic, the 4 compares run on the ALU pipe); BW = MEASURED_PEAKS "
                          "hbm_gbs; R = 148 SM x 128 FMA lanes x f"}
    # measured DRAM bytes of the dominant kernel per launch: the ncu --set full capture's bytes per
    # frame (profiles/k4_ncu_summary.json, captured on its own config) x this run's frames per launch
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k4_ncu_summary.json")) as f:
            ks = json.load(f)
        if ks.get("config") == args.config and ks.get("dram_bytes_per_frame"):
            traffic = ks["dram_bytes_per_frame"] * (B * C) / max(comp_launches[0], 1)
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
        e2e = {"value": (B * world if args.scaling == "weak" else cfg.n_envs) * C * args.e2e_steps / t_e2e,
               "unit": "env-camera frames/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": args.e2e_steps}

    # the oracle on the host cores (d.6 protocol) on env 0 of the last timed step, which also
    # gives a live parity check of that frame's sample against the GPU output
    cpu, live = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = os.cpu_count() or 1
        # three samples (median, as the reference arm's steps): env 0 of the last timed step (also
        # the live parity frame), then two more envs / pose steps
        smp = oracle_sample(cfg, scene, int(env_ids[0]), last_step, seed=0, threads=threads)
        more = [oracle_sample(cfg, scene, int(env_ids[(k * B) // 3]), (last_step + k) % n_pose_sets, seed=k,
                              threads=threads) for k in (1, 2)]
        cpu = baseline_record([smp] + more, threads, cfg, oracle_c1_full_frame(threads))
        px, py = smp["px"], smp["py"]
        g_rgb = rgb[0, 0].permute(1, 2, 0).cpu().numpy()[py, px]
        g_dep = dep[0, 0].cpu().numpy()[py, px]
        ok = ~smp["masked"]
        d_rgb = np.abs(g_rgb - smp["rgb"]).max(-1)
        d_dep = np.abs(g_dep - smp["depth"]) - (oracle.TOL_DEPTH_REL * smp["depth"] + oracle.TOL_DEPTH_ABS)
        live = {"frame": f"env {int(env_ids[0])}, camera 0, pose step {last_step}", "pixels": int(px.size),
                "masked_frac": float(np.mean(~ok)), "max_abs_rgb": float(d_rgb[ok].max()),
                "rgb_fails": int((d_rgb[ok] > oracle.TOL_RGB).sum()), "depth_fails": int((d_dep[ok] > 0).sum()),
                "tolerances": {"rgb": oracle.TOL_RGB, "depth_rel": oracle.TOL_DEPTH_REL}}

    ranks = gather_objects({"rank": rank, "device": torch.cuda.get_device_name(dev),
                            "pci": torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(
                                torch.cuda.get_device_properties(dev), "pci_bus_id") else None,
                            "envs": [int(env_ids[0]), int(env_ids[-1])] if B else [], "device_s": t_dev}, world)
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
                         "peak_basis": f"18 ops per pair x (148 SM x 128 FMA-pipe lanes x "
                                       f"{peaks.get('sm_max_mhz', 1965.0)} MHz) / 14 FMA-pipe ops per pair: the FMA "
                                       f"pipe binds (FFMA2 halves issue, not FMA-pipe time; ALU 4/64 and XU 1/16 "
                                       f"lane-cycles per pair are below 14/128); unit counts B200_PROFILING.md and "
                                       f"scripts/micro/ffma2_rate.cu, clock from MEASURED_PEAKS.json ({peaks_kind})"},
            "path_roofline": path_roof,
            "stage_ms_per_step": tsum,
            "counters": {"V_per_frame": st["V"] / (B * C), "K_per_frame": st["K"] / (B * C),
                         "P_per_frame": st["P"] / (B * C),
                         # scene statistics reported with every FPS number
                         "V_over_N": st["V"] / (B * C) / cfg.n_gaussians, "K_over_V": st["K"] / max(st["V"], 1),
                         "mean_tile_list": st["K"] / (B * C) / (((W + 15) // 16) * ((H + 15) // 16)),
                         "mean_n_eval_per_pixel": st["P"] / (B * C) / (W * H),
                         "terminated_pixel_frac": st["terminated"] / max(st["pixels"], 1),
                         "long_lists_per_step": kern[-1]["long_lists"],
                         "max_tile_list": kern[-1]["max_list"], "chunks_per_step": kern[-1]["chunks"]},
            "clocks": clocks,
            "e2e": e2e,
            "env_hash_check": hash_check,
            "ranks": ranks,
            "cpu_baseline": cpu,
            "live_parity": live,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
