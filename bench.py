#!/usr/bin/env python
"""bench.py -- Image-GS train iteration on B200 (BASELINE.json configs[1]; configs[3] at N > 1).

One step = one training iteration of the reference's fit loop
(fit.cpp:149-157): 10k sampled pixel centres, exact global top-K (K=10) over
the whole set, normalised blend, L1 loss, analytic backward with the
sample-ordered gradient reduction, Adam + constrain.

* N = 1: C2, a 2048x2048 photo-like target with 100k Gaussians (the C2
  budget) in the fit-start state (sigma = 2 px, theta = 0), the worst case
  for candidate culling.
* N > 1: C4, an 8192x8192 photo-like target with 1M random-local Gaussians
  (BASELINE.json configs[3]: "training ... at 2/4/8 GPUs").  One process per
  GPU (launched under torch.distributed.run; `--gpus N` without WORLD_SIZE
  re-executes itself that way); the step's samples are split into
  contiguous rank blocks, an NCCL all-gather completes the per-sample
  contributions in sample order, every rank reduces, rank r updates its
  1/N slice of the set (sharded Adam) and an all-gather of the parameters
  follows -- strong scaling, bit-identical to one GPU.  Rank 0 also times
  the same C4 step on one GPU first (`scaling_baseline`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* value   device-resident iterations/s (sample indices pre-uploaded), device
          time from CUDA events on the library's stream, L2 flushed (512 MiB
          memset) before every timed step; max over ranks.
* e2e     the same iteration through the public C-ABI call
          igs_train_iteration_async/igs_train_wait with HOST buffers: every
          step copies its sample indices host->device and reads the loss
          (+ status) back; device marks per step, with the host wall clock of
          the whole loop beside it.
* --impl reference times the reference's own OpenMP implementation
          (oracle/_ref: the unmodified reference library, all host threads) on
          the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASE["metric"]
NS = 10_000
K = 10
LR = (2e-4, 2e-3, 1e-3, 1e-3)
FLUSH_BYTES = 512 << 20
C2 = {"name": "C2", "W": 2048, "H": 2048, "N": 100_000,
      "workload": ("C2 train iteration: 2048x2048 photo-like target, 100k Gaussians (fit-start state: sigma 2 px, "
                   "theta 0, uniform centres), 10k sampled pixels, exact global top-K K=10, L1 loss + backward "
                   "(sample-ordered reduction) + Adam/constrain")}
C4 = {"name": "C4", "W": 8192, "H": 8192, "N": 1_000_000,
      "workload": ("C4 train iteration: 8192x8192 photo-like target (2048^2 photo-like upsampled 4x), 1M "
                   "random-local Gaussians (sigma 2-16 px), 10k sampled pixels, exact global top-K K=10, L1 loss + "
                   "backward (sample-ordered reduction) + Adam/constrain")}


def workload_for(world: int) -> dict:
    return C2 if world == 1 else C4


def make_inputs(wl: dict):
    from paper_2407_01866_b200 import synth
    if wl["name"] == "C2":
        params = synth.init_set(wl["N"], wl["W"], wl["H"], seed=11)
        target = synth.photo_like_image(wl["W"], wl["H"], 31001)
    else:
        params = synth.random_local_set(wl["N"], wl["W"], wl["H"], seed=7)
        small = synth.photo_like_image(2048, 2048, 31004)
        target = np.ascontiguousarray(small.repeat(4, axis=0).repeat(4, axis=1))
    return params, target


def bench_config(wl: dict, world: int) -> dict:
    """The workload description both arms print (same keys and values)."""
    return {"workload": wl["workload"], "image": f"{wl['W']}x{wl['H']}", "gaussians": wl["N"],
            "samples_per_iter": NS, "k": K,
            "parallelism": "single GPU" if world == 1 else
            f"dp{world}: sample blocks per rank, NCCL all-gather of the per-sample contributions, "
            "sample-ordered reduction, sharded Adam + parameter all-gather"}


# FP64 pipe ops per evaluated (pixel, candidate) pair: 13 arithmetic ops of
# mahalanobis_sq (renderer.cpp:17-23) + the threshold compare.
OPS_PER_PAIR = 14


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C1/C3 secondary measurements")
    return ap.parse_args()


class Clocks:
    """SM clock + throttle-reason sampler (NVML, every 2 ms) for the timed
    region -- the B200_PROFILING.md clocks line; nvidia-smi's 200 ms loop is
    too coarse for a region of a few tens of ms."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass
                time.sleep(0.002)

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def stop(self):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def physical_gpu(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


# --------------------------------------------------------------------------- ours
def device_steps(ctx, args, t0: int, reps: int) -> list:
    """`reps` device-resident iterations t0.. each bracketed by CUDA events
    after an L2 flush; per-step ms."""
    step_ms = []
    for s in range(reps):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.timer_begin()
        ctx.train_iterations(1, K, LR, t0 + s, want_losses=False)
        step_ms.append(ctx.timer_end())
    return step_ms


def single_gpu_baseline(ctx_dev: int, args, wl: dict, params, target, samples) -> dict:
    """The same step on one GPU (a context without a communicator): the
    denominator of the N > 1 scaling efficiency, measured in this run."""
    from paper_2407_01866_b200 import Context
    with Context(ctx_dev) as c:
        c.set_params(params)
        c.set_target(target)
        c.upload_samples(samples)
        c.train_iterations(args.warmup, K, LR, 1, want_losses=False)
        ms = device_steps(c, args, args.warmup + 1, args.steps)
    return {"n_gpus": 1, "value": 1e3 * len(ms) / sum(ms), "unit": "iters/s", "ms_per_step": sum(ms) / len(ms),
            "note": f"{wl['name']} on rank 0's GPU alone (no communicator), same steps, before the {wl['name']} "
                    "multi-rank run"}


def run_ours(args, rank, world, local_rank, dist):
    from paper_2407_01866_b200 import Context, synth
    from paper_2407_01866_b200 import dist as D
    from paper_2407_01866_b200.igs import PROF_NAMES, PROF_SCAN

    wl = workload_for(world)
    W, H, N = wl["W"], wl["H"], wl["N"]
    params, target = make_inputs(wl)
    total_steps = args.warmup + args.steps
    samples = synth.sample_indices(NS, W, H, seed=99, steps=total_steps)
    mine = D.shard(samples, rank, world)  # this rank's contiguous block of every step

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    baseline = None
    if world > 1:
        if rank == 0:
            baseline = single_gpu_baseline(local_rank, args, wl, params, target, samples)
        barrier()
    ctx = Context(local_rank)
    ctx.set_params(params)
    ctx.set_target(target)
    if world > 1:
        uid = [Context.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(uid[0], world, rank)

    fp64_peak = ctx.fp64_peak()

    # ---- device-resident value ------------------------------------------------
    ctx.upload_samples(mine)
    ctx.train_iterations(args.warmup, K, LR, 1, want_losses=False)
    ctx.sync()
    clocks = Clocks(physical_gpu(local_rank))
    barrier()
    ctx.sync()
    clocks.start()
    launches0 = ctx.kernel_launches
    step_ms = device_steps(ctx, args, args.warmup + 1, args.steps)
    ctx.sync()
    barrier()
    clk = clocks.stop()
    launches = ctx.kernel_launches - launches0  # our kernels only (the L2 flush is a memset)
    # per-family breakdown: the same steps again from the same start state
    # (the trajectory is deterministic), with profiling events between the
    # families -- which break the launch chain, so this pass is not timed
    ctx.set_params(params)
    ctx.train_iterations(args.warmup, K, LR, 1, want_losses=False)
    ctx.profile_enable(True)
    for s in range(args.steps):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.train_iterations(1, K, LR, args.warmup + 1 + s, want_losses=False)
    ctx.sync()
    prof = {PROF_NAMES[f]: ctx.profile_read(f) for f in range(len(PROF_NAMES))}
    ctx.profile_enable(False)
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = args.steps / (total_ms / 1e3)

    # ---- e2e through the public host-buffer call --------------------------------
    # igs_train_iteration_async / igs_train_wait pipelined two deep, as igs_fit
    # drives it: every step copies its sample indices from pinned host memory
    # and reads its loss + status back.  Device marks bracket each step (after
    # its L2 flush, through its D2H read); the host enqueue of step s+1
    # overlaps step s.  The host wall clock of the whole loop (flushes
    # included) is reported beside it.
    ctx.set_params(params)  # fresh state: moments zero, same trajectory start
    for s in range(args.warmup):
        ctx.train_iteration(mine[s], K, LR, s + 1)
    barrier()
    ctx.sync()
    wall0 = time.perf_counter()
    for s in range(args.steps):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.timer_mark(2 * s)
        ctx.train_iteration_async(mine[args.warmup + s], K, LR, args.warmup + 1 + s)
        ctx.timer_mark(2 * s + 1)
        if s > 0:
            ctx.train_wait()
    ctx.train_wait()
    wall = time.perf_counter() - wall0
    e2e_ms = [ctx.timer_between(2 * s, 2 * s + 1) for s in range(args.steps)]
    # the flushes inside the wall-clock loop, timed alone (device events)
    flush_ms = []
    for _ in range(args.steps):
        ctx.timer_begin()
        ctx.flush_l2(FLUSH_BYTES)
        flush_ms.append(ctx.timer_end())
    wall_excl_flush = max(wall - sum(flush_ms) / 1e3, 1e-9)
    barrier()
    e2e_total = max_over_ranks(sum(e2e_ms))
    e2e_value = args.steps / (e2e_total / 1e3)
    wall = max_over_ranks(wall)
    wall_excl_flush = max_over_ranks(wall_excl_flush)

    # ---- roofline of the dominant kernel family ----------------------------------
    fam_ms = {k: v[0] for k, v in prof.items()}
    dom = max(fam_ms, key=fam_ms.get)
    scan_ms, scan_launches, scan_pairs = prof["scan"]
    roof = None
    if scan_ms > 0:
        achieved = scan_pairs * OPS_PER_PAIR / (scan_ms * 1e-3)
        roof = {"kernel": "top-K candidate scan (IGS_PROF_SCAN)", "bound": "fp64",
                "achieved": achieved / 1e9, "peak": fp64_peak / 1e9, "unit": "Gop/s (fp64 add/mul pipe)",
                "frac": achieved / fp64_peak, "traffic": ncu_traffic("knn_points16_kernel"),
                "work_per_launch": f"{scan_pairs / max(scan_launches, 1):.4g} (pixel, candidate) pairs x "
                                   f"{OPS_PER_PAIR} fp64 ops",
                "peak_source": "measured in this run (igs_fp64_peak: independent DMUL/DADD chains, all SMs); "
                               "MEASURED_PEAKS.json has no fp64 figure",
                "avg_launch_us": scan_ms * 1e3 / max(scan_launches, 1),
                # the fraction uses executed pairs; the reference's
                # own work (its global scan) is NS x N pairs per iteration
                "reference_equivalent_pairs_per_launch": float(NS) * N / world,
                "reference_equivalent_gop_s": float(NS) * N / world * OPS_PER_PAIR / (
                    scan_ms * 1e-3 / max(scan_launches, 1)) / 1e9}
    # the search is issue-bound (ncu: ~54 % of issue slots busy), so its
    # other roofline is instruction issue: the committed capture's warp
    # instructions per launch over this run's launch time, against 4 warp
    # instructions per cycle per SM at the SM clock
    issue_roof = None
    ninstr = ncu_field("knn_points16_kernel", "warp_instructions_per_launch")
    if scan_ms > 0 and ninstr:
        try:
            import torch
            sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
        except Exception:
            sms = 148
        mhz = float(clk.get("sm_max_mhz") or 1965.0)
        peak_wi = sms * 4 * mhz * 1e6
        wi_s = ninstr / (scan_ms * 1e-3 / max(scan_launches, 1))
        issue_roof = {"kernel": "top-K candidate scan (knn_points16_kernel)", "bound": "issue",
                      "achieved": wi_s / 1e9, "peak": peak_wi / 1e9, "unit": "G warp-instructions/s",
                      "frac": wi_s / peak_wi,
                      "work_per_launch": f"{ninstr:.4g} warp instructions (profiles/r2_traffic.json, ncu at "
                                        "--steps 20 --warmup 5)",
                      "peak_source": f"{sms} SMs x 4 schedulers x {mhz:.0f} MHz"}
    adam_ms, adam_launches, adam_bytes = prof["adam"]
    hbm = None
    try:
        hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs")
    except Exception:
        pass
    adam_roof = None
    if adam_ms > 0 and hbm:
        gbs = adam_bytes / (adam_ms * 1e-3) / 1e9
        adam_roof = {"kernel": "fused Adam+constrain+prepare", "bound": "hbm", "achieved": gbs, "peak": hbm,
                     "unit": "GB/s", "frac": gbs / hbm, "traffic": ncu_traffic("segment_adam_kernel"),
                     "bytes_per_gaussian": 596}

    # ---- secondary: full render Mpix/s (tile-row bands across ranks) ---------------
    render = None
    if not args.no_render:
        r0, r1 = D.row_band(H, rank, world)
        ctx.render_image_rows(W, H, K, r0, r1, host=False)
        ctx.sync()
        rms = []
        for _ in range(3):
            ctx.flush_l2(FLUSH_BYTES)
            barrier()
            ctx.timer_begin()
            ctx.render_image_rows(W, H, K, r0, r1, host=False)
            rms.append(ctx.timer_end())
        r_ms = max_over_ranks(min(rms))
        ctx.profile_enable(True)
        ctx.render_image_rows(W, H, K, r0, r1, host=False)
        ctx.sync()
        r_pairs = ctx.profile_read(PROF_SCAN)[2]
        ctx.profile_enable(False)
        render = {"metric": f"global top-K render Mpix/s (render_image, {W}x{H}, {N // 1000}k G, K=10)",
                  "value": W * H / (r_ms * 1e-3) / 1e6, "unit": "Mpix/s", "ms": r_ms,
                  "pairs_per_pixel": r_pairs / max(r1 - r0, 1) / W,
                  "roofline": {"bound": "fp64", "achieved": r_pairs * OPS_PER_PAIR / (r_ms * 1e-3) / 1e9,
                               "peak": fp64_peak / 1e9, "unit": "Gop/s",
                               "frac": r_pairs * OPS_PER_PAIR / (r_ms * 1e-3) / fp64_peak,
                               "work": "executed (pixel, candidate) pairs x 14 fp64 ops (rank 0's band)"},
                  "state": f"the set after {args.warmup + args.steps} training steps",
                  "note": f"L2 flushed before each render; {world} rank(s), each renders its tile-row band "
                          "(igs_render_image_rows, no communication); time = max over ranks"}
    secondary = None
    if world == 1 and not args.no_secondary:
        secondary = {"c1": secondary_c1(ctx), "c3": secondary_c3(ctx), "c4": secondary_c4(ctx),
                     "c5": secondary_c5(ctx), "fit_c2": secondary_fit(ctx)}
    elif world > 1 and not args.no_secondary:
        # configs[4] across the ranks: 64 textures, 64 / N per GPU, no communication;
        # the sweep time is the max over ranks
        barrier()
        c5 = secondary_c5(ctx, range(rank, 64, world))
        c5_ms = max_over_ranks(c5["sweep_ms"])
        secondary = {"c5_all_ranks": {"config": f"C5: 64 x 1024x1024 textures over {world} GPUs ({64 // world} each), "
                                                "50k G, 5 LoD prefixes each, blocked (n_max 64)",
                                      "sweep_ms_max_over_ranks": c5_ms, "renders": 320,
                                      "mpix_s_incl_partition": 320 * 1024 * 1024 / c5_ms / 1e3}}

    out = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded mt19937_64 generators of the reference test suite)",
        "config": bench_config(wl, world),
        "options": {"l2": "flushed before every timed step (512 MiB memset on the stream, outside the events)",
                    "cull": ctx.get_option(1), "deterministic_reduction": ctx.get_option(2),
                    "shard_adam": ctx.get_option(5)},
        "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": int(mine.shape[1]) * 4,
                "d2h_bytes_per_step": 8 + 32 + int(mine.shape[1]) * 8 * world,
                "wall_clock_value": args.steps / wall,
                "wall_clock_value_excl_flush": args.steps / wall_excl_flush,
                "call": "igs_train_iteration_async + igs_train_wait, pipelined two deep (host sample indices in; "
                        "host status, loss and the per-sample losses the host sums in sample order out, every "
                        "step)",
                "wall_clock_note": "host perf_counter over the whole loop, including the 512 MiB L2 flush "
                                   "memsets between steps; _excl_flush subtracts those memsets' device time "
                                   "(timed alone)"},
        "roofline": roof, "roofline_issue": issue_roof, "roofline_adam": adam_roof,
        "profile_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]},
        "knn_hard_points_per_step": prof["knn_hard"][2] / args.steps,
        "pairs_per_sample": prof["scan"][2] / args.steps / max(NS // world, 1),
        "dominant_family": dom,
        "clocks": clk, "gpu_launches": int(launches),
        "render": render, "secondary": secondary,
    }
    if baseline:
        out["scaling_baseline"] = baseline
    return out, ctx


def _best_ms(ctx, f, reps=3):
    best = 1e30
    for _ in range(reps):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.timer_begin()
        f()
        best = min(best, ctx.timer_end())
    return best


def secondary_c1(ctx):
    """configs[0] (C1): random-local N = 10k at 512x512, K = 10 --
    one global render, one train step (NS = 10k) + Adam (t = 1)."""
    from paper_2407_01866_b200 import synth
    W = H = 512
    params = synth.random_local_set(10_000, W, H, seed=7)
    ctx.set_params(params)
    ctx.set_target(synth.photo_like_image(W, H, 31002))
    sidx = synth.sample_indices(NS, W, H, seed=99)[0]
    ctx.render_image(W, H, K, host=False)
    r_ms = _best_ms(ctx, lambda: ctx.render_image(W, H, K, host=False))

    def step():
        ctx.set_params(params)
        ctx.train_iteration(sidx, K, LR, 1)
    step()
    t_ms = _best_ms(ctx, step)
    return {"config": "C1: random-local 10k G at 512x512, K=10", "render_ms": r_ms,
            "render_mpix_s": W * H / r_ms / 1e3, "train_step_plus_adam_ms": t_ms,
            "note": "the train step time includes re-uploading the set (set_params) so every repetition is t = 1"}


def secondary_c3(ctx):
    """configs[2] (C3): random-local N = 250k at 4096x4096 -- build_partition(64),
    IGS2 encode, decode (device unpack + rebuild_partition from the stored
    corners, the decoded set becoming resident), blocked render of the
    decoded set, random point queries; and the global render."""
    from paper_2407_01866_b200 import synth
    W = H = 4096
    ctx.set_params(synth.random_local_set(250_000, W, H, seed=7))
    ctx.partition_build(64)
    build_ms = _best_ms(ctx, lambda: ctx.partition_build(64))
    # the IGS2 file (set + block corners, binary16) and its decode:
    # unpack + constrain on the device, rebuild_partition from the corners
    data = ctx.encode(W, H, K, with_partition=True)
    encode_ms = _best_ms(ctx, lambda: ctx.encode(W, H, K, with_partition=True))
    ctx.decode(data)
    decode_ms = _best_ms(ctx, lambda: ctx.decode(data))
    ctx.render_image_blocked(W, H, K, host=False)
    blocked_ms = _best_ms(ctx, lambda: ctx.render_image_blocked(W, H, K, host=False))
    rng = np.random.default_rng(1)
    uv10k, uv1m = rng.random((10_000, 2)), rng.random((1_000_000, 2))
    ctx.render_points_blocked(uv10k, K)
    pts10k_ms = _best_ms(ctx, lambda: ctx.render_points_blocked(uv10k, K))
    pts1m_ms = _best_ms(ctx, lambda: ctx.render_points_blocked(uv1m, K))
    ctx.render_image(W, H, K, host=False)
    glob_ms = _best_ms(ctx, lambda: ctx.render_image(W, H, K, host=False))
    return {"config": "C3: random-local 250k G at 4096x4096, K=10, n_max=64", "partition_build_ms": build_ms,
            "encode_ms": encode_ms, "file_bytes": len(data), "decode_ms": decode_ms,
            "blocked_render_ms": blocked_ms,
            "blocked_render_mpix_s": W * H / blocked_ms / 1e3, "point_queries_10k_ms": pts10k_ms,
            "point_queries_1m_ms": pts1m_ms, "global_render_ms": glob_ms,
            "global_render_mpix_s": W * H / glob_ms / 1e3,
            "note": "point queries include the host->device copy of (u, v) and the result copy back"}


def secondary_c4(ctx):
    """configs[3] (C4) on one GPU: random-local N = 1M, 8192x8192 photo-like
    target (a 2048x2048 photo-like image upsampled 4x, nearest -- the
    generator itself takes a minute at 8192^2), train iterations/s (20 steps,
    L2 flushed before each), and the global render."""
    from paper_2407_01866_b200 import synth
    W = H = 8192
    ctx.set_params(synth.random_local_set(1_000_000, W, H, seed=7))
    small = synth.photo_like_image(2048, 2048, 31004)
    ctx.set_target(np.ascontiguousarray(small.repeat(4, axis=0).repeat(4, axis=1)))
    ctx.upload_samples(synth.sample_indices(NS, W, H, seed=99, steps=30))
    ctx.train_iterations(5, K, LR, 1, want_losses=False)
    ms = []
    for s in range(20):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.timer_begin()
        ctx.train_iterations(1, K, LR, 6 + s, want_losses=False)
        ms.append(ctx.timer_end())
    ctx.render_image(W, H, K, host=False)
    glob_ms = _best_ms(ctx, lambda: ctx.render_image(W, H, K, host=False))
    return {"config": "C4 (1 GPU): random-local 1M G, 8192x8192, NS=10k, K=10",
            "train_iters_per_s": 1e3 * len(ms) / sum(ms), "ms_per_step": sum(ms) / len(ms),
            "global_render_ms": glob_ms, "global_render_mpix_s": W * H / glob_ms / 1e3}


def secondary_c5(ctx, textures=range(8)):
    """configs[4] (C5): texture-like 1024x1024 sets of 50k random-local
    Gaussians; for each, the LoD prefixes {25k, 31.25k, 37.5k, 43.75k, 50k}
    (fit.cpp:182-201's stage counts) are partitioned (n_max 64) and rendered
    blocked.  One GPU's share of the 64 textures is 8 of them; with N ranks
    rank r takes textures r, r + N, ... (64 / N each)."""
    from paper_2407_01866_b200 import synth
    W = H = 1024
    sets = [synth.random_local_set(50_000, W, H, seed=100 + t) for t in textures]
    prefixes = [25_000, 31_250, 37_500, 43_750, 50_000]

    def sweep():
        for p in sets:
            for m in prefixes:
                ctx.set_params(p[:m])
                ctx.partition_build(64)
                ctx.render_image_blocked(W, H, K, host=False)
    sweep()
    ms = _best_ms(ctx, sweep, reps=2)
    n = 5 * len(sets)
    return {"config": f"C5: {len(sets)} x 1024x1024 textures on this GPU, 50k G, 5 LoD prefixes each, blocked "
                      "(n_max 64)", "sweep_ms": ms, "renders": n, "mpix_s_incl_partition": n * W * H / ms / 1e3}


def secondary_fit(ctx):
    """configs[1] as its text states it: a full C2 optimisation (SURVEY.md 8d
    compressed schedule) -- igs_fit end to end (host init and alias tables,
    device iterations, device BSP evaluation renders), after a short warm-up
    fit."""
    import time
    from paper_2407_01866_b200 import Context, synth
    target = synth.photo_like_image(C2["W"], C2["H"], 31001)
    ctx.fit(target, Context.fit_config(budget=100_000, iterations=200, eval_interval=1000, warmup_iters=100,
                                       densify_interval=50))
    cfg = Context.fit_config(budget=100_000, iterations=5000, eval_interval=500, warmup_iters=1000,
                             densify_interval=1000)
    t0 = time.perf_counter()
    rep = ctx.fit(target, cfg)
    wall = time.perf_counter() - t0
    # the trained state (t = 5000: larger, rotated Gaussians, deeper searches):
    # 20 more device-resident iterations from it, L2 flushed before each
    ctx.upload_samples(synth.sample_indices(NS, C2["W"], C2["H"], seed=98, steps=25))
    ctx.train_iterations(5, K, LR, 5001, want_losses=False)
    ms = []
    clocks = Clocks(physical_gpu(int(os.environ.get("LOCAL_RANK", "0"))))
    clocks.start()
    for s in range(20):
        ctx.flush_l2(FLUSH_BYTES)
        ctx.timer_begin()
        ctx.train_iterations(1, K, LR, 5006 + s, want_losses=False)
        ms.append(ctx.timer_end())
    clk = clocks.stop()
    return {"config": "C2 fit (SURVEY.md 8d schedule): 2048x2048, budget 100k (50k init + 4 x 12.5k), 5000 "
                      "iterations, warmup 1000, densify every 1000, eval every 500",
            "wall_s": wall, "iters_per_s_incl_everything": 5000 / wall, "final_count": rep["final_count"],
            "psnr_per_eval": [round(e["psnr"], 4) for e in rep["evals"]],
            "trained_state_step": {"t": "5006-5025", "iters_per_s": 1e3 * len(ms) / sum(ms),
                                   "ms_per_step": sum(ms) / len(ms),
                                   "ms_per_step_median": statistics.median(ms),
                                   "ms_per_step_min_max": [min(ms), max(ms)], "clocks": clk,
                                   "note": "the fitted 100k set (t = 5000), uniform samples, L2 flushed per step"}}


def ncu_field(kernel: str, field: str):
    try:
        return json.loads((ROOT / "profiles" / "r2_traffic.json").read_text())[kernel][field]
    except Exception:
        return None


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture summary (profiles/r2_traffic.json), or None."""
    try:
        d = json.loads((ROOT / "profiles" / "r2_traffic.json").read_text())
        return d[kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------- reference
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_steps(steps: int, warmup: int, budget_s: float, wl: dict = C2):
    """The unmodified reference (oracle/_ref) fit iteration on the same workload."""
    import oracle
    from paper_2407_01866_b200 import synth
    if not oracle.available("reference"):
        return None
    R = oracle.get("reference")
    params, target = make_inputs(wl)
    W_IMG, H_IMG = wl["W"], wl["H"]
    samples = synth.sample_indices(NS, W_IMG, H_IMG, seed=99, steps=max(steps + warmup, 1))
    import ctypes as C
    p = np.ascontiguousarray(params.copy())
    m = np.zeros_like(p); v = np.zeros_like(p)
    tg = np.ascontiguousarray(target)
    lr = np.ascontiguousarray(LR, np.float64)
    loss = C.c_double(0)
    dp = C.POINTER(C.c_double)

    def one(s, t):
        si = np.ascontiguousarray(samples[s])
        code = R.lib.ref_train_iteration(p.ctypes.data_as(dp), p.shape[0], m.ctypes.data_as(dp),
                                         v.ctypes.data_as(dp), tg.ctypes.data_as(C.POINTER(C.c_float)), W_IMG,
                                         H_IMG, si.ctypes.data_as(C.POINTER(C.c_uint32)), NS, K,
                                         lr.ctypes.data_as(dp), t, C.byref(loss))
        if code:
            raise RuntimeError(f"reference train iteration failed: {code}")

    for s in range(warmup):
        one(s, s + 1)
    times = []
    t_start = time.perf_counter()
    for s in range(steps):
        t0 = time.perf_counter()
        one(warmup + s, warmup + s + 1)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s and len(times) >= 2:
            break
    return times


def cpu_baseline_block(budget_s=20.0):
    times = run_reference_steps(steps=1000, warmup=1, budget_s=budget_s)
    if times is None:
        return None
    return {"value": len(times) / sum(times), "unit": "iters/s", "cores": cpu_threads(), "kind": "reference",
            "sample": f"{len(times)} full C2 iterations (100k G, 10k samples, K=10) of the unmodified reference "
                      f"(oracle/_ref, OpenMP, {cpu_threads()} threads) after 1 warm-up, ~{budget_s:.0f} s budget"}


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without a launcher: one process per GPU under
    torch.distributed.run (the driver's own launch line), same arguments."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        wl = workload_for(world)
        steps = args.steps
        times = run_reference_steps(steps, args.warmup, budget_s=150.0, wl=wl)
        if times is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libigs_ref.so not built"}))
            return 0
        v = len(times) / sum(times)
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world,
               "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded mt19937_64 generators of the reference test suite)",
               "config": bench_config(wl, world),
               "cpu_baseline": {"value": v, "unit": "iters/s", "cores": cpu_threads(), "kind": "reference",
                                "sample": f"{len(times)} of {steps} requested full {wl['name']} iterations of the "
                                          f"unmodified reference (oracle/_ref, OpenMP, {cpu_threads()} threads; "
                                          "150 s cap)"},
               "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return 0

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    out, ctx = run_ours(args, rank, world, local_rank, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_block()
    if rank == 0:
        print(json.dumps(out))
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
