#!/usr/bin/env python
"""Benchmark of the B200 MPM hot path (BASELINE.json metric: particle-substeps/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c5|c1|c2|c3] [--replicas R]

One step = one frame (dt 0.02 s; 10 MLS substeps, or 1 PB-MPM step of 10 iterations for
c3) of every scene on this rank.  Default workload: C5 shard = R=512 independent
64,800-particle cutting replicas per GPU (the batched RL data-generation config of
BASELINE.json; 4096 replicas over 8 GPUs), weak scaling over ranks, no data-path
collective.  ``value`` is device-resident (CUDA events on the library's stream, max over
ranks); ``e2e`` goes through the public facade with host buffers every frame (pose-table
H2D from pinned memory, FrameResult D2H).  ``--impl reference`` times the UNMODIFIED
reference CPU implementation (oracle/_ref, compiled from /root/reference) on the host
cores with all threads, on the same workload and metric.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

METRIC = "particle-substeps/sec"
UNIT = "particle-substeps/s"
DT_FRAME = 0.02
# Algorithmic (compulsory) bytes per particle per launch:
#   p2g   108 = read x, v, C, F, mass, volume0, flags
#   g2p   148 = read x, F, flags (52) + write x, v, C, F (96)
#   fused k_g2p2g (G2P of substep s + P2G of s+1): v and C need not persist between the two
#         phases, so the compulsory state traffic is read x, F, mass, volume0, flags (60) +
#         write x, F (48) = 108 B, plus the grid: the G2P phase reads and the P2G phase
#         accumulates ~0.2 active nodes per particle (SURVEY.md §8 probe) x 16 B each = 6.4 B.
#         §8d: "report it with its own denominator (108 + grid); do not divide by 204".
#   PB-MPM (c3) per particle-iteration: 168 B (P2G reads x, v, C, mass, flags = 68; G2P reads
#         x, F, flags = 52 and writes v, C = 48); the fused PB kernel moves one iteration.
GRID_BYTES = 0.2 * 2 * 16.0
ALG_BYTES = {"p2g": 108.0, "g2p": 148.0, "grid": 0.0, "sort": 224.0, "fused": 108.0 + GRID_BYTES}
ALG_BYTES_PB = {"p2g": 68.0, "g2p": 100.0, "grid": 0.0, "sort": 224.0, "fused": 168.0}
SUBSTEP_BYTES = 204.0
SUBSTEP_BYTES_PB = 172.8
# Untimed pre-roll frames before the warm-up: the cutting workloads' blade reaches the tissue
# only after it has fallen and bounced (oracle probe, C5 replica 0: first blade impulse and
# push-out at frame 53, t = 1.08 s), so the timed frames start inside the cut.
PREROLL = {"c5": 55, "c2": 55, "m1": 65}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c1", "c2", "c3", "c4", "m1"])
    ap.add_argument("--preroll", type=int, default=None,
                    help="untimed frames before the warm-up (default: PREROLL[workload], 0 for others)")
    ap.add_argument("--replicas", type=int, default=512, help="C5 replicas per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dd", action="store_true", help="c4 through slab DD even at N=1 (one slab)")
    ap.add_argument("--fusion", type=int, default=1, choices=[0, 1, 2],
                    help="substep fusion (mpmb_set_fusion): 0 off, 1 auto, 2 always")
    return ap.parse_args()


def shard_replicas(rank, replicas):
    """Replica ids of this rank: a contiguous block of `replicas` (weak scaling; replica r
    has seed 4242 + r and its own blade jitter, so the union over ranks is 0..N*R-1)."""
    return list(range(rank * replicas, (rank + 1) * replicas))


def workload_specs(name, rank, replicas):
    from paper_2502_18437_b200 import scenes
    if name == "c5":
        return [scenes.c5_cutting_replica(r) for r in shard_replicas(rank, replicas)]
    return [{"c1": scenes.c1_cube_drop, "c2": scenes.c2_cutting, "c3": scenes.c3_suture,
             "c4": scenes.c4_slab, "m1": scenes.m1_cutting}[name]()]


def preroll_of(args):
    return PREROLL.get(args.workload, 0) if args.preroll is None else args.preroll


def reduce_over_ranks(ms, ms_e2e, n_particles, world, device):
    """Whole-job timing = MAX over ranks of the device-timed region; particle count = SUM."""
    if world <= 1:
        return ms, ms_e2e, float(n_particles)
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms, ms_e2e], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    cnt = torch.tensor([float(n_particles)], device=device, dtype=torch.float64)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    return float(t[0]), float(t[1]), float(cnt[0])


def workload_desc(name, replicas, n_per_gpu):
    if name == "c5":
        return (f"C5 shard: {replicas} independent cutting replicas x 64,800 p per GPU, 84^3 grid each, "
                f"MLS 10 substeps/frame, quad-slicer blade (BASELINE.json configs[4])")
    return {"c1": "C1 cube drop, MLS, 32,768 p, 64^3", "c2": "C2 cutting, MLS, 262,144 p, 128^3",
            "m1": "M1 north-star scene: one 1,049,600-particle MLS tissue block cut by the quad-slicer blade "
                  "(cutting.json rescaled to 128^3, dx 1.4/128)",
            "c4": "C4 tissue slab on a floor, MLS 20 substeps/frame, 8,388,608 p, 512^3 (slab DD over NCCL "
                  "when N > 1)",
            "c3": "C3 suture, PB-MPM K=10, 262,144 p, 128^3, arc needle + 16 free thread capsules"}[name]


def substeps_of(spec):
    return spec.get("iterations", 10) if spec["solver"] == "pbmpm" else spec.get("substeps", 10)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 50 ms from before the warm-up on.
    stop() keeps the samples stamped inside the timed region (mark_start / mark_end); a region
    shorter than nvidia-smi's start-up + one period falls back to the samples under load just
    before it (the warm-up frames), flagged in_region = False."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark_start(self):
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f")
                rows.append((ts, float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        inside = [r for r in rows if self.t0 and self.t1 and self.t0 <= r[0] <= self.t1]
        sel, in_region = inside, True
        if not sel:  # region too short for the sampler: the samples just before it
            sel, in_region = [r for r in rows if self.t1 is None or r[0] <= self.t1][-3:], False
        reasons = set()
        for r in sel:
            for nm, val in zip(names, r[3]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm = [r[1] for r in sel]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": sel[-1][2] if sel else None,
                "reasons": sorted(reasons), "samples": len(sm), "in_region": in_region}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per particle per launch from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


# ------------------------------------------------------------------ reference arm
def reference_scenes(specs):
    import backends
    out = []
    for sp in specs:
        sc = backends.make_scene("ref", sp)
        out.append((sc, sp))
    return out


class RefSet:
    """`threads` independent reference scenes (oracle/_ref/libmpmref.so: the UNMODIFIED
    reference code), advanced together on `threads` host threads, one scene per thread."""

    def __init__(self, specs, threads, preroll=0):
        import ctypes as C
        import backends
        self.lib = backends.reference()
        self.scs = reference_scenes(specs)
        self.hs = (C.c_uint64 * len(self.scs))(*[sc.h for sc, _ in self.scs])
        self.threads = threads
        self.n = sum(sc.particle_count() for sc, _ in self.scs)
        self.sub = substeps_of(specs[0])
        if preroll:
            self.advance(preroll)

    def advance(self, frames):
        """Wall seconds of `frames` frames of every scene (advance + fetch_results)."""
        return self.lib.mpmref_advance_many(self.hs, len(self.scs), DT_FRAME, frames, self.threads)

    def rate(self, frames, wall):
        return self.n * self.sub * frames / wall

    def destroy(self):
        for sc, _ in self.scs:
            sc.destroy()


def cpu_specs_fn(workload):
    from paper_2502_18437_b200 import scenes

    def fn(threads):
        if workload == "c5":
            return [scenes.c5_cutting_replica(i) for i in range(threads)]
        return workload_specs(workload, 0, 1) * 1
    return fn


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank):
    if rank != 0:
        return None
    if args.workload == "c4":
        from paper_2502_18437_b200 import scenes
        vals, t_total = [], 0.0
        for _ in range(args.warmup):
            time_reference_substeps(scenes.c4_slab(), args.cpu_seconds / max(args.steps, 1))
        for _ in range(args.steps):
            r, w, n, k = time_reference_substeps(scenes.c4_slab(), args.cpu_seconds / max(args.steps, 1))
            vals.append(r)
            t_total += w
        value = statistics.median(vals)
        return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * t_total / max(args.steps, 1), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
                "config": {"workload": workload_desc("c4", 0, None), "parallelism": "1 host thread"},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                                 "sample": f"{k} step_mls substeps per step on all {n} particles"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    threads = cpu_threads() if args.workload == "c5" else 1
    pre = preroll_of(args) if args.workload != "m1" else 0
    rs = RefSet(cpu_specs_fn(args.workload)(threads), threads, pre)
    # size one step to ~cpu_seconds/steps: probe one frame first (it is part of the pre-roll)
    wall1 = rs.advance(1)
    frames = max(1, int(round(args.cpu_seconds / max(wall1, 1e-3) / max(args.steps, 1))))
    for _ in range(args.warmup):
        rs.advance(frames)
    vals, t_total = [], 0.0
    for _ in range(args.steps):
        w = rs.advance(frames)
        vals.append(rs.rate(frames, w))
        t_total += w
    n, sub = rs.n, rs.sub
    rs.destroy()
    value = statistics.median(vals)
    sample = (f"{threads} concurrent reference scenes ({'C5 replicas' if args.workload == 'c5' else args.workload}), "
              f"{frames} frame(s) x {sub} substeps per step, {n} particles total, after {pre + 1} untimed frames")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_total / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_desc(args.workload, args.replicas, None) +
                       (f"; timed frames after {pre + 1} untimed pre-roll frames (blade in the tissue)" if pre else ""),
                       "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


# ------------------------------------------------------------------ our arm
def build_batch(specs):
    from paper_2502_18437_b200 import api, scenes
    cfg = api.scene_config(**scenes.config_kwargs(specs[0]))
    if len(specs) == 1:
        b = api.SceneBatch(cfg, 1)
    else:
        b = api.SceneBatch(cfg, len(specs))
    for sc, sp in zip(b.scenes, specs):
        scenes.populate(sc, sp)
    return b


def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    specs = workload_specs(args.workload, rank, args.replicas)
    sub = substeps_of(specs[0])
    t0 = time.time()
    batch = build_batch(specs)
    batch.set_fusion(args.fusion)
    # a real (non-legacy) stream shared by the library launches and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    batch.set_stream(stream.cuda_stream)
    lib = batch.lib
    n_particles = sum(s.particle_count() for s in batch.scenes)
    n_shapes = sum(len(s.shapes) for s in batch.scenes)
    setup_s = time.time() - t0

    # clocks: nvidia-smi needs ~0.1 s to start; it runs from the warm-up on
    clocks = ClockSampler(local_rank)
    clocks.start()
    pre = preroll_of(args)
    # untimed pre-roll (cutting workloads: until the blade is in the tissue), then the warm-up
    if pre:
        batch.advance_frames(DT_FRAME, pre)
        batch.fetch_results()
    batch.advance_frames(DT_FRAME, max(args.warmup, 1))
    batch.fetch_results()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def fresh_batch(old):
        """A new batch warmed like the first, so it simulates the SAME frames (later frames
        cost more: the tissue lands on the floor)."""
        old.destroy()
        b = build_batch(specs)
        b.set_fusion(args.fusion)
        b.set_stream(stream.cuda_stream)
        if pre:
            b.advance_frames(DT_FRAME, pre)
            b.fetch_results()
        b.advance_frames(DT_FRAME, max(args.warmup, 1))
        b.fetch_results()
        barrier()
        torch.cuda.synchronize()
        return b

    # Timing rule: between timed steps either flush L2 or use inputs larger than L2.  A state
    # of at least twice the L2 is streamed through it every substep; a smaller one (C1-C3) is
    # timed step by step with a write of twice the L2 between steps (outside the events), and
    # a device sleep after it so the host has the whole frame enqueued before the first event.
    l2_bytes = torch.cuda.get_device_properties(local_rank).L2_cache_size
    flush_l2 = n_particles * 112 < 2 * l2_bytes
    scrub = torch.empty(2 * l2_bytes // 4, dtype=torch.int32, device="cuda") if flush_l2 else None

    def timed(b):
        """device ms of args.steps frames of batch b (frames fetched after the last event)"""
        if not flush_l2:
            t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            b.advance_frames(DT_FRAME, args.steps)
            t1e.record(stream)
            t1e.synchronize()
            b.fetch_results()
            return t0e.elapsed_time(t1e)
        total = 0.0
        for k in range(args.steps):
            scrub.fill_(k)
            torch.cuda._sleep(4_000_000)  # ~2 ms: the host enqueues the frame meanwhile
            t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            b.advance_frames(DT_FRAME, 1)
            t1e.record(stream)
            t1e.synchronize()
            total += t0e.elapsed_time(t1e)
            b.fetch_results()
        return total

    # ---- value: device-resident, CUDA events on the library stream; no per-kernel events
    # inside (they cost up to 35% on small scenes) -- the kernel split comes from a profiled
    # replay of the same frames below
    barrier()
    torch.cuda.synchronize()
    launches0 = lib.mpmb_kernel_launch_count()
    clocks.mark_start()
    ms = timed(batch)
    clocks.mark_end()
    torch.cuda.synchronize()
    launches = lib.mpmb_kernel_launch_count() - launches0
    clk = clocks.stop()

    # ---- kernel split (roofline): the same frames with per-kernel-class CUDA events
    batch = fresh_batch(batch)
    batch.set_profiling(True)
    ms_profiled = timed(batch)
    prof = batch.profile()
    batch.set_profiling(False)

    # ---- e2e: public facade, host buffers every frame, on the same frames again: the two
    # numbers differ only by the host path.  The caller's FrameResult arrays (one x / v /
    # active array over every scene, allocated once like a data-generation consumer would)
    # are bound with mpmb_bind_results, so each frame's D2H lands in them directly; the
    # frame's arrays are complete (mpmb_result_wait) before the next frame's copy is issued,
    # and the last frame's copy is inside the timed region.
    batch = fresh_batch(batch)
    hx = np.empty((n_particles, 3), np.float32)
    hv = np.empty((n_particles, 3), np.float32)
    ha = np.empty(n_particles, np.uint8)
    batch.bind_results(hx, hv, ha)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    batch.advance(DT_FRAME)
    for k in range(args.steps):
        batch.fetch_results()
        if k + 1 < args.steps:
            batch.advance(DT_FRAME)  # frame k+1 runs on the device while frame k's arrays land
        batch.wait_results()  # frame k's x / v / active are in hx / hv / ha
    f1.record(stream)
    f1.synchronize()
    ms_e2e = f0.elapsed_time(f1)
    batch.bind_results()

    ms, ms_e2e, n_total = reduce_over_ranks(ms, ms_e2e, n_particles, world, "cuda")

    ps = n_total * sub * args.steps
    value = ps / (ms / 1e3)
    e2e = ps / (ms_e2e / 1e3)
    peak, peak_src = measured_peak()
    # dominant kernel class and its roofline (per-launch averages over the timed region)
    # with substep fusion (mpmb_set_fusion) the frame runs P2G and G2P alone once each and
    # k_g2p2g sub-1 times
    # operations per class in the profiled replay, counted by the library (substep fusion and
    # cross-frame fusion change how many standalone P2G / G2P launches a frame has)
    launches_per_class = {"p2g": prof["n_p2g"], "g2p": prof["n_g2p"], "grid": prof["n_grid"],
                          "sort": prof["n_sort"], "fused": prof["n_fused"]}
    cls_ms = {"p2g": prof["ms_p2g"], "g2p": prof["ms_g2p"], "grid": prof["ms_grid"], "sort": prof["ms_sort"],
              "fused": prof["ms_fused"]}
    dom = max(cls_ms, key=lambda k: cls_ms[k])
    per_launch_ms = cls_ms[dom] / max(launches_per_class[dom], 1)
    pb = specs[0]["solver"] == "pbmpm"
    alg_table = ALG_BYTES_PB if pb else ALG_BYTES
    alg = alg_table[dom] * n_particles
    achieved = alg / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    tr = ncu_traffic()
    traffic = None
    if tr and dom in tr.get("bytes_per_particle", {}):
        traffic = tr["bytes_per_particle"][dom] * n_particles
    h2d = sub * n_shapes * (64 + 1)
    d2h = n_particles * (12 + 12 + 1) + 5 * 8 * len(batch.scenes) + 16 * len(batch.scenes)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(args.workload, args.replicas, n_particles) +
                   (f"; timed frames {pre + max(args.warmup, 1)}..{pre + max(args.warmup, 1) + args.steps - 1} "
                    f"after {pre} untimed pre-roll frames (blade in the tissue)" if pre else ""),
                   "particles_per_gpu": n_particles, "scenes_per_gpu": len(batch.scenes),
                   "substeps_per_step": sub, "parallelism": f"scene replicas x{world} (no collective)",
                   "l2": ("L2 flushed between timed steps (a %.0f MB write outside the events; particle "
                          "state %.1f MB < 2x the %.0f MB L2); e2e not flushed" %
                          (2 * l2_bytes / 1e6, n_particles * 112 / 1e6, l2_bytes / 1e6)) if flush_l2 else
                         ("inputs larger than L2 (%.1f GB particle state per GPU, L2 %.0f MB)" %
                          (n_particles * 112 / 1e9, l2_bytes / 1e6))},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_particle": alg_table[dom], "per_launch_ms": per_launch_ms,
                     "timing": "per-kernel-class CUDA events on the library stream, profiled replay of the "
                               "timed frames (%.2f ms/step with the events vs %.2f without)"
                               % (ms_profiled / args.steps, ms / args.steps),
                     "substep_frac": value * (SUBSTEP_BYTES_PB if pb else SUBSTEP_BYTES) / 1e9 / peak,
                     "substep_bytes_per_particle": SUBSTEP_BYTES_PB if pb else SUBSTEP_BYTES},
        "kernel_ms": {k: v / max(launches_per_class[k], 1) for k, v in cls_ms.items()},
        "clocks": clk,
        "setup_s": setup_s,
    }
    if pb:  # a PB-MPM "substep" is one transfer iteration; steps/s alongside
        line["pbmpm"] = {"iterations_per_step": sub, "particle_steps_per_s": value / sub,
                         "e2e_particle_steps_per_s": e2e / sub}
    return line, batch


def spawn_spec_particles(spec):
    """Every particle of a single-object spec via the product's host spawner
    (mpmb_spawn_box = the reference's create_particle_object lattice, bit-exact)."""
    import ctypes as C
    from paper_2502_18437_b200 import api, capi, scenes
    lib = capi.load_product()
    g = spec["grid"]
    (ob,) = spec["particle_objects"]
    cells = np.prod((np.array(ob["box_max"]) - np.array(ob["box_min"])) / g["dx"] + 2)
    cap = int(cells * ob["particles_per_cell"]) + 1024
    x, m, vol = np.zeros((cap, 3), np.float32), np.zeros(cap, np.float32), np.zeros(cap, np.float32)
    n = C.c_int64()
    api.check(lib.mpmb_spawn_box((capi.i3)(*g["dims"]), float(np.float32(g["dx"])), api._fp(np.array(g["origin"], np.float32)),
                                 api._fp(np.array(ob["box_min"], np.float32)), api._fp(np.array(ob["box_max"], np.float32)),
                                 ob["particles_per_cell"], float(np.float32(ob["density"])), ob["seed"], cap,
                                 api._fp(x), api._fp(m), api._fp(vol), C.byref(n)), lib, "spawn_box")
    k = n.value
    p = api.empty_particles(k)
    p["x"], p["mass"], p["volume0"] = x[:k].copy(), m[:k].copy(), vol[:k].copy()
    mats = [scenes.material_params(ob["material"])]
    shapes = [scenes.shape_spec(s, g["dx"]) for s in spec["shapes"]]
    return p, mats, shapes


def time_reference_substeps(spec, target_s):
    """Bounded CPU sample for a scene too large for whole frames (C4: ~8 s per substep on
    one core): the compiled reference's step_mls with the contact hook on the full particle
    set, as many substeps as fit in ~target_s."""
    import backends
    g = spec["grid"]
    p, mats, shapes = spawn_spec_particles(spec)
    st = backends.state("ref", tuple(g["dims"]), g["dx"], tuple(g["origin"]))
    st.set_materials(mats)
    st.set_particles(p, with_stress=False)
    st.set_shapes(shapes)
    dt = spec["dt_frame"] / spec["substeps"]
    t0 = time.time()
    st.step_mls(dt, spec["gravity"], contact=True)
    one = time.time() - t0
    k = max(1, int(target_s / max(one, 1e-3)))
    t0 = time.time()
    for _ in range(k):
        st.step_mls(dt, spec["gravity"], contact=True)
    wall = time.time() - t0
    n = len(p["mass"])
    return n * k / wall, wall, n, k


def run_ours_dd(args, rank, world, local_rank):
    """C4 across N GPUs: one scene, slab domain decomposition over NCCL through the library's
    device-resident driver (mpmb_dd_run, csrc/dd_driver.cpp: exchanges, contact all-reduce and
    migration issued from C++ on the slab's stream, no host synchronisation inside a frame).
    Strong scaling: the same 8.4M particles whatever N; timing = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2502_18437_b200 import dd, scenes
    torch.cuda.set_device(local_rank)
    spec = scenes.c4_slab()
    g = spec["grid"]
    dims, dx, origin = tuple(g["dims"]), g["dx"], tuple(g["origin"])
    sub = spec["substeps"]
    dt = spec["dt_frame"] / sub
    t0 = time.time()
    p, mats, shapes = spawn_spec_particles(spec)
    n_all = len(p["mass"])
    bx = dd.base_x(p["x"][:, 0], origin[0], dx)
    bounds = dd.slab_bounds(dims[0], world, np.bincount(np.clip(bx, 0, dims[0] - 1), minlength=dims[0]), margin=2)
    mine = np.nonzero(dd.owner_of(bx, bounds) == rank)[0]
    lo, hi = bounds[rank]
    d = dd.SlabDomain(dims, dx, origin, lo, hi, margin=2, capacity=int(1.5 * len(mine)) + 4096)
    d.set_materials(mats)
    d.set_shapes(shapes)
    d.set_particles({k: v[mine] for k, v in p.items()}, mine.astype(np.uint32))
    stream = torch.cuda.Stream()
    d.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [dd.NativeGroup.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        grp = dd.NativeGroup([d], nccl=(uid[0], world, rank))
    else:
        grp = dd.NativeGroup([d])
    setup_s = time.time() - t0
    kw = dict(contact=True, boundary=0, pushout=True, deactivate=True)
    with torch.cuda.stream(stream):
        dd.run_native(grp, sub * max(args.warmup, 1), dt, spec["gravity"], chunk=sub, **kw)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        syncs0, waits0 = grp.stats()["host_syncs"], grp.stats()["host_waits"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):  # one run per frame: the halo window is set per run
            grp.run(sub, dt, spec["gravity"], **kw)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        syncs = grp.stats()["host_syncs"] - syncs0
        grp.check()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        d2h = 0
        for _ in range(args.steps):
            grp.run(sub, dt, spec["gravity"], **kw)
            r = d.download()
            d2h = len(r["ids"]) * (4 + 12 + 12 + 1)
        f1.record(stream)
        f1.synchronize()
        ms_e2e = f0.elapsed_time(f1)
    st = grp.stats()
    ms, ms_e2e, _ = reduce_over_ranks(ms, ms_e2e, 0, world, "cuda")
    ps = n_all * sub * args.steps
    line = {"metric": METRIC, "value": ps / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc("c4", 0, n_all), "particles_total": n_all,
                       "substeps_per_step": sub, "parallelism": f"slab DD x{world} (NCCL halo + migration, "
                                                                "device-resident driver)",
                       "slabs": bounds},
            "e2e": {"value": ps / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h},
            "dd": {"stream_drains_in_timed_region": syncs, "host_waits_in_timed_region": st["host_waits"] - waits0,
                   "fused_substeps": st["fused"], "substeps": st["substeps"], "rebins": st["rebins"]},
            "setup_s": setup_s}
    return line, None


def cpu_baseline(args):
    if args.no_cpu_baseline:
        return None
    from paper_2502_18437_b200 import scenes  # noqa: F401
    import backends
    if not backends.have_reference():
        return None
    if args.workload == "c4":
        rate, wall, n, k = time_reference_substeps(scenes.c4_slab(), args.cpu_seconds)
        return {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"C4 (1 core): {k} step_mls substeps with the contact hook on all {n} particles, "
                          f"{wall:.1f} s wall"}
    threads = cpu_threads() if args.workload == "c5" else 1
    pre = preroll_of(args) if args.workload != "m1" else 0
    rs = RefSet(cpu_specs_fn(args.workload)(threads), threads, pre)
    wall1 = rs.advance(1)
    frames = max(1, int(round(args.cpu_seconds / max(wall1, 1e-3))))
    wall = rs.advance(frames)
    rate, n, sub = rs.rate(frames, wall), rs.n, rs.sub
    rs.destroy()
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{threads} concurrent reference scenes ({args.workload}), {frames} frames x {sub} substeps, "
                      f"{n} particles, {wall:.1f} s wall, after {pre + 1} untimed frames"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.workload == "c4" and (world > 1 or args.dd):
        line, batch = run_ours_dd(args, rank, world, local_rank)
    else:
        line, batch = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1:
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
