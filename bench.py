#!/usr/bin/env python
"""Benchmark of the PSFS hot path (BASELINE.json metric: voxel-camera
projections/s and frames/s, 128^3 grid, 8 cameras 640x480, on 1/2/4/8 B200).

A step = one pass of the whole hot path (stage 1 likelihood terms + stage 2
projection / fusion / threshold / bit packing) over one batch of B distinct
synthetic frame sets (config C2, BASELINE.json configs[1]).  Multi-GPU is
frame-parallel (weak scaling): every rank reconstructs its own batch, no
collective on the data path; time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Prints one JSON line on rank 0.  `--impl reference` times the CPU oracle (this
tier's reference arm) on the host cores on the same workload.
"""
from __future__ import annotations

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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "voxel-camera projections/s and frames/s (128^3, 8 cams) at 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64, help="frames per step per GPU")
    ap.add_argument("--pool", type=int, default=64, help="distinct frame sets cycled")
    ap.add_argument("--overlap", type=int, default=0,
                    help="overlap stage 1 of group g+1 with stage 2 of group g; value = k_voxel "
                         "blocks/SM cap (0: none); -1: serial schedule")
    ap.add_argument("--fuse", type=int, default=16, help="frames fused per exact-path pass")
    ap.add_argument("--coarse", type=int, default=1, choices=[0, 1],
                    help="coarse passes for the bits-only headline (psfs_set_coarse; 0: exact path)")
    ap.add_argument("--coarse-frames", type=int, default=64, help="frames per coarse pass")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--ty", type=int, default=1)
    ap.add_argument("--kz", type=int, default=4)
    ap.add_argument("--stage1", type=int, default=6, choices=[0, 1, 2, 3, 4, 5, 6],
                    help="stage-1 kernel: 0 one pixel/thread, 1 TMA ring, 2 pipelined, "
                         "3 four pixels/thread, 4 warp-row loads, 5 cp.async ring, 6 persistent 4-pixel (default)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-zslab", action="store_true", help="skip the C4 z-slab section")
    ap.add_argument("--zslab-frames", type=int, default=64, help="frame sets per z-slab call (even)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondaries", action="store_true",
                    help="skip the full-output, NEXT-3 and other-config legs")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (1024^3, 32 cameras) leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: no clocks sampling / cpu baseline / e2e")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks

_NVML_SAMPLER = r"""
import sys, time
import pynvml as N
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
        N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
while True:
    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(f"{sm},{mx}," + ",".join("Active" if r & b else "Not Active" for b in bits), flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clock + throttle reasons sampled every ~2 ms during the timed region by a
    separate NVML process (no GIL contention with the launching thread; started
    and confirmed running before the timed region).  Falls back to nvidia-smi."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_SAMPLER, str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline()  # blocks until NVML is up
            if not first:
                raise RuntimeError("nvml sampler failed")
            self.lines.append(first.strip())
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
                return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Index of the next sample: call around the timed region."""
        self.marks.append(len(self.lines))

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampler unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        lines = self.lines
        if len(self.marks) >= 2 and self.marks[1] > self.marks[0]:
            lines = lines[self.marks[0]:self.marks[1] + 1]  # samples inside the timed region
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- helpers

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def make_workload(config, n_distinct, seed_offset=0):
    from synth.scene import make_frames, make_scene
    s = make_scene(config)
    frames = np.stack([make_frames(s, seed_offset + f) for f in range(n_distinct)])
    return s, frames


def gather_sectors(scene, F):
    """Algorithmic L1 wavefront count of one k_voxel launch.  The L1TEX data pipe
    serves about one 128-byte line per clock whatever number of its sectors a
    request touches (scripts/micro/gather.cu), so the unit is the line:
    * F <= 8 (k_voxel): for every warp (8 x 4 voxels in x, y at one z), camera
      and slice, the distinct pixels its 32 voxel centres project to (a pixel's
      F terms are one sector of one line);
    * F = 16 (k_voxel16, lane pairs): two gathers per warp and camera, over the
      16 even and the 16 odd voxels of the tile; a pixel's 64-byte record is two
      sectors of one line.
    Nearest pixel in double precision (the pinned FP32 pixel differs on ~0.1 %
    of voxel-cameras, irrelevant for a count).  Returns (wavefronts, useful bytes
    per wavefront)."""
    g = scene.grid
    i = np.arange(g.xlen)
    j = np.arange(g.ylen)
    X = g.origin[0] + g.spacing * (i + 0.5)
    Y = g.origin[1] + g.spacing * (j + 0.5)
    total = 0
    for c in range(scene.ncam):
        P = scene.P[c]
        for k in range(g.zlen):
            Z = g.origin[2] + g.spacing * (k + 0.5)
            x = P[0, 0] * X[None, :] + P[0, 1] * Y[:, None] + P[0, 2] * Z + P[0, 3]
            y = P[1, 0] * X[None, :] + P[1, 1] * Y[:, None] + P[1, 2] * Z + P[1, 3]
            w = P[2, 0] * X[None, :] + P[2, 1] * Y[:, None] + P[2, 2] * Z + P[2, 3]
            u = np.floor(x / w + 0.5).astype(np.int64)
            v = np.floor(y / w + 0.5).astype(np.int64)
            inview = (w > 0) & (u >= 0) & (u < scene.widths[c]) & (v >= 0) & (v < scene.heights[c])
            pix = np.where(inview, v * (scene.widths[c] + 1) + u, -1)   # -1: the zero pad
            # [ylen, xlen] -> warps of 4 rows x 8 columns
            t = pix.reshape(g.ylen // 4, 4, g.xlen // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
            groups = [t] if F <= 8 else [t[:, 0::2], t[:, 1::2]]
            for tt in groups:
                tt = np.sort(tt, axis=1)
                total += int((1 + (np.diff(tt, axis=1) != 0).sum(axis=1)).sum())
    return total, 4 * F


def cpu_baseline(scene, frames, seconds, nthreads):
    """The oracle as it stands, on the host cores, over whole frames until
    `seconds` of work (at least one frame)."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    n = 0
    while True:
        oracle.scene_reconstruct(scene, frames[n % len(frames)], nthreads=nthreads)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return n / el, n, el


def cpu_info():
    """CPU model and core counts of the host (lscpu; SURVEY.md 8(d) oracle timing)."""
    info = {"logical_cpus": os.cpu_count(), "affinity_cpus": host_cores()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        tpc = int(kv.get("Thread(s) per core", "1") or 1)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        sockets = int(kv.get("Socket(s)", "1") or 1)
        info["physical_cores"] = cps * sockets if cps else None
        info["threads_per_core"] = tpc
    except Exception as e:  # reported, not fatal
        info["lscpu_error"] = str(e)[:100]
    return info


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    rank, world, local = dist_setup(args)
    if rank != 0:
        return  # rank 0 alone runs and prints the CPU oracle arm
    from synth.scene import CONFIGS
    scene, frames = make_workload(args.config, min(args.pool, 4))
    nthreads = host_cores()
    import oracle
    oracle.build()
    for w in range(max(args.warmup, 0)):
        oracle.scene_reconstruct(scene, frames[w % len(frames)], nthreads=nthreads)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        oracle.scene_reconstruct(scene, frames[k % len(frames)], nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    fps = args.steps / total
    nvc = scene.grid.nvox * scene.ncam
    out = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "voxel_camera_projections_per_s": fps * nvc,
        "config": {"workload": f"{args.config}: {CONFIGS[args.config]['desc']}",
                   "frames_per_step": 1, "grid": [scene.grid.xlen] * 3, "cameras": scene.ncam},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": nthreads, "kind": "oracle",
                         "sample": f"1 full {args.config} frame per step (plain C oracle, "
                                   f"OpenMP over z-slices, {nthreads} threads)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- our arm

def device_us(fn, dev, reps=20):
    """Device time of one fn() call (µs): fn's launches captured once in a CUDA
    graph and replayed `reps` times between CUDA events, so Python / ctypes
    launch overhead (tens of µs per call) is not what is measured."""
    import torch
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        fn(s)  # warm-up outside the capture (lazy scratch allocations)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    g.replay()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / reps * 1e3


def pct(xs, q):
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


def step_stats(xs):
    return {"median": statistics.median(xs), "p10": pct(xs, 10), "p90": pct(xs, 90), "min": min(xs),
            "max": max(xs)}


def timed_calls(fn, steps, stream, flush=None):
    """Device time (ms) of each fn() call on `stream` between CUDA events, after
    a synchronize; the L2 is flushed before each call (outside the events) when a
    (write, read) buffer pair is given."""
    import torch
    out = []
    for k in range(steps):
        if flush is not None:
            flush[0].fill_(k)
            flush[1].sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(k)
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return out


def max_over_ranks(ms, world, dev):
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def roi_pixels(rec):
    """Stage-1 pixels of one frame set as the library plans them (per-row spans
    of the region of interest; psfs_roi_pixels)."""
    return rec.roi_pixels()


def full_output_leg(args, scene, frames_dev, B, pool, dev, stream, flush, world, hbm_peak, gather_peak,
                    hbm_src):
    """The north star's whole output (Eq 3 log-odds, and the bitmask): the
    same C2 step as the headline with log-odds requested, i.e. the exact int32
    path (16-frame passes of k_likelihood_x4p + k_voxel16, stage 1 of pass g+1
    overlapped with stage 2 of pass g), 8 MiB of float log-odds per frame.
    Rooflines: stage 1 against HBM (algorithmic bytes = ROI px x (24 B model +
    16 x (3 B image + 4 B term))), stage 2 against the binding one of the L2
    gather (the live probe of its access pattern) and the HBM store of the
    log-odds (nvox x 16 x 4 B per launch)."""
    import torch
    from paper_1311_6811_b200 import from_scene
    rec = from_scene(scene, device=dev.index)
    L, Bits = rec.alloc_outputs(B)

    tabs = [rec.frame_pointers(frames_dev[i0:i0 + B], B) for i0 in range(0, pool - B + 1, B)]

    def step(k):
        rec.reconstruct_batch(tabs[k % len(tabs)], B, logodds=L, bits=Bits, stream=stream)

    for k in range(3):
        step(k)
    torch.cuda.synchronize(dev)
    rec.set_profiling(True)
    rec.kernel_times(reset=True)
    ms = timed_calls(step, args.steps, stream, flush)
    kt = rec.kernel_times(reset=True)
    launches = rec.last_launch_count
    rec.set_profiling(False)
    total = max_over_ranks(sum(ms), world, dev)
    F = 16
    roi_px = roi_pixels(rec)
    l_ms, l_n = kt["k_likelihood"]
    v_ms, v_n = kt["k_voxel"]
    s1_bytes = roi_px * (24 + 7 * F)
    s1_t = (l_ms / max(l_n, 1)) / 1e3
    lines, wf = gather_sectors(scene, F)
    g_bytes = lines * wf
    st_bytes = scene.grid.nvox * F * 4
    v_t = (v_ms / max(v_n, 1)) / 1e3
    t_gather = g_bytes / (gather_peak * 1e9) if gather_peak else None
    t_store = st_bytes / (hbm_peak * 1e9)
    bound_t = max(t_gather or 0.0, t_store)
    out = {
        "value": world * B * args.steps / (total / 1e3), "unit": "frames/s",
        "ms_per_step": total / args.steps, "step_ms": step_stats(ms),
        "voxel_camera_projections_per_s": world * B * args.steps / (total / 1e3) * scene.grid.nvox * scene.ncam,
        "outputs": "float32 log-odds (8 MiB/frame) + occupancy bitmask (256 KiB/frame)",
        "path": "exact int32 terms, 16-frame passes, stage 1 of pass g+1 beside stage 2 of pass g",
        "launches_per_step": launches,
        "stage1": {"kernel": "k_likelihood_x4p<16>", "bound": "hbm", "unit": "GB/s",
                   "avg_launch_us": s1_t * 1e6, "algorithmic_bytes_per_launch": s1_bytes,
                   "achieved": s1_bytes / s1_t / 1e9, "peak": hbm_peak, "frac": s1_bytes / s1_t / 1e9 / hbm_peak,
                   "peak_source": hbm_src},
        "stage2": {"kernel": "k_voxel16 (log-odds + bits)", "bound": "l2_gather + hbm_store",
                   "avg_launch_us": v_t * 1e6,
                   "gather": {"algorithmic_bytes_per_launch": g_bytes, "lines_per_launch": lines,
                              "achieved_gbs": g_bytes / v_t / 1e9, "peak_gbs": gather_peak,
                              "frac": (g_bytes / v_t / 1e9 / gather_peak) if gather_peak else None},
                   "store": {"bytes_per_launch": st_bytes, "achieved_gbs": st_bytes / v_t / 1e9,
                             "peak_gbs": hbm_peak, "frac": st_bytes / v_t / 1e9 / hbm_peak},
                   "frac": bound_t / v_t,
                   "note": "frac = max(gather bytes / gather probe, store bytes / HBM) / launch time"},
        "kernel_share": {"stage1": l_ms / max(l_ms + v_ms, 1e-12), "stage2": v_ms / max(l_ms + v_ms, 1e-12)},
    }
    del rec, L, Bits
    return out


def variant_leg(args, config, dev, stream, flush, world, nframes=64, pool=16, channels=3, sampling=0,
                motion=False, note=""):
    """A secondary configuration through the same API, bits only: frames/s over
    `nframes`-frame calls cycling `pool` distinct frame sets (host rendering of
    large frames is slow), L2 flushed between calls."""
    import torch
    from paper_1311_6811_b200 import from_scene
    from synth.scene import CONFIGS, make_frames, make_scene
    s = make_scene(config, channels=channels)
    distinct = [torch.from_numpy(make_frames(s, f * 19 if motion else f, motion=motion)).to(dev)
                for f in range(pool)]
    rec = from_scene(s, device=dev.index, sampling=sampling)
    _, Bits = rec.alloc_outputs(nframes, logodds=False)
    lists = [rec.frame_pointers([distinct[(k * nframes + f) % pool] for f in range(nframes)], nframes)
             for k in range(4)]

    def step(k):
        rec.reconstruct_batch(lists[k % 4], nframes, bits=Bits, stream=stream)

    for k in range(2):
        step(k)
    torch.cuda.synchronize(dev)
    ms = timed_calls(step, max(3, min(args.steps, 10)), stream, flush)
    total = max_over_ranks(sum(ms), world, dev)
    fps = world * nframes * len(ms) / (total / 1e3)
    out = {"config": f"{config}: {CONFIGS[config]['desc']}" + (f"; {note}" if note else ""),
           "frames_per_call": nframes, "distinct_frame_sets": pool, "frames_per_s": fps,
           "ms_per_frame": 1e3 / fps * world, "voxel_camera_projections_per_s": fps * s.grid.nvox * s.ncam,
           "call_ms": step_stats(ms), "coarse_passes": rec.coarse_status()[0],
           "launches_per_call": rec.last_launch_count}
    del rec, Bits, distinct, lists
    torch.cuda.empty_cache()
    return out, s


def c1_graph_leg(dev):
    """C1 (32^3 x 4 cameras at 64x48, BASELINE.json configs[0]): launch-bound, so
    the call is captured once in a CUDA graph and replayed; device time per
    replay.  One frame per call (the latency view) and 64 frames per call
    (one coarse pass)."""
    import torch
    from paper_1311_6811_b200 import from_scene
    from synth.scene import make_frames, make_scene
    s = make_scene("C1")
    fr = torch.from_numpy(np.stack([make_frames(s, f) for f in range(64)])).to(dev)
    out = {"config": "C1: 32^3 grid, 4 cameras at 64x48 (launch-bound; CUDA-graph replays)"}
    for n in (1, 64):
        rec = from_scene(s, device=dev.index)
        _, Bits = rec.alloc_outputs(n, logodds=False)
        us = device_us(lambda st: rec.reconstruct_batch(fr[:n], n, bits=Bits, stream=st), dev, reps=50)
        out[f"frames_per_call_{n}"] = {"us_per_call": us, "frames_per_s": n / (us * 1e-6),
                                       "launches_per_call": rec.last_launch_count}
    return out


def c5_oracle_sample(scene, frame, nthreads):
    """The oracle on a voxel sample of C5 (C5 is reported as
    voxel-cam/s on the parity sample, extrapolated to s/frame): 2^14 random voxels,
    single-threaded and all-core."""
    import oracle
    rng = np.random.default_rng(5)
    vox = np.unique(rng.integers(0, scene.grid.nvox, 1 << 14))
    res = {}
    for name, th in (("single_thread", 1), ("all_cores", nthreads)):
        t0 = time.perf_counter()
        oracle.fuse_sample(scene.P, scene.widths, scene.heights, scene.grid, frame, scene.mu, scene.sigma,
                           vox, nthreads=th)
        el = time.perf_counter() - t0
        vc = vox.size * scene.ncam / el
        res[name] = {"threads": th, "voxel_cam_per_s": vc,
                     "extrapolated_s_per_frame": scene.grid.nvox * scene.ncam / vc}
    res["sample"] = f"{vox.size} random voxels of one C5 frame (oracle_fuse_sample: Eq 1-9 per voxel-camera)"
    return res


def zslab_bench(args, scene, frames_dev, rank, world, local, dev, stream, variants=None):
    """z-slab partition (BASELINE.json configs[3]): every rank
    owns zlen/N slices of the grid, computes stage 1 over its band of rows and
    stage 2 over its slab, and the full bitmask reaches every rank -- through
    the fused peer exchange (stage 2 stores into every rank's buffer) or an
    NCCL all-gather.  N = 1: one handle, nothing to exchange.  All ranks
    reconstruct the same frames (the same seeded scene)."""
    import torch
    import torch.distributed as dist
    from paper_1311_6811_b200.parallel import ZSlabReconstructor
    if variants is None:
        variants = ((("fused_peer", True), ("nccl_allgather", False), ("smoothed_nccl_halo", False))
                    if world > 1 else (("single_gpu", False), ("smoothed", False)))
    nf = int(frames_dev.shape[0])
    fr = frames_dev.contiguous()
    g = scene.grid
    out = {"frames_per_call": nf, "slices_per_rank": g.zlen // world, "world": world}
    for name, peer in variants:
        smooth = name.startswith("smoothed")
        z = ZSlabReconstructor(scene, rank=rank, world=world, device=local, peer=peer,
                               max_frames=nf)
        bits = None if peer else torch.zeros((nf, g.nwords), dtype=torch.int32, device=dev)
        # the smoothed variant materialises the int32 sums of its frames (512 MiB per
        # C4 frame at N = 1): 16 frames per call
        nfc = min(nf, 16) if smooth else nf
        frc = fr[:nfc]
        call = (lambda: z.reconstruct_smoothed(frc, nfc, bits=bits, stream=stream)) if smooth else \
            (lambda: z.reconstruct_batch(fr, nf, bits=bits, stream=stream))
        for _ in range(2):
            call()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        reps = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            call()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if peer:
            z.rec.peer_status(stream)
        t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item()) / reps / nfc
        out[name] = {"ms_per_frame": ms, "frames_per_s": 1e3 / ms, "frames_per_call": nfc,
                     "voxel_camera_projections_per_s": g.nvox * scene.ncam * 1e3 / ms}
        del z
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_setup(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1311_6811_b200 import build as pbuild
    if rank == 0:
        pbuild.build()
    if world > 1:
        dist.barrier()
    from paper_1311_6811_b200 import from_scene
    from synth.scene import CONFIGS

    B = args.batch
    pool = max(args.pool, B)
    # every rank reconstructs different frames (frame-parallel, weak scaling)
    scene, frames = make_workload(args.config, pool, seed_offset=rank * pool)
    rec = from_scene(scene, device=local)
    rec.set_max_fuse(args.fuse)
    rec.set_stage1_path(args.stage1)
    rec.set_voxel_tile(args.ty, args.kz)
    rec.set_overlap(args.overlap >= 0, max(args.overlap, 0))
    rec.set_coarse(args.coarse, args.coarse_frames)
    coarse = rec.coarse_status()[0]
    frames_dev = torch.from_numpy(frames).to(dev)
    L, Bits = rec.alloc_outputs(B, logodds=False, bits=True)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    flush_rd = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    nvox, ncam = scene.grid.nvox, scene.ncam
    per_cam = frames[0, 0].nbytes

    # the ABI's frame-pointer tables, built once: the timed region holds no
    # Python-side pointer arithmetic
    tables = {}
    gathered = []

    def table(k):
        i0 = (k * B) % pool
        if i0 not in tables:
            idx = [(i0 + b) % pool for b in range(B)]
            if idx == list(range(idx[0], idx[0] + B)):
                fr = frames_dev[idx[0]: idx[0] + B]
            else:
                fr = frames_dev[idx].contiguous()
                gathered.append(fr)
            tables[i0] = rec.frame_pointers(fr, B)
        return tables[i0]

    for k in range(args.warmup + args.steps + 2):
        table(k)

    def step(k):
        rec.reconstruct_batch(table(k), B, logodds=None, bits=Bits, stream=stream)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    sampler = ClockSampler(local) if not args.profile else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    rec.set_profiling(True)
    rec.kernel_times(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    if sampler:
        sampler.start()
    # two more untimed steps: the GPU was idle while the sampler started
    for k in range(2):
        flush.fill_(k)
        flush_sum = flush_rd.sum()
        step(k)
    torch.cuda.synchronize(dev)
    rec.kernel_times(reset=True)
    rec.coarse_status(reset=True)
    if sampler:
        sampler.mark()
    launches = 0
    for k in range(args.steps):
        # L2 flush outside the step events: write a buffer larger than L2, then
        # read another one so the L2 holds clean lines (no write-backs charged to
        # the next step)
        flush.fill_(k)
        flush_sum = flush_rd.sum()
        ev[k][0].record(stream)
        step(args.warmup + k)
        ev[k][1].record(stream)
        launches += rec.last_launch_count
    torch.cuda.synchronize(dev)
    if sampler:
        sampler.mark()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    kt = rec.kernel_times(reset=True)
    fixups = rec.coarse_status(reset=True)[1]
    rec.set_profiling(False)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    frames_total = world * B * args.steps
    fps = frames_total / (total_ms / 1e3)

    # ---- roofline of the dominant kernel (per-launch averages inside the timed region)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = ("of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks
               else "of fallback 6.65 TB/s (B200_PROFILING.md)")
    from paper_1311_6811_b200.psfs import probe_gather_bandwidth, probe_l1_bandwidth
    l1_peak = probe_l1_bandwidth() / 1e9 if not args.profile else None
    # k_voxel16's access pattern measured live: lane pairs on two-sector lines of a
    # 64 MB L2-resident table, non-allocating 256-bit loads (psfs_probe_gather_bandwidth)
    wide = coarse and args.coarse_frames > 32  # k_voxel_c8w: 64-byte records, lane pairs
    # the probe of the kernel's access pattern at MAXIMUM residency (8 blocks x 256
    # threads per SM requested; the probe's own register use decides how many are
    # resident): the pattern's rate, not the kernel's occupancy
    gather_probe = {}
    if not args.profile:
        for bps in (2, 3, 4, 8):
            gather_probe[bps] = probe_gather_bandwidth((64 if (wide or not coarse) else 32) << 20,
                                                       2 if (wide or not coarse) else 1, bps) / 1e9
    gather_peak = max(gather_probe.values()) if gather_probe else None
    gather_peak_16 = None
    if not args.profile:  # k_voxel16's pattern (full-output leg): lane pairs on 2-sector lines
        gather_peak_16 = max(probe_gather_bandwidth(64 << 20, 2, bps) / 1e9 for bps in (3, 8))
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(args.config + ("_coarse" if coarse else ""), {})
    except Exception:
        pass
    roi_px = roi_pixels(rec)  # stage-1 pixels (per-row spans of the ROI)
    F = args.coarse_frames if coarse else args.fuse
    l_ms, l_n = kt["k_likelihood"]
    v_ms, v_n = kt["k_voxel"]
    # stage 1 algorithmic bytes per launch (F frames fused): the model as
    # given (mu, sigma: 24 B/px) once, image 3 B/px and term 4 B/px per frame, over
    # the planned pixel rectangle
    # (coarse passes: 1-byte codes instead of 4-byte terms)
    s1_bytes = roi_px * (24 + (4 if coarse else 7) * F)
    s1_avg_s = (l_ms / max(l_n, 1)) / 1e3
    # stage 2: the gather is bound by the L1TEX data pipe, one line-wavefront per
    # clock per SM (ncu: l1tex__data_pipe_lsu_wavefronts); algorithmic wavefronts =
    # distinct pixels per warp-gather for this tiling (gather_sectors), each
    # carrying wf_bytes useful bytes (32: one sector, F = 8; 64: two sectors of
    # one line, F = 16); peak = 1 wavefront/clk/SM x wf_bytes
    v_avg_s = (v_ms / max(v_n, 1)) / 1e3
    # coarse: 32-B records one per lane (narrow), 64-B records by lane pairs (wide, as k_voxel16)
    sectors, wf_bytes = gather_sectors(scene, 16 if wide else (8 if coarse else F))
    s2_bytes = sectors * wf_bytes
    sm_clk = (clocks or {}).get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    import torch as _t
    nsm = _t.cuda.get_device_properties(dev).multi_processor_count
    l1_sector_peak = nsm * sm_clk * 1e6 * wf_bytes / 1e9
    s1_name = ("k_likelihood_c8p" if (scene.widths % 4 == 0).all() else "k_likelihood_c8") if coarse \
        else "k_likelihood"
    s2_name = (("k_voxel_c8w" if wide else "k_voxel_c8") + " + k_fixup_c8") if coarse else \
        ("k_voxel16" if F == 16 else "k_voxel")
    per_kernel = {
        "k_likelihood": {"name": s1_name,
            "bound": "hbm", "achieved": s1_bytes / s1_avg_s / 1e9, "peak": hbm_peak,
            "unit": "GB/s", "peak_source": hbm_src, "algorithmic_bytes_per_launch": s1_bytes,
            "avg_launch_us": s1_avg_s * 1e6, "traffic": traffic.get("k_likelihood")},
        "k_voxel": {"name": s2_name,
            "bound": "l1", "achieved": s2_bytes / v_avg_s / 1e9, "peak": l1_sector_peak,
            "unit": "GB/s",
            "peak_source": f"derived: {nsm} SMs x 1 L1TEX data-pipe wavefront/clk x {wf_bytes} "
                           f"useful bytes per wavefront x {sm_clk:.0f} MHz (median SM clock of "
                           "this run); DESIGN.md section 8",
            "algorithmic_bytes_per_launch": s2_bytes, "wavefronts_per_launch": sectors,
            "avg_launch_us": v_avg_s * 1e6,
            "voxel_cam_frames_per_s": nvox * ncam * F / v_avg_s, "traffic": traffic.get("k_voxel"),
            "l1_load_probe_gbs": l1_peak},
    }
    if coarse and gather_peak:
        kv = per_kernel["k_voxel"]
        kv["all_hit_l1_line_bound"] = {"peak": kv["peak"], "frac": kv["achieved"] / kv["peak"],
                                       "peak_source": kv["peak_source"]}
        # the L1TEX data pipe returns one wavefront per lane pair's 64-byte record
        # (per lane's 32-byte record, narrow) whatever the locality: ncu counts 16
        # per warp request (profiles/r02n_ncu_full.md), i.e. one per voxel-camera
        # -- the pipe's 1 wavefront/clk/SM sets a floor under the kernel's time
        wf_launch = nvox * ncam
        floor_us = wf_launch / (nsm * sm_clk * 1e6) * 1e6
        kv["l1_data_pipe_bound"] = {
            "wavefronts_per_launch": wf_launch, "floor_us": floor_us, "frac": floor_us / (v_avg_s * 1e6),
            "source": "one L1TEX data-pipe wavefront per voxel-camera record (ncu: 16 per warp request, "
                      "l1tex__data_pipe_lsu_wavefronts) at 1/clk/SM x the run's SM clock; DESIGN.md section 8"}
        kv.update({"bound": "l2_gather", "peak": gather_peak,
                   "fixups_per_step": fixups / max(args.steps, 1),
                   "probe_gbs_by_blocks_per_sm": gather_probe,
                   "peak_source": ("measured live: psfs_probe_gather_bandwidth(64 MB, 2 sectors/line) -- "
                                   "lane pairs read both 32-byte sectors of random 128-byte lines of an "
                                   "L2-resident table (k_voxel_c8w's pattern)"
                                   if wide else
                                   "measured live: psfs_probe_gather_bandwidth(32 MB, 1 sector/line) -- "
                                   "every lane reads one 32-byte sector of its own random 128-byte line "
                                   "of an L2-resident table (k_voxel_c8's pattern)")
                                  + ", non-allocating 256-bit loads, the best of 2/3/4/8 blocks x 256 "
                                    "threads per SM (maximum residency, not the kernel's 2); the timed "
                                    "launch includes k_fixup_c8; DESIGN.md section 8"})
    elif F == 16 and gather_peak:
        # the binding roofline of the 16-frame gather: the same access pattern's
        # measured rate from L2 (the all-hit L1 line rate kept beside it)
        kv = per_kernel["k_voxel"]
        kv["all_hit_l1_line_bound"] = {"peak": kv["peak"], "frac": kv["achieved"] / kv["peak"],
                                       "peak_source": kv["peak_source"]}
        kv.update({"bound": "l2_gather", "peak": gather_peak, "probe_gbs_by_blocks_per_sm": gather_probe,
                   "peak_source": "measured live: psfs_probe_gather_bandwidth(64 MB) -- lane pairs "
                                  "reading both 32-byte sectors of random 128-byte lines of an "
                                  "L2-resident table with k_voxel16's non-allocating 256-bit load "
                                  "and residency; DESIGN.md section 8"})
    for v in per_kernel.values():
        v["frac"] = v["achieved"] / v["peak"]
    dominant = "k_likelihood" if l_ms >= v_ms else "k_voxel"
    other = "k_voxel" if dominant == "k_likelihood" else "k_likelihood"
    share = {"k_likelihood": l_ms / max(l_ms + v_ms, 1e-12), "k_voxel": v_ms / max(l_ms + v_ms, 1e-12)}
    roofline = dict(kernel=per_kernel[dominant].pop("name"), **per_kernel[dominant])
    roofline["kernel_share"] = {per_kernel[k].get("name", k) if k != dominant else roofline["kernel"]: v
                                for k, v in share.items()}
    roofline["other_kernel"] = dict(kernel=per_kernel[other].pop("name"), **per_kernel[other])
    # SURVEY.md 8(d)'s issue / MUFU / gather bounds as the hardware counters read
    # them (ncu --set full, --cache-control none; profiles/r02_ncu_full.md):
    # per-pipe % of peak of each kernel of this path
    if traffic.get("pipes_pct"):
        roofline["ncu_pipes_pct_of_peak"] = dict(traffic["pipes_pct"], source=traffic.get("note"))

    # ---- end to end through the C ABI with HOST buffers (pinned), per step:
    # H2D of the batch's frames, both stages, D2H of the bitmask
    e2e = None
    if not args.no_e2e and not args.profile:
        hframes = torch.from_numpy(frames).pin_memory()
        hbits = torch.zeros((B, scene.grid.nwords), dtype=torch.int32).pin_memory()
        hb = [hframes[(k * B) % (pool - B + 1):(k * B) % (pool - B + 1) + B] for k in range(4)]
        for k in range(3):
            rec.reconstruct_host(hb[k % 4], B, None, hbits, stream=stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            rec.reconstruct_host(hb[k % 4], B, None, hbits, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * B * args.steps / (e_ms / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(B * 3 * roi_px),
               "d2h_bytes_per_step": int(B * scene.grid.nwords * 4),
               "ms_per_step": e_ms / args.steps,
               "how": "psfs_reconstruct_host: pinned host frames (the per-row spans of each image's "
                      "region of interest, read over PCIe by the zero-copy upload kernel k_h2d_rows on a "
                      "copy stream) -> device staging, both stages, bitmask -> pinned host (second "
                      "copy stream), double-buffered"}

    # ---- secondary: the two kernels in isolation (serial schedule), so their
    # roofline fractions are not diluted by the overlap of the headline schedule
    isolated = None
    if not args.profile and args.overlap >= 0:
        rec.set_overlap(False)
        rec.set_profiling(True)
        rec.kernel_times(reset=True)
        for k in range(min(args.steps, 10)):
            flush.fill_(k)
            flush_sum = flush_rd.sum()
            step(args.warmup + k)
        torch.cuda.synchronize(dev)
        kti = rec.kernel_times(reset=True)
        rec.set_profiling(False)
        rec.set_overlap(True, max(args.overlap, 0))
        isolated = {}
        for name, (ms_, n_) in kti.items():
            avg = (ms_ / max(n_, 1)) / 1e3
            ab = s1_bytes if name == "k_likelihood" else s2_bytes
            pk = per_kernel[name]["peak"]
            isolated[name] = {"avg_launch_us": avg * 1e6, "achieved": ab / avg / 1e9,
                              "frac": ab / avg / 1e9 / pk}
        roofline["isolated_serial"] = isolated

    # ---- secondary: bits-only early exit (psfs_set_carve), identical bitmask;
    # reported beside the headline, never as it
    carve = None
    if not args.profile:
        rec.set_carve(True)
        for k in range(args.warmup):
            step(k)
        torch.cuda.synchronize(dev)
        cms = 0.0
        for k in range(args.steps):
            flush.fill_(k)
            flush_sum = flush_rd.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(args.warmup + k)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            cms += e0.elapsed_time(e1)
        rec.set_carve(False)
        if world > 1:
            t = torch.tensor([cms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cms = float(t.item())
        carve = {"value": world * B * args.steps / (cms / 1e3), "unit": "frames/s",
                 "ms_per_step": cms / args.steps,
                 "note": "bits-only early exit (psfs_set_carve): a warp stops adding cameras once "
                         "its voxels are provably unoccupied; bitmask identical; not the headline"}

    # ---- secondary: the exact int32 path for the same bits-only step (coarse off);
    # the bitmask is identical (tests/test_gpu_coarse.py)
    exact = None
    if not args.profile and coarse:
        rec.set_coarse(0, args.coarse_frames)
        for k in range(2):
            step(k)
        torch.cuda.synchronize(dev)
        xms = 0.0
        for k in range(args.steps):
            flush.fill_(k)
            flush_sum = flush_rd.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(args.warmup + k)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            xms += e0.elapsed_time(e1)
        rec.set_coarse(args.coarse, args.coarse_frames)
        if world > 1:
            t = torch.tensor([xms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            xms = float(t.item())
        exact = {"value": world * B * args.steps / (xms / 1e3), "unit": "frames/s",
                 "ms_per_step": xms / args.steps,
                 "note": f"the exact int32 path (k_likelihood + k_voxel16, {args.fuse}-frame passes) "
                         "for the same bits-only step; identical bitmask; not the headline"}

    # ---- secondary (N > 1 only): z-slab partition of the same grid across the
    # ranks, 16 frames per call, with the bitmask exchange fused into stage 2
    # (peer stores + device barriers) and, for comparison, the NCCL all-gather
    zslab = None
    if not args.profile and not args.no_zslab:
        try:
            from synth.scene import make_frames, make_scene
            zs = make_scene("C4")
            two = torch.from_numpy(np.stack([make_frames(zs, f) for f in range(2)])).to(dev)
            zfr = two.repeat(args.zslab_frames // 2, 1, 1, 1, 1)  # 2 distinct (host rendering is slow)
            del two
            zslab = zslab_bench(args, zs, zfr, rank, world, local, dev, stream)
            zslab["config"] = ("C4: 512^3 grid, 16 cameras at 1920x1080, z-slab partition over "
                               f"{world} GPU(s), {args.zslab_frames} frame sets per call (2 distinct, repeated)")
            del zfr
        except Exception as e:  # reported, never fatal for the headline
            zslab = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    # ---- secondary: NEXT-2 surface extraction (psfs_surface) of one frame's bitmask
    surface = None
    if not args.profile:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        idx = torch.empty(nvox, dtype=torch.int64, device=dev)
        sbits = torch.empty_like(Bits[0])
        us = device_us(lambda st: rec.surface(Bits[0], surface_bits=sbits, indices=idx, count=cnt,
                                              stream=st), dev)
        surface = {"us_per_frame": us, "surface_voxels": int(cnt.item()),
                   "occupied_voxels": int(torch.bitwise_and(
                       Bits[0].view(-1, 1) >> torch.arange(32, device=dev, dtype=torch.int32), 1).sum().item()),
                   "note": "NEXT-2 inner-voxel removal (P:301): bit-parallel 6-neighbour test + ordered "
                           "compaction, 3 launches (device time, CUDA-graph replay), not part of the "
                           "headline step"}

    # ---- secondary: one frame set per call (no batching: F = 1, latency view of
    # the same C2 workload), L2 flushed before every call (outside the events)
    single = None
    if not args.profile:
        _, B1 = rec.alloc_outputs(1, logodds=False)
        for k in range(3):
            rec.reconstruct(frames_dev[k], bits=B1, stream=stream)
        torch.cuda.synchronize(dev)
        tms = []
        for k in range(args.steps):
            flush.fill_(k)
            flush_sum = flush_rd.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rec.reconstruct(frames_dev[k % pool], bits=B1, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            tms.append(e0.elapsed_time(e1))
        single = {"ms_per_frame": float(np.median(tms)), "frames_per_s": 1e3 / float(np.median(tms)),
                  "note": "latency view: psfs_reconstruct of one frame set per call (no fusion), "
                          "median over calls, L2 flushed before each"}

    # ---- secondary: NEXT-4 voxel colour (psfs_color) of one frame's surface voxels,
    # chained on the device after psfs_surface (count never read on the host)
    color = None
    if not args.profile:
        _, Bc = rec.alloc_outputs(1, logodds=False)
        rec.reconstruct(frames_dev[0], bits=Bc, stream=stream)
        ccnt = torch.zeros(1, dtype=torch.int64, device=dev)
        cidx = torch.empty(nvox, dtype=torch.int64, device=dev)
        rec.surface(Bc[0], indices=cidx, count=ccnt, stream=stream)
        crgb = torch.empty((nvox, 3), dtype=torch.float32, device=dev)
        cnv = torch.empty(nvox, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        us = device_us(lambda st: rec.color(frames_dev[0], cidx, count=ccnt, rgb=crgb, nviews=cnv,
                                            stream=st), dev)
        nsurf = int(ccnt.item())
        color = {"us_per_frame": us, "surface_voxels": nsurf,
                 "coloured_voxels": int((cnv[:nsurf] > 0).sum().item()),
                 "note": "NEXT-4 voxel colour (P:222, P:273-275): mean RGB over in-view cameras "
                         "with SLM > 1/2 at each surface voxel, 1 launch (device time, CUDA-graph "
                         "replay), not part of the headline step"}

    # ---- secondary: NEXT-3 background training (psfs_train_background) of one
    # camera from 32 frames, outputs only (the bench's model stays installed)
    train = None
    if not args.profile:
        tf = frames_dev[:32, 0].contiguous()
        us = device_us(lambda st: rec.train_background(0, tf, install=False, stream=st), dev)
        tbytes = tf.numel() + 2 * 4 * tf[0].numel()
        train = {"us_per_camera": us, "frames": int(tf.shape[0]),
                 "achieved_gbs": tbytes / (us * 1e-6) / 1e9,
                 "note": "NEXT-3 background training (S:99-107): per-pixel mean and population "
                         "std over 32 frames of one 640x480 camera, 1 launch (device time, "
                         "CUDA-graph replay); bytes = frames read + mean/sigma written"}

    # ---- secondary: NEXT-1 merged filtering + thresholding (psfs_smooth_threshold)
    smooth = None
    if not args.profile:
        Lf, Bf = rec.alloc_outputs(1)
        rec.reconstruct(frames_dev[0], logodds=Lf, bits=Bf, stream=stream)
        smv = torch.empty_like(Lf[0])
        smb = torch.empty_like(Bf[0])
        torch.cuda.synchronize(dev)
        us = device_us(lambda st: rec.smooth_threshold(Lf[0], smoothed=smv, bits=smb, stream=st), dev)
        smooth = {"us_per_frame": us,
                  "note": "NEXT-1 posterior 3x3x3 box filter + threshold (P:111, P:300), "
                          "2 launches (device time, CUDA-graph replay), not part of the headline step"}

    # ---- secondary: the full output (log-odds + bits), the same C2 step
    full_output = None
    flush_pair = (flush, flush_rd)
    if not args.profile and not args.no_secondaries:
        try:
            full_output = full_output_leg(args, scene, frames_dev, B, pool, dev, stream, flush_pair, world,
                                          hbm_peak, gather_peak_16, hbm_src)
        except Exception as e:
            full_output = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    # ---- secondary: NEXT-1 merged with reconstruction (exact sums -> k_box_sums),
    # the same 64 C2 frame sets per call, smoothed bitmask out
    smooth_merged = None
    if not args.profile and not args.no_secondaries:
        try:
            rs = from_scene(scene, device=local)
            _, Bs = rs.alloc_outputs(B, logodds=False)
            tab = rs.frame_pointers(frames_dev[:B], B)
            rs.reconstruct_smoothed(tab, B, bits=Bs, stream=stream)
            torch.cuda.synchronize(dev)
            ms = timed_calls(lambda k: rs.reconstruct_smoothed(tab, B, bits=Bs, stream=stream),
                             max(3, min(args.steps, 10)), stream, flush_pair)
            tot = max_over_ranks(sum(ms), world, dev)
            smooth_merged = {"frames_per_s": world * B * len(ms) / (tot / 1e3), "call_ms": step_stats(ms),
                             "launches_per_call": rs.last_launch_count,
                             "note": "NEXT-1 merged (P:269-271): psfs_reconstruct_smoothed, exact int32 sums "
                                     "(16-frame passes) then k_box_sums (posterior on the fly, 3x3x3 box, "
                                     "threshold); no float log-odds / posterior volume; smoothed bitmask out"}
            del rs, Bs
        except Exception as e:
            smooth_merged = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    # ---- secondary configurations (BASELINE.json configs) and NEXT-3 variants,
    # bits only, through the same API; reported beside the headline, never as it
    configs_out = {}
    c5_scene = None
    if not args.profile and not args.no_secondaries:
        legs = [
            ("C2_grayscale", dict(config="C2", channels=1, note="NEXT-3 grayscale input (U = 256^-1), exact path")),
            ("C2_bilinear", dict(config="C2", sampling=1, note="NEXT-3 bilinear SLM sampling, 8-frame passes")),
            ("C3_sequence", dict(config="C3", nframes=300, pool=16, motion=True,
                                 note="300-frame walking / arm-waving sequence in one call (16 distinct "
                                      "frame sets of the sequence, every 19th frame, cycled)")),
        ]
        legs.append(("C2_overlap128", dict(config="C2", nframes=128, pool=64,
                                           note="128 frames per call: two 64-frame coarse passes, stage 1 of "
                                                "the second beside stage 2 of the first (the handle's "
                                                "overlapped schedule); per-kernel times overlap, so the "
                                                "headline keeps the one-pass step")))
        if not args.no_c5:
            legs.append(("C5", dict(config="C5", nframes=64, pool=1,
                                    note="one 64-frame coarse pass (1 distinct frame set repeated: host "
                                         "rendering of 32 x 1920x1080 views is slow)")))
        for name, kw in legs:
            try:
                configs_out[name], sc = variant_leg(args, dev=dev, stream=stream, flush=flush_pair,
                                                    world=world, **kw)
                if name == "C5":
                    c5_scene = sc
            except Exception as e:
                configs_out[name] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
        try:
            configs_out["C1"] = c1_graph_leg(dev)
        except Exception as e:
            configs_out["C1"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        nthreads = host_cores()
        v, n, el = cpu_baseline(scene, frames, args.cpu_seconds, nthreads)
        v1, n1, el1 = cpu_baseline(scene, frames, args.cpu_seconds / 2, 1)
        cpu = {"value": v, "unit": "frames/s", "cores": nthreads, "kind": "oracle",
               "sample": f"{n} full {args.config} frames ({el:.1f} s of work), plain C oracle "
                         f"(double; OpenMP over z-slices, {nthreads} threads)",
               "single_thread": {"value": v1, "unit": "frames/s", "cores": 1,
                                 "sample": f"{n1} full {args.config} frames ({el1:.1f} s)"},
               "host": cpu_info(),
               "gpu_over_oracle": {"all_cores": fps / v, "single_thread": fps / v1,
                                   "paper_context": "HD 6870 vs one i7-860 core: 399x (P:376), whole pipeline "
                                                    "incl. APF"}}
        if c5_scene is not None:
            try:
                from synth.scene import make_frames
                cpu["C5_sample"] = c5_oracle_sample(c5_scene, make_frames(c5_scene, 0), nthreads)
            except Exception as e:
                cpu["C5_sample"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("f32+u8+i32 (coarse codes; f64 exact fix-up)" if coarse else "f64+f32+i32"),
            "data": "synthetic",
            "voxel_camera_projections_per_s": fps * nvox * ncam,
            "config": {"workload": f"{args.config}: {CONFIGS[args.config]['desc']}",
                       "batching": (f"each frame set (one frame of every camera) reconstructed independently; "
                                    f"{B} distinct frame sets per step per GPU, {(B + F - 1) // F} pass(es) of "
                                    f"{F} frames"),
                       "frames_per_step_per_gpu": B, "fused_frames_per_pass": F,
                       "path": ("coarse passes (8-bit bracketing codes, exact fix-up; bitmask "
                                "identical to the exact path)" if coarse else "exact int32 terms"),
                       "grid": [scene.grid.xlen, scene.grid.ylen, scene.grid.zlen],
                       "cameras": ncam, "image": [int(scene.widths[0]), int(scene.heights[0])],
                       "distinct_frame_sets": pool, "parallelism": f"frame-parallel x{world}",
                       "schedule": ("stage 1 of group g+1 overlapped with stage 2 of group g"
                                    + (f" (k_voxel capped at {args.overlap} blocks/SM)" if args.overlap > 0 else "")
                                    if args.overlap >= 0 else "serial"),
                       "l2": "flushed between steps (256 MiB write + 256 MiB read, outside the step events)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "carve": carve, "exact_path": exact,
            "single_frame": single, "surface": surface, "color": color, "smooth": smooth,
            "train": train, "zslab": zslab, "full_output": full_output, "smooth_merged": smooth_merged,
            "configs": configs_out,
            "gpu_launches": launches, "clocks": clocks,
            "step_ms": dict(step_stats(step_ms), all=[round(x, 4) for x in step_ms]),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
