#!/usr/bin/env python
"""Benchmark of the fused kernel-map decode + filter + fusion (arXiv 2202.05977).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kmd|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

A step is one pass of the whole hot path (load,
shared exp, normalise, filter, fusion weights, fuse, store) over one 1920x1080
frame with the paper's kernel-size set {3,5,7,9,11,13} (BASELINE.json
configs[2], the configuration the metric is quoted on).  Multi-GPU runs are
frame-parallel ("weak" scaling, configs[4]'s sharding): every rank processes
its own frame each step, no collective on the data path.

Inputs are synthetic (paper_2202_05977_b200/inputs.py), resident in HBM, and
rotate over 4 distinct frames (597 MB > 126 MB L2), so no step reads another
step's inputs from L2.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

PAPER_SIZES = [3, 5, 7, 9, 11, 13]
METRIC = "1080p Mpix/s (decode+filter+fusion)"
UNIT = "Mpix/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["kmd", "reference"], default="kmd")
    ap.add_argument("--mode", choices=["frame", "band", "mr", "bwd", "temporal", "sweep", "batch"], default="frame",
                    help="frame: one frame per rank per step (weak scaling, default); band: ONE "
                         "frame split into row bands across ranks with an NCCL halo exchange "
                         "every step (strong scaling, BASELINE.json configs[3], default 4K)")
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--sizes", type=str, default=",".join(map(str, PAPER_SIZES)))
    ap.add_argument("--rotate", type=int, default=4, help="distinct resident frames per rank")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--batch", type=int, default=256,
                    help="--mode batch: frames in the whole batch, sharded over the ranks (BASELINE.json configs[4])")
    ap.add_argument("--albedo", action="store_true",
                    help="NEXT row 1: fuse the albedo remodulation epilogue (out = Rhat * albedo)")
    ap.add_argument("--bf16", action="store_true",
                    help="NEXT row 4 alternative: bf16 importance maps and logits (kmd_decode_filter_fuse_bf16)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU seconds for the oracle sample")
    return ap.parse_args()


# ----------------------------------------------------------------- distributed
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        reasons = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(s)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def lib_sources_hash():
    import hashlib
    from paper_2202_05977_b200 import _build
    h = hashlib.sha256()
    for p in sorted(_build._deps()):
        h.update(open(p, "rb").read())
    return h.hexdigest()[:16]


def recorded_traffic(workload: str):
    """dram bytes per launch from the committed ncu --set full capture
    (profiles/traffic.json), if it was taken on the current kernel sources."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        e = d.get(workload)
        if e and e.get("lib_sha") == lib_sources_hash():
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


# ----------------------------------------------------------------- oracle legs
def cpu_model() -> str:
    """The host CPU's model name (lscpu / /proc/cpuinfo), for cpu_baseline."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rows_time(inp_cpu, sizes, rows, threads=0):
    import oracle
    t0 = time.perf_counter()
    ref = oracle.decode_filter_fuse(inp_cpu[0], inp_cpu[1], inp_cpu[2], sizes, rows=rows,
                                    threads=threads)
    return time.perf_counter() - t0, ref


def calibrate_rows(inp_cpu, sizes, H, seconds):
    t1, _ = oracle_rows_time(inp_cpu, sizes, (H // 2, H // 2 + 2))
    per_row = t1 / 2
    return max(1, min(H, int(seconds / max(per_row, 1e-9)))), per_row


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2202_05977_b200 import inputs as gen
    sizes = [int(s) for s in args.sizes.split(",")]
    H, W, M = args.height, args.width, len(sizes)
    inp = gen.make_inputs(1, H, W, M)
    inp_cpu = (inp.radiance.numpy(), inp.importance.numpy(),
               None if inp.blend is None else inp.blend.numpy())
    budget = 150.0
    total = args.steps + args.warmup
    rows, per_row = calibrate_rows(inp_cpu, sizes, H, budget / max(total, 1))
    for s in range(args.warmup):
        y0 = (s * rows) % max(1, H - rows + 1)
        oracle_rows_time(inp_cpu, sizes, (y0, y0 + rows))
    el = 0.0
    for s in range(args.steps):
        y0 = ((s + args.warmup) * rows) % max(1, H - rows + 1)
        dt, _ = oracle_rows_time(inp_cpu, sizes, (y0, y0 + rows))
        el += dt
    px = rows * W * args.steps
    value = px / el / 1e6
    cores = oracle.max_threads()
    sample = (f"each step: {rows} rows x {W} px of a {W}x{H} M={M} frame "
              f"({rows * W} px, fp64 oracle, OpenMP {cores} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{W}x{H} frame, sizes {sizes}, fusion (configs[2])",
                   "global_batch": 1, "parallelism": "host OpenMP"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- kmd leg
def run_kmd(args, rank, world, local):
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd

    dev = torch.device("cuda", local)
    sizes = [int(s) for s in args.sizes.split(",")]
    H, W, M = args.height, args.width, len(sizes)
    F = max(1, args.rotate)
    K, Wm = args.steps, args.warmup
    assert Wm >= 3, "timing rules: at least 3 warm-up steps"
    kmd.lib()
    # resident inputs: F distinct frames per rank (frame ids rank*F .. rank*F+F-1)
    inp = gen.make_inputs(F, H, W, M, frame_offset=rank * F, device=dev)
    if args.bf16:
        # the network's output in bf16; the oracle below sees the same values widened
        assert not args.albedo, "--bf16 has no albedo epilogue"
        inp = gen.FrameInputs(inp.radiance, inp.importance.to(torch.bfloat16),
                              None if inp.blend is None else inp.blend.to(torch.bfloat16))
    outs = torch.empty((F, 3, H, W), device=dev)
    alb = gen.make_albedo(F, H, W, frame_offset=rank * F, device=dev) if args.albedo else None
    views = [(inp.radiance[f:f + 1], inp.importance[f:f + 1],
              None if inp.blend is None else inp.blend[f:f + 1], outs[f:f + 1],
              None if alb is None else alb[f:f + 1])
             for f in range(F)]
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)

    def step(s, strm=None):
        r, i, b, o, a = views[s % F]
        kmd.decode_filter_fuse(r, i, b, sizes, out=o, stream=strm, albedo=a)

    for s in range(Wm):
        step(s, stream)
    torch.cuda.synchronize(dev)

    # ---- CUDA graphs: G launches per graph (frames rotate), remainder graph --
    # Launching through graphs keeps the GPU back-to-back busy; from Python the
    # per-launch host cost would otherwise exceed the ~25-100 us kernel.
    G = 2 * F
    reps, rem = divmod(K, G)

    def capture(n):
        if n == 0:
            return None
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for j in range(n):
                step(j)
        return g

    g_main, g_rem = capture(G), capture(rem)
    torch.cuda.synchronize(dev)
    for _ in range(max(1, Wm // G)):
        g_main.replay() if g_main else g_rem.replay()
    torch.cuda.synchronize(dev)

    # ---- timed region: exactly K launches, events around every graph replay --
    n_rep = reps + (1 if rem else 0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n_rep)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for r in range(n_rep):
            ev[r][0].record(stream)
            (g_main if r < reps else g_rem).replay()
            ev[r][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    el_ms = t_start.elapsed_time(t_end)
    per_launch = sorted(a.elapsed_time(b) / (G if r < reps else rem) for r, (a, b) in enumerate(ev))
    kern_avg_ms = sum(a.elapsed_time(b) for a, b in ev) / K
    kern_ms = per_launch
    el_ms_max = max_over_ranks(el_ms, world)

    px_per_step = H * W * world
    value = px_per_step * K / (el_ms_max / 1e3) / 1e6
    bytes_launch = kmd.algorithmic_bytes(1, H, W, sizes, inp.blend is not None) + \
        (12 * H * W if args.albedo else 0)
    if args.bf16:  # importance and logits at 2 B instead of 4 (48 B/px at M = 6)
        bytes_launch -= 2 * H * W * (M + (M if inp.blend is not None else 0))
    achieved = bytes_launch / (kern_avg_ms / 1e3) / 1e9
    peak, peak_src = measured_peak_hbm()
    cfg_name = {(1920, 1080): "configs[2]", (1280, 720): "configs[1]"}.get((W, H), "custom size")
    workload = f"{W}x{H} frame, sizes {sizes}, fusion (BASELINE.json {cfg_name})" + \
        (" + albedo remodulation (NEXT row 1)" if args.albedo else "") + \
        (", bf16 importance/logits (NEXT row 4 alternative)" if args.bf16 else "")

    # ---- e2e: through the C ABI with pinned HOST buffers ---------------------
    e2e = None
    if args.e2e_steps > 0:  # bf16 importance / logits: kmd_decode_filter_fuse_host_bf16
        hr = inp.radiance[:1].cpu().pin_memory()
        hi = inp.importance[:1].cpu().pin_memory()
        hb = None if inp.blend is None else inp.blend[:1].cpu().pin_memory()
        ho = torch.empty((1, 3, H, W)).pin_memory()
        ws = torch.empty(kmd.host_workspace_bytes(1, H, W, sizes), dtype=torch.uint8, device=dev)
        for _ in range(3):
            kmd.decode_filter_fuse_host(hr, hi, hb, sizes, ho, ws, stream=stream)
        torch.cuda.synchronize(dev)
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            kmd.decode_filter_fuse_host(hr, hi, hb, sizes, ho, ws, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(a.elapsed_time(b), world)
        h2d = sum(t.numel() * t.element_size() for t in (hr, hi, hb) if t is not None)
        e2e = {"value": px_per_step * args.e2e_steps / (e2e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": ho.numel() * 4,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "path": ("kmd_decode_filter_fuse_host_bf16" if args.bf16 else "kmd_decode_filter_fuse_host") +
                       " (pinned host -> HBM -> kernel -> host)"}

    # ---- CPU oracle baseline + sampled parity (rank 0, N=1 only) -------------
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import numpy as np
        import oracle
        inp_cpu = (inp.radiance[:1].cpu().numpy(), inp.importance[:1].float().cpu().numpy(),
                   None if inp.blend is None else inp.blend[:1].float().cpu().numpy())
        rows, _ = calibrate_rows(inp_cpu, sizes, H, args.cpu_seconds)
        y0 = max(0, (H - rows) // 2)
        dt, ref = oracle_rows_time(inp_cpu, sizes, (y0, y0 + rows))
        # and one thread on a few rows (the per-core figure)
        r1 = max(1, min(8, rows))
        dt1, _ = oracle_rows_time(inp_cpu, sizes, (y0, y0 + r1), threads=1)
        cpu = {"value": rows * W / dt / 1e6, "unit": UNIT, "cores": oracle.max_threads(),
               "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"rows {y0}..{y0 + rows} ({rows * W} px) of frame 0 of the {W}x{H} "
                         f"M={M} workload, fp64 oracle, {dt:.1f} s",
               "value_1thread": r1 * W / dt1 / 1e6,
               "sample_1thread": f"rows {y0}..{y0 + r1} ({r1 * W} px), one thread, {dt1:.2f} s"}
        r0, i0, b0, o0, a0 = views[0]
        kmd.decode_filter_fuse(r0, i0, b0, sizes, out=o0, stream=stream)
        torch.cuda.synchronize(dev)
        got = outs[0:1, :, y0:y0 + rows].cpu().numpy().astype(np.float64)
        rel = np.abs(got - ref) / np.where(ref == 0, 1.0, np.abs(ref))
        parity = {"max_rel_err": float(rel.max()), "pixels": int(rows * W), "tol": 1e-5,
                  "rows": [y0, y0 + rows]}

    if rank != 0:
        return
    # BASELINE.md holds the paper's number for one workload only: 1280x720,
    # M = 6 {3..13} with fusion, 1.10 ms per frame (RTX 2080 Ti)
    paper_720p = (W, H) == (1280, 720) and sizes == PAPER_SIZES and not args.albedo
    vs = value / (1280 * 720 / 1.10e-3 / 1e6) if paper_720p else None
    metric = METRIC if (W, H) == (1920, 1080) else f"{W}x{H} Mpix/s (decode+filter+fusion)"
    line = {
        "metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": Wm, "ms_per_step": el_ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": vs, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload, "global_batch": world, "frames_per_rank_per_step": 1,
                   "height": H, "width": W, "sizes": sizes,
                   "parallelism": f"frame-parallel x{world} (no data-path collective)",
                   "l2": f"inputs rotate over {F} resident frames per rank "
                         f"({F * bytes_launch / 1e6:.0f} MB > 126 MB L2)"},
        "ms_per_frame": el_ms_max / K,
        "kernel_ms": {"avg": kern_avg_ms, "p10": kern_ms[len(kern_ms) // 10],
                      "p50": kern_ms[len(kern_ms) // 2], "p90": kern_ms[(9 * len(kern_ms)) // 10],
                      "how": f"CUDA events around each replay of a {G}-launch CUDA graph, per launch"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": recorded_traffic(workload),
                     "algorithmic_bytes_per_launch": bytes_launch, "peak_source": peak_src,
                     "kernel": f"fused decode+filter+fuse (libkmd, {kmd.last_kernel()})"},
        "gpu_launches": K * kmd.launches_per_call(),
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "paper_context": "RTX 2080 Ti, 1280x720, M=6: 1.10 ms reconstruction (PAPER.md:472)",
    }
    print(json.dumps(line), flush=True)


def run_band(args, rank, world, local):
    """configs[3]: one 3840x2160 frame per step, split into `world` row bands
    (strong scaling).  Each step is libkmd's kmd_band_step: the r_max halo rows
    of the 3 radiance and M importance planes go to / come from the
    neighbouring ranks in ONE grouped NCCL call on a side stream (libkmd's own
    communicator, its unique id broadcast over torch.distributed), while the
    band's interior tile rows run on the compute stream; the seam tile rows
    follow the exchange.  At N = 1 it is the whole 4K frame on one GPU."""
    from paper_2202_05977_b200 import bands as B
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    sizes = [int(s) for s in args.sizes.split(",")]
    H = args.height if args.height != 1080 else 2160
    W = args.width if args.width != 1920 else 3840
    M = len(sizes)
    F = 2
    K, Wm = args.steps, args.warmup
    assert Wm >= 3, "timing rules: at least 3 warm-up steps"
    kmd.lib()
    band = B.split_rows(H, world, sizes)[rank]
    r = B.rmax_of(sizes)
    up = rank - 1 if band.halo_top > 0 else -1
    down = rank + 1 if band.halo_bot > 0 else -1
    full = gen.make_inputs(F, H, W, M, device=dev)      # identical on every rank (same seeds)
    rad = [B.slice_band(full.radiance[f:f + 1], band) for f in range(F)]
    imp = [B.slice_band(full.importance[f:f + 1], band) for f in range(F)]
    bl = [full.blend[f:f + 1, :, band.y0:band.y0 + band.rows].contiguous() for f in range(F)]
    out = torch.empty((1, 3, band.rows, W), device=dev)
    del full
    comm = B.make_comm() if world > 1 else None
    side = torch.cuda.Stream(dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)

    def step(s):
        f = s % F
        kmd.band_step(comm, rad[f], imp[f], bl[f], sizes, out, y0=band.y0, band_rows=band.rows, halo=r,
                      peer_up=up, peer_down=down, H_global=H, stream=stream, comm_stream=side)

    def kernel_only(s):
        f = s % F
        kmd.decode_filter_fuse_band_part(rad[f], imp[f], bl[f], sizes, kmd.BAND_ALL, y0=band.y0,
                                         band_rows=band.rows, halo_top=band.halo_top,
                                         halo_bot=band.halo_bot, H_global=H, out=out, stream=stream)

    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        a.record(stream)
        for s in range(K):
            step(s)
        b.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    el = max_over_ranks(a.elapsed_time(b), world)
    # the band kernel alone (no exchange), for the roofline: same buffers
    Kk = min(K, 200)
    for s in range(3):
        kernel_only(s)
    torch.cuda.synchronize(dev)
    a.record(stream)
    for s in range(Kk):
        kernel_only(s)
    b.record(stream)
    torch.cuda.synchronize(dev)
    kern_ms = a.elapsed_time(b) / Kk
    kind = kmd.last_kernel()
    if comm is not None:
        comm.destroy()
    if rank != 0:
        return
    value = H * W * K / (el / 1e3) / 1e6
    halo_bytes = r * W * (3 + M) * 4 if world > 1 else 0
    algo = kmd.algorithmic_bytes(1, band.rows, W, sizes, True)
    peak, peak_src = measured_peak_hbm()
    achieved = algo / (kern_ms / 1e3) / 1e9
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s (decode+filter+fusion, row bands)", "value": value, "unit": UNIT,
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": el / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{W}x{H} frame split into {world} row bands + NCCL halo exchange "
                               f"(BASELINE.json configs[3])", "sizes": sizes,
                   "band_rows": band.rows, "halo_bytes_per_seam_per_direction": halo_bytes,
                   "parallelism": f"row bands x{world}",
                   "l2": f"inputs rotate over {F} frames ({F * algo * world / 1e6:.0f} MB > 126 MB L2)"},
        "kernel_ms": {"avg": kern_ms, "how": f"CUDA events around {Kk} band launches without the exchange "
                                             f"(rank 0's band, {band.rows} rows)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "algorithmic_bytes_per_launch": algo,
                     "peak_source": peak_src, "kernel": f"band kernel (libkmd, {kind})"},
        "clocks": clk.summary(), "gpu_launches": K * (1 if world == 1 else 2),
        "timing": "CUDA events around K steps (kmd_band_step: NCCL exchange on a side stream overlapped "
                  "with the interior, then the seams), max over ranks"}),
        flush=True)


def run_mr(args, rank, world, local):
    """NEXT row 2: "Ours MR" (3 levels x sizes {3,5} + Eq. 7) on a 1080p frame
    per rank per step (weak scaling), CUDA-graph launched like the main mode."""
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    H, W = args.height, args.width
    sizes = [list(s) for s in gen.MR_SIZES]
    K, Wm, F = args.steps, args.warmup, 2
    frames = [gen.make_mr_inputs(1, H, W, seed=gen.BASE_SEED + 11 + 97 * (rank * F + f), device=dev)
              for f in range(F)]
    outs = [torch.empty((1, 3, H, W), device=dev) for _ in range(F)]
    ws = torch.empty(kmd.mr_workspace_bytes(1, H, W, sizes), dtype=torch.uint8, device=dev)

    def step(s):
        mi = frames[s % F]
        kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, sizes,
                                  out=outs[s % F], workspace=ws)

    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(2 * F):
            step(j)
    reps = max(1, K // (2 * F))
    g.replay()
    torch.cuda.synchronize(dev)
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize(dev)
    barrier(world)
    steps = reps * 2 * F
    el = max_over_ranks(a.elapsed_time(b), world)
    if rank != 0:
        return
    # inputs + output, each read/written once: radiance 12, level-l maps
    # (2 importance + 2 logits) 16 / 4^l, alpha 4 / 4^l (l < 2), out 12
    algo = H * W * (12 + 12 + sum((16 + (4 if l < 2 else 0)) / 4 ** l for l in range(3)))
    ms = el / steps
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s (Ours MR: 3 levels x sizes {{3,5}} + Eq. 7)", "value": H * W * steps * world / (el / 1e3) / 1e6,
        "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": Wm, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{W}x{H} multi-resolution reconstruction (NEXT row 2)",
                                        "levels": 3, "sizes": sizes},
        "roofline": {"bound": "hbm", "achieved": algo / (ms / 1e3) / 1e9, "peak": measured_peak_hbm()[0],
                     "unit": "GB/s", "frac": algo / (ms / 1e3) / 1e9 / measured_peak_hbm()[0],
                     "algorithmic_bytes_per_launch": algo,
                     "traffic": recorded_traffic(f"{W}x{H} multi-resolution reconstruction (NEXT row 2)"),
                     "note": "4 launches per step on the paper's levels (one 2-level downsample, 3 fused level "
                             "kernels, the Eq. 7 combines in the level epilogues); algorithmic = inputs + output once"},
        "clocks": clk.summary(), "gpu_launches": steps * (4 if kmd.last_kernel() == "v3-tma28-mr-cmb" else 6),
        "paper_context": "Ours MR reconstruction 0.85 ms at 1280x720 on an RTX 2080 Ti (PAPER.md:435)"}),
        flush=True)


def run_bwd(args, rank, world, local):
    """NEXT row 3: backward (dL/dI, dL/dB given dL/dRhat) on a 1080p frame per
    rank per step (weak scaling), CUDA-graph launched like the main mode."""
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    H, W = args.height, args.width
    sizes = [int(x) for x in args.sizes.split(",")]
    M = len(sizes)
    K, Wm, F = args.steps, args.warmup, 2
    frames = [gen.make_inputs(1, H, W, M, frame_offset=rank * F + f, device=dev) for f in range(F)]
    grads = [torch.randn((1, 3, H, W), device=dev) for _ in range(F)]
    gI = [torch.empty((1, M, H, W), device=dev) for _ in range(F)]
    gB = [torch.empty((1, M, H, W), device=dev) for _ in range(F)]
    ws = torch.empty(kmd.backward_workspace_bytes(1, H, W, sizes), dtype=torch.uint8, device=dev)

    def step(s):
        fi = frames[s % F]
        kmd.decode_filter_fuse_backward(fi.radiance, fi.importance, fi.blend, grads[s % F], sizes,
                                        grad_importance=gI[s % F], grad_blend=gB[s % F], workspace=ws)

    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(2 * F):
            step(j)
    reps = max(1, K // (2 * F))
    g.replay()
    torch.cuda.synchronize(dev)
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize(dev)
    barrier(world)
    steps = reps * 2 * F
    el = max_over_ranks(a.elapsed_time(b), world)
    if rank != 0:
        return
    # read radiance 12, importance 4M, logits 4M, grad_out 12; write dL/dI 4M, dL/dB 4M
    algo = H * W * (24 + 16 * M)
    ms = el / steps
    peak = measured_peak_hbm()[0]
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s (backward: dL/dI, dL/dB)", "value": H * W * steps * world / (el / 1e3) / 1e6,
        "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": Wm, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{W}x{H} backward of the fused decoder (NEXT row 3)",
                                        "sizes": sizes},
        "roofline": {"bound": "hbm", "achieved": algo / (ms / 1e3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": algo / (ms / 1e3) / 1e9 / peak,
                     "algorithmic_bytes_per_launch": algo,
                     "traffic": recorded_traffic(f"{W}x{H} backward of the fused decoder (NEXT row 3)"),
                     "kernel": kmd.last_kernel(),
                     "note": f"{kmd.backward_launches_per_call(M)} launches per step (log-sum-exp of the logits, pass A: s_i = a_i / den_i and d_i = G.R_i, pass B: "
                             "transposed box + dL/dI, pass C: dL/dB); algorithmic = inputs + outputs once, the "
                             "(s_i, d_i, L) workspace (8 M + 4 B/px written and read) is not counted"},
        "clocks": clk.summary(), "gpu_launches": steps * kmd.backward_launches_per_call(M)}),
        flush=True)


def run_temporal(args, rank, world, local):
    """NEXT row 4: the temporal accumulation pre-pass (reproject + consistency +
    accumulate) on a 1080p frame per rank per step (weak scaling)."""
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    H, W = args.height, args.width
    K, Wm, F = args.steps, args.warmup, 4
    frames = [gen.make_temporal_inputs(1, H, W, seed=gen.BASE_SEED + 23 + 97 * (rank * F + f), device=dev)
              for f in range(F)]
    accs = [torch.empty((1, 3, H, W), device=dev) for _ in range(F)]
    masks = [torch.empty((1, H, W), device=dev, dtype=torch.uint8) for _ in range(F)]

    def step(s):
        t = frames[s % F]
        kmd.temporal_accumulate(t.cur_rad, t.prev_rad, t.prev_pos, t.prev_nrm, t.prev_valid, t.cur_pos,
                                t.cur_nrm, t.motion, t.pos_tol, accum=accs[s % F], mask=masks[s % F])

    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(2 * F):
            step(j)
    reps = max(1, K // (2 * F))
    g.replay()
    torch.cuda.synchronize(dev)
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize(dev)
    barrier(world)
    steps = reps * 2 * F
    el = max_over_ranks(a.elapsed_time(b), world)
    if rank != 0:
        return
    # current radiance / position / normal 36, motion 8, previous radiance /
    # position / normal 36 + validity 1 (gathered), accum 12 + mask 1
    algo = H * W * 94
    ms = el / steps
    peak = measured_peak_hbm()[0]
    mask_rate = float(masks[0].float().mean())
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s (temporal accumulation pre-pass)",
        "value": H * W * steps * world / (el / 1e3) / 1e6,
        "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": Wm, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{W}x{H} reproject + consistency + EMA (NEXT row 4)",
                                        "history_kept": round(mask_rate, 3),
                                        "l2": f"{F} resident frames of 94 B/px rotate ({F * H * W * 94 / 1e6:.0f} MB > 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": algo / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": algo / (ms / 1e3) / 1e9 / peak, "algorithmic_bytes_per_launch": algo,
                     "traffic": recorded_traffic(f"{W}x{H} reproject + consistency + EMA (NEXT row 4)")},
        "clocks": clk.summary(), "gpu_launches": steps}), flush=True)


def _graph_time_ms(step, n_launch, K, Wm, dev):
    """Mean ms per launch of `step` (CUDA-graph captured, n_launch per graph)."""
    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j in range(n_launch):
            step(j)
    g.replay()
    torch.cuda.synchronize(dev)
    reps = max(1, K // n_launch)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize(dev)
    return a.elapsed_time(b) / (reps * n_launch)


def run_sweep(args, rank, world, local):
    """SURVEY.md §8(d) sweep-M / sweep-k: time per frame vs the number of fused
    sizes (cumulative {3}, {3,5}, ..., {3..13}: the analogue of the paper's
    Fig. 10/11) and vs one kernel size k at M = 1
    (the box-sum kernel is ~flat in k; k > 13 takes the direct v1 kernel)."""
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    H, W, F = args.height, args.width, 3
    K, Wm = max(64, args.steps // 8), max(3, args.warmup)
    peak = measured_peak_hbm()[0]
    rows = []
    with ClockSampler(local) as clk:
        for sizes in [PAPER_SIZES[:m] for m in range(1, 7)] + [[k] for k in (3, 5, 9, 13, 21, 31)]:
            M = len(sizes)
            inp = gen.make_inputs(F, H, W, M, device=dev, with_blend=M > 1)
            out = torch.empty((F, 3, H, W), device=dev)

            def step(s, inp=inp, out=out, sizes=sizes):
                f = s % F
                kmd.decode_filter_fuse(inp.radiance[f:f + 1], inp.importance[f:f + 1],
                                       None if inp.blend is None else inp.blend[f:f + 1], sizes,
                                       out=out[f:f + 1])
            ms = _graph_time_ms(step, 2 * F, K, Wm, dev)
            algo = kmd.algorithmic_bytes(1, H, W, sizes, inp.blend is not None)
            rows.append({"sizes": sizes, "M": M, "us_per_frame": round(ms * 1e3, 2),
                         "mpix_s": round(H * W / (ms / 1e3) / 1e6, 1), "kernel": kmd.last_kernel(),
                         "roofline_frac": round(algo / (ms / 1e3) / 1e9 / peak, 3)})
            del inp, out
    if rank != 0:
        return
    full = rows[5]
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s vs fused sizes (sweep-M) and kernel size (sweep-k)", "value": full["mpix_s"],
        "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": Wm, "ms_per_step": full["us_per_frame"] / 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{W}x{H}: M = 1..6 cumulative paper sizes, then M = 1 with k in 3..31 "
                               "(SURVEY.md §8(d) sweep-M / sweep-k)"},
        "sweep": rows, "clocks": clk.summary(), "gpu_launches": K * len(rows),
        "paper_context": "reconstruction time grows with the number of fused kernels (PAPER.md:472, 654)"}),
        flush=True)


def run_batch(args, rank, world, local):
    """BASELINE.json configs[4]: a batch of --batch (256) 1080p frames sharded
    across the ranks (rank g takes frames [g B / N, (g+1) B / N), one launch per
    rank per step; no data-path collective).  The total batch is fixed as N
    grows: strong scaling of the batch."""
    from paper_2202_05977_b200 import inputs as gen
    from paper_2202_05977_b200 import kmd
    dev = torch.device("cuda", local)
    H, W, Bg = args.height, args.width, args.batch
    f0, f1 = rank * Bg // world, (rank + 1) * Bg // world
    B = f1 - f0
    sizes = [int(x) for x in args.sizes.split(",")]
    M = len(sizes)
    # this rank's shard of the batch resident (global frame ids f0 .. f1-1): generated in chunks
    rad = torch.empty((B, 3, H, W), device=dev)
    imp = torch.empty((B, M, H, W), device=dev)
    bl = torch.empty((B, M, H, W), device=dev) if M > 1 else None
    for c0 in range(0, B, 16):
        n = min(16, B - c0)
        x = gen.make_inputs(n, H, W, M, frame_offset=f0 + c0, device=dev)
        rad[c0:c0 + n], imp[c0:c0 + n] = x.radiance, x.importance
        if bl is not None:
            bl[c0:c0 + n] = x.blend
        del x
    out = torch.empty((B, 3, H, W), device=dev)
    K, Wm = max(3, args.steps // 400), max(3, args.warmup // 4)

    def step(s):
        kmd.decode_filter_fuse(rad, imp, bl, sizes, out=out)

    for s in range(Wm):
        step(s)
    torch.cuda.synchronize(dev)
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        a.record()
        for s in range(K):
            step(s)
        b.record()
        torch.cuda.synchronize(dev)
    barrier(world)
    el_local = a.elapsed_time(b)
    el = max_over_ranks(el_local, world)
    if rank != 0:
        return
    ms = el / K
    algo = kmd.algorithmic_bytes(B, H, W, sizes, bl is not None)
    peak = measured_peak_hbm()[0]
    print(json.dumps({
        "metric": f"{W}x{H} Mpix/s, batch of {Bg} frames sharded over the GPUs", "value": Bg * H * W * K / (el / 1e3) / 1e6,
        "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"batch {Bg} x {W}x{H}, sizes {sizes} (BASELINE.json configs[4])",
                   "global_batch": Bg, "frames_per_rank": B,
                   "resident_gb_per_rank": round((rad.numel() + imp.numel() + out.numel() + (bl.numel() if bl is not None else 0)) * 4 / 1e9, 1),
                   "parallelism": f"frame-parallel x{world} (no data-path collective)",
                   "l2": "inputs of one step >> 126 MB L2"},
        "ms_per_frame": ms / Bg,
        "roofline": {"bound": "hbm", "achieved": algo / (el_local / K / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": algo / (el_local / K / 1e3) / 1e9 / peak, "algorithmic_bytes_per_launch": algo,
                     "traffic": None, "kernel": f"{kmd.last_kernel()} on rank 0's {B} frames"},
        "clocks": clk.summary(), "gpu_launches": K}), flush=True)


def main():
    args = parse()
    rank, world, local = dist_setup()
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif args.mode == "band":
            run_band(args, rank, world, local)
        elif args.mode == "mr":
            run_mr(args, rank, world, local)
        elif args.mode == "bwd":
            run_bwd(args, rank, world, local)
        elif args.mode == "temporal":
            run_temporal(args, rank, world, local)
        elif args.mode == "sweep":
            run_sweep(args, rank, world, local)
        elif args.mode == "batch":
            run_batch(args, rank, world, local)
        else:
            run_kmd(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
