#!/usr/bin/env python
"""WIPES rasterizer benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Metric (BASELINE.json): fwd+bwd iters/s (and render FPS) of the WIPES
rasterizer. A step = one full pass of the hot path over one batch of synthetic
input: preprocess -> count/scan -> duplicate -> radix sort -> tile ranges ->
render forward -> render backward -> preprocess backward (all SURVEY §8(a)
rows), every kernel ours (libwipes.so through the C ABI).

Default workload: configs[1] (C2) — Kodak-shaped 768x512 image, 70k 2D wavelet
primitives, weighted sum (Eq. 4). Under torchrun the same image
is split by tile rows (row r -> rank r mod N) and the
per-primitive gradients are summed by one NCCL all_reduce (strong scaling;
`--replicas` gives every rank its own image instead). The default line also
carries `nvs_c3`: the 3D static NVS batch (C3: 8 x 1080p views, 1M primitives,
alpha blending) with views sharded across the ranks and the gradients
all_reduced — the "1080p 3D" half of BASELINE's metric. `--config c3|c4|c5`
makes any of them the main line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FWD_WORK = {"sum": (9, 2), "alpha": (13, 2)}     # (+FP32, MUFU) per in-ellipse pair
BWD_WORK = {"sum": (48, 3), "alpha": (66, 4)}
CAND_FP32 = 7                                      # FP32 per tile-method candidate test


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="C2 at N > 1: independent images per rank (weak) instead of one image "
                         "sharded by tile rows + gradient all_reduce (default, strong)")
    ap.add_argument("--no-c3", action="store_true",
                    help="skip the C3 (8 x 1080p 3D, view-sharded) sub-record of the default run")
    ap.add_argument("--c3-steps", type=int, default=5)
    ap.add_argument("--grad-chunks", type=int, default=4,
                    help="N > 1: parameter-row buckets of the overlapped gradient all_reduce")
    ap.add_argument("--e2e-sets", type=int, default=None,
                    help="device buffer sets the pipelined e2e loop rotates through (default 3)")
    ap.add_argument("--cpu-pixels", type=int, default=65536)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-fit", action="store_true",
                    help="skip the NEXT-2 fitting-step measurement (2D configs)")
    ap.add_argument("--no-mlp", action="store_true",
                    help="skip the NEXT-4 deformation-MLP measurement")
    ap.add_argument("--mlp-rows", type=int, default=300000,
                    help="rows (primitives x frames) of the NEXT-4 MLP measurement")
    ap.add_argument("--sh", type=int, default=None,
                    help="3D configs: SH colour of this degree (NEXT-3) instead of flat RGB")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise deterministic backward (per-intersection moment slots)")
    ap.add_argument("--tile", type=int, default=16, choices=[8, 16, 32],
                    help="tile size in pixels (16 is the paper's and the default)")
    ap.add_argument("--proj", default="paper", choices=["paper", "exact"],
                    help="3D projection: Eq. 7 as written (default) or NEXT-1 exact z-marginal")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def load_alu_peaks(clk_hz):
    """Render roofline denominators: FP32 and MUFU lane-op rates MEASURED on a
    B200 by tools/peaks.cu (profiles/peaks.json), per SM per clock, times 148
    SMs times the SM clock. Falls back to the unit counts (128 FP32 / 16 MUFU
    lanes per SM per clock) only if the file is missing."""
    p = os.path.join(ROOT, "profiles", "peaks.json")
    sms = 148
    if os.path.exists(p):
        d = json.load(open(p))
        u = d["roofline_use"]
        return (sms * u["fp32_lane_ops_per_sm_clk"] * clk_hz, sms * u["mufu_ops_per_sm_clk"] * clk_hz,
                "measured (profiles/peaks.json: FFMA2 %.1f, MUFU.EX2 %.1f lane-ops/SM/clk)"
                % (u["fp32_lane_ops_per_sm_clk"], u["mufu_ops_per_sm_clk"]))
    return sms * 128 * clk_hz, sms * 16 * clk_hz, "unit counts (profiles/peaks.json missing)"


def hist_bytes(n, passes, cap, rts_tiles=1024, tile=2048):
    """Histogram-side bytes of one sort of n keys (capacity cap) over `passes` digits."""
    tiles = -(-cap // tile)
    if tiles >= rts_tiles:
        return passes * (4 * n + 16 * 256 * tiles)
    return 4 * n


def hbm_fractions(kt, steps, L, hbm_gbs):
    """SURVEY §8(d) gate G2: achieved algorithmic bytes / CUDA-event time of the
    HBM-bound kernel groups against the measured copy bandwidth, per STEP (a
    group may be several launches: camera chunks, sort passes, the ALPHA
    presort's key kernels). L = dict(BN, dup, BT, alpha, B, param_bytes,
    grad_bytes). Sort keys and values are 32-bit: one pass reads and writes
    16 B per element; the ALPHA path first presorts the BN (view, primitive)
    depth keys (4 depth bytes + the view bytes) and then sorts the dup tile
    keys."""
    BN, dup, alpha = L["BN"], L["dup"], L["alpha"]
    vb = 0
    while (1 << vb) < L["B"]:
        vb += 1
    # the presort of a large frame runs segmented by view: 4 depth passes, no view pass
    seg_cap = L["B"] * (-(-(BN // max(L["B"], 1)) // 2048)) * 2048  # B views x whole tiles
    seg = alpha and seg_cap // 2048 >= 1024
    pre = (4 if seg else 4 + (vb + 7) // 8) if alpha else 0
    tb = 0
    while (1 << tb) < L["BT"]:
        tb += 1
    tile_passes = (tb + 7) // 8
    # ALPHA tile sort segmented by view when the view-local tile ids need fewer
    # passes (Layout::tile_seg; cap-based tile bound >= 1024)
    T = L["BT"] // max(L["B"], 1)
    tv = 0
    while (1 << tv) < T:
        tv += 1
    if alpha and L["B"] > 1 and (tv + 7) // 8 < tile_passes and \
            -(-L.get("cap", dup) // 2048) + L["B"] >= 1024:
        tile_passes = (tv + 7) // 8
    per_step = {
        # params read + rect 16, count 4, flag 1, depth 4, record 64 written per (view, prim)
        "preprocess2d": L["param_bytes"] + 89 * BN,
        "preprocess3d": L["param_bytes"] + 89 * BN,
        # rect 16 + offset 8 + count 4 read per (view, prim); key 4 + value 4 per dup;
        # ALPHA also the presort key build (4 in, 8 out) and count gather (8 in, 4 out)
        "duplicate": 28 * BN + 8 * dup + (24 * BN if alpha else 0),
        # onesweep sorts: one read of the keys per sort (all passes' histograms);
        # reduce-then-scan sorts (>= 1024 tiles of 2048 keys, sort.cu): per pass
        # one key read + the digit-major tile counts (4 B written, 4 B read and
        # 8 B written by the flat scan per (digit, tile))
        "radix_hist": sum(hist_bytes(n, p, c) for n, p, c in
                          ((dup, tile_passes, L.get("cap", dup)),) +
                          (((BN, pre, seg_cap if seg else BN),) if alpha else ())),
        # per pass: key + value read and written
        "radix_scatter": 16 * (tile_passes * dup + pre * BN),
        # sorted keys read, CSR offsets written
        "tile_ranges": 4 * dup + 4 * (L["BT"] + 1),
        # moments (48 B / (view, primitive)) + params read, gradients written
        "preprocess2d_bwd": 48 * BN + L["param_bytes"] + L["grad_bytes"],
        "preprocess3d_bwd": 48 * BN + L["param_bytes"] + L["grad_bytes"],
    }
    out = {}
    for k, b in per_step.items():
        if k not in kt or not kt[k][1]:
            continue
        t = kt[k][0] / 1e3 / steps
        gbs = b / t / 1e9
        out[k] = {"bytes_per_step": int(b), "us_per_step": t * 1e6,
                  "launches_per_step": kt[k][1] / steps, "GB/s": gbs, "frac": gbs / hbm_gbs}
    return out


def gpu_local_cpus(dev_index):
    """Host cores on the GPU's NUMA node (sysfs local_cpulist of its PCI
    function): the e2e leg pins its thread there before allocating pinned
    buffers, so H2D/D2H copies use node-local host memory."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(dev_index)
        bus = "%04x:%02x:%02x.0" % (getattr(pr, "pci_domain_id", 0), pr.pci_bus_id,
                                    pr.pci_device_id)
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return bus, sorted(cpus & os.sched_getaffinity(0))
    except Exception:
        return None, []


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(2)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) > 8 for k in range(4)
                          if r[5 + k].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------ CPU ---
def fit_rate(H, W, N, args, flush, dev, params):
    """NEXT-2: full fitting iterations (render -> L2 loss -> backward -> Adam,
    one CUDA graph per iteration, raster.Fitter2D) on the bench frame's own
    primitives (the C2 distribution: the same parameters as the fwd+bwd line,
    opacity taken as given), timed with CUDA events over args.steps replays
    (L2 flushed between)."""
    import torch
    from paper_2508_12615_b200 import gen
    from paper_2508_12615_b200.train import Fitter2D
    tgt = gen.smooth_target(H, W, seed=args.seed)
    fit = Fitter2D(torch.from_numpy(tgt).to(dev), {k: torch.from_numpy(v) for k, v in params.items()},
                   cov2="sigma", opacity_act="none")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush.zero_()
        fit.step()
    torch.cuda.synchronize()
    ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fit.step()
        b.record(stream)
        b.synchronize()
        ms += a.elapsed_time(b)
    loss, over = fit.poll()
    return {"value": args.steps / (ms / 1e3), "unit": "fitting iters/s",
            "ms_per_step": ms / args.steps, "loss": loss, "overflowed": over,
            "steps_applied": fit.steps_taken(),
            "workload": f"NEXT-2 image fit {W}x{H} on the bench frame's {N} primitives (C2 "
                        "distribution), L2 + Adam (preprocess, bin/sort, render, loss, backward, "
                        "Adam: one CUDA graph)"}


def mlp_rate(args, flush, dev, peaks, precision="bf16x3"):
    """NEXT-4: the D-3DGS-shaped deformation field (8 x 256, skip 4, Lx 10,
    Lt 6) forward + backward on the tcgen05 tensor cores for args.mlp_rows
    rows (C4's 300k primitives x 1 frame, one D-3DGS training iteration),
    CUDA-event timed over args.steps iterations (L2 flushed between).
    precision "bf16x3" (default: split-bf16 operands, R38) or "bf16".
    Roofline: the METHOD's FLOPs (the FP32 network's 2 M sum W K per pass,
    forward + backward) over the time against the measured bf16 tensor peak —
    the emulation's own MMA work (3x with bf16x3) is reported beside it; the
    compulsory HBM bytes (parameters in, frame rows out) are ~100 B per row,
    far below the ridge, so the tensor pipe is the bound."""
    import torch
    from paper_2508_12615_b200 import gen
    from paper_2508_12615_b200.deform import Deformation
    N = args.mlp_rows
    d = Deformation(N, precision=precision)
    theta = d.init_theta(seed=args.seed, head_scale=0.1)
    p = gen.gen3d(N, seed=args.seed)
    canon = {k: torch.from_numpy(v).to(dev) for k, v in p.items()}
    frame = d.forward(theta, canon, [0.5])
    g = {k: torch.randn_like(frame[k]) for k in ("mean", "quat", "scale", "freq")}
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush.zero_()
        d.forward(theta, canon, [0.5], frame)
        d.backward(theta, canon, g)
    torch.cuda.synchronize()
    fwd = bwd = 0.0
    for _ in range(args.steps):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        d.forward(theta, canon, [0.5], frame)
        e[1].record(stream)
        d.backward(theta, canon, g)
        e[2].record(stream)
        e[2].synchronize()
        fwd += e[0].elapsed_time(e[1])
        bwd += e[1].elapsed_time(e[2])
    fwd /= args.steps
    bwd /= args.steps
    fl = sum(2 * d.width * d.layer_in(l) for l in range(d.depth)) + 2 * 13 * d.width
    fwd_fl = N * fl
    bwd_fl = N * (2 * fl - 2 * d.width * d.layer_in(0))
    peak = float(peaks.get("bf16_tflops", 1695.0))
    ach = (fwd_fl + bwd_fl) / ((fwd + bwd) / 1e3) / 1e12
    mult = 3 if precision == "bf16x3" else 1
    return {"workload": f"NEXT-4 deformation MLP (D-3DGS 8x256, skip 4, PE 10/6), {N} rows, "
                        f"forward + backward, {precision} operands on tcgen05 GEMMs with fp32 "
                        "accumulation",
            "precision": precision,
            "fwd_ms": fwd, "bwd_ms": bwd, "iters_per_s": 1e3 / (fwd + bwd),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak,
                         "flops": "the method's (FP32 network) 2 M sum(W K) per pass",
                         "mma_tflops_executed": ach * mult,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"},
            "compulsory_bytes_per_row": 4 * (3 + 4 + 3 + 3) * 2}


def host_link(hp, hdl, hg, dp, ddl, dg, s_up, s_down, e2e_ms, reps=10):
    """The lease's host copy path, measured on the e2e buffers: the step's
    uploads alone, its download alone, and both directions together (their
    own streams, as in the e2e pipeline). Context for `e2e`: a step cannot
    finish faster than its copies, and the copy rate differs between leases."""
    import torch

    def timed(up, down):
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s_up)
        b0.record(s_down)
        for _ in range(reps):
            if up:
                with torch.cuda.stream(s_up):
                    dp.copy_(hp, non_blocking=True)
                    ddl.copy_(hdl, non_blocking=True)
            if down:
                with torch.cuda.stream(s_down):
                    hg.copy_(dg, non_blocking=True)
        a1.record(s_up)
        b1.record(s_down)
        torch.cuda.synchronize()
        return max(a0.elapsed_time(a1) if up else 0.0, b0.elapsed_time(b1) if down else 0.0) / reps
    up_b = (hp.numel() + hdl.numel()) * 4
    dn_b = hg.numel() * 4
    t_up, t_dn, t_both = timed(True, False), timed(False, True), timed(True, True)
    return {"h2d_GBps": up_b / t_up / 1e6, "d2h_GBps": dn_b / t_dn / 1e6,
            "both_ms_per_step": t_both, "e2e_ms_per_step": e2e_ms,
            "note": "the step's uploads and download alone and together on this lease; "
                    "e2e per step >= both_ms_per_step"}


def sharding(name, world, args):
    """(rows, frames, shared) of a config at this world size."""
    from paper_2508_12615_b200 import gen
    base = gen.CONFIGS[name]
    # one image, tile rows sharded: C5 always; C2 (the default) at N > 1 unless
    # --replicas, so that N = 1 is BENCH's workload and N > 1 splits the same image
    rows = base.get("shard") == "rows" or (name == "c2" and world > 1 and not args.replicas)
    frames = base["kind"] == "6d"                 # per-frame parameter rows (view_stride = N)
    shared = base["kind"] == "3d" or rows or frames  # one problem shared by all ranks
    return rows, frames, shared


def workload_config(name, c, world, args):
    """The `config` dict of the JSON line — identical in both arms (ours and
    --impl reference) for the same command line."""
    rows, frames, shared = sharding(name, world, args)
    return {"workload": f"{name}: {c['desc']}"
                        + (" (exact z-integration)" if args.proj == "exact" and c["kind"] != "2d" else "")
                        + (f" (SH degree {c['sh_degree']} colour)" if c.get("sh_degree") is not None else "")
                        + (" (deterministic backward)" if args.deterministic else ""),
            "H": c["H"], "W": c["W"], "N": c["N"], "views": c.get("B", 1), "blend": c["blend"],
            "l2": "flushed between timed steps (256 MiB write, untimed)",
            "parallelism": (f"tile rows r = rank (mod {world}) of one image per GPU + "
                            "NCCL all_reduce of per-primitive gradients") if rows else
                           (f"frames round-robin over {world} GPU(s), per-frame "
                            "parameters disjoint: no exchange") if frames else
                           (f"views sharded over {world} GPU(s) + NCCL all_reduce of "
                            "per-primitive gradients (row buckets overlapping the preprocess "
                            "backward)") if shared else
                           f"replicas: {world} independent image(s), one per GPU"}


def nvs_subrecord(args, rank, world, dev, flush):
    """The "1080p 3D" half of BASELINE's metric, reported beside the default C2
    line: C3 (8 x 1920x1080 views, 1M 3D primitives, alpha blending, SURVEY
    §8(d)) with the views sharded round-robin over the ranks and the
    per-primitive gradients summed by one NCCL all_reduce; each
    step = every rank's frame (CUDA-graph replay) + the all_reduce, CUDA-event
    timed, max over ranks, L2 flushed between steps."""
    import torch
    import torch.distributed as dist
    from paper_2508_12615_b200 import gen
    from paper_2508_12615_b200 import dist as wdist
    from paper_2508_12615_b200.raster import FrameGraph, Rasterizer
    c = gen.make_config("c3", seed=args.seed)
    views = wdist.shard_views(c["B"], rank, world)
    cams = [c["cams"][v] for v in views]
    r = Rasterizer(c["W"], c["H"], prim="3d", blend="alpha", device=dev)
    params = {k: torch.from_numpy(v).to(dev) for k, v in c["params"].items()}
    dL = torch.from_numpy(gen.gen_dLdC(len(cams), c["H"], c["W"], seed=args.seed + rank)).to(dev)
    grads = {k: torch.empty_like(v) for k, v in params.items()}
    bucket = wdist.GradBucket(grads) if world > 1 else None
    ov = wdist.OverlappedReduce(bucket) if bucket is not None else None
    fg = FrameGraph(r, params, cams, 0, dL, grads)
    stream = torch.cuda.current_stream()

    def one_step():
        fg.forward()
        if ov is None:
            fg.backward()
        else:  # bucketed all_reduce overlapping the chunked preprocess backward
            r.backward(dL, grads, row_chunks=args.grad_chunks, on_rows=ov.on_rows)
            ov.finish()

    for _ in range(3):
        flush.zero_()
        one_step()
    torch.cuda.synchronize()
    tot = red = 0.0
    for _ in range(args.c3_steps):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        if world > 1:
            dist.barrier()
        e[0].record(stream)
        fg.forward()
        e[1].record(stream)
        if ov is None:
            fg.backward()
        else:
            r.backward(dL, grads, row_chunks=args.grad_chunks, on_rows=ov.on_rows)
            ov.finish()
        e[2].record(stream)
        e[2].synchronize()
        tot += e[0].elapsed_time(e[2])
        red += e[1].elapsed_time(e[2])
    t = torch.tensor([tot, red], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n, over = r.check_overflow()
    assert not over
    ms = float(t[0]) / args.c3_steps
    out = {"workload": f"c3: {c['desc']}", "value": 1e3 / ms, "unit": "iters/s",
           "render_fps": c["B"] * 1e3 / ms, "ms_per_step": ms,
           "bwd_and_allreduce_ms": float(t[1]) / args.c3_steps, "steps": args.c3_steps,
           "views_per_rank": len(views), "dup": int(n),
           "grad_bytes": sum(v.numel() * 4 for v in grads.values()),
           "parallelism": f"views round-robin over {world} GPU(s) + NCCL all_reduce of the "
                          f"per-primitive gradients in {args.grad_chunks} row buckets, each "
                          "overlapping the next bucket's preprocess backward",
           "scaling": "strong"}
    del fg, r, params, grads, bucket
    torch.cuda.empty_cache()
    return out


def cpu_oracle_sample(c, npix, seed):
    """The oracle as it stands (double-precision brute force over ALL primitives
    per pixel, no tiling) on a bounded random pixel sample of the workload;
    returns (seconds for the sample, extrapolation factor, cores)."""
    import oracle
    H, W, B = c["H"], c["W"], c.get("B", 1)
    rng = np.random.default_rng(seed)
    npix = min(npix, B * H * W)
    pix = np.sort(rng.choice(B * H * W, npix, replace=False))
    dL = rng.uniform(-1, 1, (npix, 3))
    kind = c["kind"]
    cfg = oracle.Cfg(width=W, height=H, prim3d=kind != "2d", alpha_blend=c["blend"] == "alpha",
                     dilation=float(np.float32(0.3)) if kind != "2d" else 0.0)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.forward_backward(cfg, c["params"], dL, cams=c.get("cams"),
                            view_stride=c.get("view_stride", 0), pix=pix, nthreads=cores)
    dt = time.perf_counter() - t0
    return dt, (B * H * W) / npix, cores


def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host
    cores, same config/metric/unit; each step is a bounded pixel sample of the
    workload, extrapolated to the full frame."""
    if rank != 0:
        return
    from paper_2508_12615_b200 import gen
    c = gen.make_config(args.config, seed=args.seed)
    per = max(64, args.cpu_pixels // 8)
    times = []
    cores = os.cpu_count() or 1
    for s in range(args.warmup + args.steps):
        dt, fac, cores = cpu_oracle_sample(c, per, seed=1000 + s)
        if s >= args.warmup:
            times.append(dt * fac)
    ms = 1e3 * statistics.mean(times)
    value = 1e3 / ms
    sample = (f"{per} random pixels of {c['B'] if 'B' in c else 1}x{c['H']}x{c['W']} per step, "
              f"fwd+bwd against all {c['N']} primitives, extrapolated linearly to the full frame")
    line = {"impl": "reference", "metric": "fwd+bwd iters/s", "value": value, "unit": "iters/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if sharding(args.config, world, args)[2] else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args.config, c, world, args),
            "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU ---
def main():
    args = parse()
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist
    if world > 1:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend)
        # the process group must report every rank the launcher started
        if dist.get_world_size() != world:
            raise RuntimeError(f"{backend} reports {dist.get_world_size()} ranks, WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2508_12615_b200 import abi, build, gen, hostmem
    from paper_2508_12615_b200.raster import FrameGraph, Rasterizer
    from paper_2508_12615_b200 import dist as wdist
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks, peak_src = load_peaks()

    name = args.config
    rows, frames, shared = sharding(name, world, args)
    # 2D (C2): one image, tile rows sharded + gradient all_reduce at N > 1
    # (--replicas: every rank its own independent image, weak scaling);
    # 3D batch (C3): one scene, views sharded across ranks + gradient all_reduce;
    # 6D (C4): frames sharded round-robin, per-frame parameters are disjoint so
    # there is no exchange; C5: tile rows sharded + all_reduce.
    over = {"sh_degree": args.sh} if (args.sh is not None and gen.CONFIGS[name]["kind"] != "2d") else {}
    c = gen.make_config(name, seed=args.seed + (0 if shared else rank), **over)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    blend = c["blend"]
    cams = c["cams"]
    vs = c["view_stride"]
    my_views = list(range(rank, B, world)) if (shared and not rows) else None
    if my_views is not None:
        cams = [cams[v] for v in my_views]
    Bl = len(cams) if cams is not None else 1
    r = Rasterizer(W, H, prim="2d" if c["kind"] == "2d" else "3d", blend=blend, device=dev,
                   tile=args.tile, proj=args.proj if c["kind"] != "2d" else "paper",
                   sh_degree=c.get("sh_degree"),
                   row_mod=world if (rows and world > 1) else 0, row_rem=rank if rows else 0,
                   deterministic=int(args.deterministic))
    hp = c["params"]
    if frames and world > 1:  # this rank's frames' parameter rows (view_stride = N)
        hp = {k: np.ascontiguousarray(np.concatenate(
            [v[f * N:(f + 1) * N] for f in my_views], 0)) for k, v in hp.items()}
        c = dict(c, params=hp)
    params = {k: torch.from_numpy(v).to(dev) for k, v in hp.items()}
    dL_host = gen.gen_dLdC(Bl, H, W, seed=args.seed + rank)
    dL = torch.from_numpy(dL_host).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    grads = {k: torch.empty_like(v) for k, v in params.items() if k not in ("depth",)}
    flat = None
    if shared and world > 1 and not frames:
        flat = wdist.GradBucket(grads, deterministic=args.deterministic)

    def step_eager(sync=False):
        r.preprocess(params, cams, vs, sync=sync)
        r.bin_sort()
        r.render(*(r._saved if r._saved is not None else (None, None, None)))
        r.backward(dL, grads)
        if flat is not None:
            flat.all_reduce()

    # one synced step sizes the workspace; then the frame is captured as CUDA
    # graphs (public API: raster.FrameGraph) — the timed steps replay them
    step_eager(sync=True)
    l0 = abi.launch_count()
    fg = FrameGraph(r, params, cams, vs, dL, grads)
    kernels_per_step = None

    # multi-rank with a large gradient exchange (3D views, 4K rows): the all_reduce
    # in row buckets overlapping the chunked preprocess backward; C2's 3.4 MB
    # bucket stays one all_reduce after the captured backward graph
    ov = wdist.OverlappedReduce(flat) if (flat is not None and name != "c2") else None

    def step(ev0=None, ev1=None, ev2=None):
        if ev0 is not None:
            ev0.record(stream)
        fg.forward()
        if ev1 is not None:
            ev1.record(stream)
        if ov is not None:
            r.backward(dL, grads, row_chunks=args.grad_chunks, on_rows=ov.on_rows)
            ov.finish()
        else:
            fg.backward()
            if flat is not None:
                flat.all_reduce()
        if ev2 is not None:
            ev2.record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    n_tot, over = r.check_overflow()
    assert not over, "capacity overflow"

    sampler = ClockSampler(local)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    for k in range(args.steps):
        flush.zero_()
        step(*evs[k])
    torch.cuda.synchronize()
    # per-kernel CUDA-event timing (same kernels, eager launches on the same
    # stream, inside the clock-sampled window): roofline numerator + breakdown
    nk = max(3, min(args.steps, 10))
    abi.timing_enable(True)
    l1 = abi.launch_count()
    for k in range(nk):
        flush.zero_()
        step_eager()
    torch.cuda.synchronize()
    kernels_per_step = (abi.launch_count() - l1) / nk
    abi.timing_enable(False)
    kt = abi.timing_collect()
    kt = {k: (v[0] / nk * args.steps, v[1] / nk * args.steps) for k, v in kt.items()}
    launches = int(round(kernels_per_step * args.steps))
    clocks = sampler.stop()
    n_tot2, over = r.check_overflow()
    assert not over
    fwd_ms = [a.elapsed_time(b) for a, b, _ in evs]
    tot_ms = [a.elapsed_time(c_) for a, _, c_ in evs]
    my_total = sum(tot_ms)
    my_fwd = sum(fwd_ms)
    t = torch.tensor([my_total, my_fwd], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, total_fwd_ms = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    units = world * args.steps if not shared else args.steps   # iterations (problems) processed
    value = units / (total_ms / 1e3)
    render_fps = (world * args.steps * Bl if not shared else args.steps * B) / (total_fwd_ms / 1e3)
    if rows:
        render_fps = args.steps / (total_fwd_ms / 1e3)

    # ---- e2e: same metric through the public API with HOST buffers --------
    bus, local_cpus = gpu_local_cpus(local)
    saved_aff = os.sched_getaffinity(0)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    # page-locked in place after a first touch on this thread (hostmem.py: torch's
    # pin_memory() buffers uploaded at 10-21 GB/s on some leases, these at ~53)
    host_params = {k: torch.from_numpy(v) for k, v in c["params"].items()}
    host_dL = hostmem.pinned_empty(dL_host.shape)
    host_dL.copy_(torch.from_numpy(dL_host))
    host_grads = {k: torch.empty(v.shape, dtype=torch.float32) for k, v in grads.items()}
    h2d = sum(v.numel() * 4 for v in host_params.values()) + host_dL.numel() * 4
    d2h = sum(v.numel() * 4 for v in host_grads.values())
    n_e2e = max(50, args.steps)  # at least 50 pipelined steps: host enqueue jitter averages out
    exchange = flat is not None  # multi-rank step with a gradient sum
    # Pipelined through the public API: two device buffer sets, each with its
    # captured frame; step k uploads its inputs on a copy stream while step
    # k - 1 computes, and its gradients come back on the copy stream. Each
    # set's parameter groups (and gradient groups) are views of one flat
    # buffer, as a training loop would keep them, so a step is one upload of
    # the parameters, one of dL/dC and one download of the gradients.
    def flat_views(shapes, device, pin=False):
        sizes = {k: int(np.prod(sh)) for k, sh in shapes.items()}
        offs, o = {}, 0
        for k, n in sizes.items():
            offs[k] = o
            o += (n + 3) // 4 * 4  # 16-byte aligned groups
        buf = (hostmem.pinned_empty((o,)) if pin
               else torch.zeros(o, dtype=torch.float32, device=device))
        return buf, {k: buf[offs[k]:offs[k] + sizes[k]].view(shapes[k]) for k in shapes}

    pshapes = {k: tuple(v.shape) for k, v in host_params.items()}
    gshapes = {k: tuple(v.shape) for k, v in grads.items()}
    host_pflat, hp = flat_views(pshapes, "cpu", pin=True)
    for kk, v in host_params.items():
        hp[kk].copy_(v)
    sets, gflats = [], []
    # three sets: step k+1's upload no longer waits for step k-1's download
    # (C5 e2e 180 -> 219 iters/s, C4 11.3 -> 14.1; C2/C3 unchanged)
    nsets = max(2, args.e2e_sets or 3)
    for _ in range(nsets):
        pflat, pv = flat_views(pshapes, dev)
        pflat.copy_(host_pflat)
        dLb = torch.empty_like(dL)
        dLb.copy_(dL)
        gflat, gv = flat_views(gshapes, dev)
        sets.append((pflat, dLb, FrameGraph(r, pv, cams, vs, dLb, gv)))
        gflats.append(gflat)
    host_g = [flat_views(gshapes, "cpu", pin=True)[0] for _ in range(nsets)]
    h2d = host_pflat.numel() * 4 + host_dL.numel() * 4
    d2h = host_g[0].numel() * 4
    s_copy, s_comp, s_back = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    s_comm = torch.cuda.Stream() if exchange else s_comp
    up = [torch.cuda.Event() for _ in range(nsets)]
    comp = [torch.cuda.Event() for _ in range(nsets)]
    done = [torch.cuda.Event() for _ in range(nsets)]
    def pipeline(n):
        for k in range(n):
            b = k % nsets
            pb, dlb, fgb = sets[b]
            with torch.cuda.stream(s_copy):
                if k >= nsets:
                    s_copy.wait_event(done[b])
                pb.copy_(host_pflat, non_blocking=True)
                dlb.copy_(host_dL, non_blocking=True)
                up[b].record(s_copy)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(up[b])
                fgb.forward()
                fgb.backward()
                comp[b].record(s_comp)
            if exchange:  # the gradient sum across ranks on its own stream: it overlaps
                with torch.cuda.stream(s_comm):  # the next step's frame (other buffer set)
                    s_comm.wait_event(comp[b])
                    wdist.reduce_flat(gflats[b], deterministic=args.deterministic)
                    comp[b].record(s_comm)
            with torch.cuda.stream(s_back):  # D2H on its own stream: uploads never queue behind it
                s_back.wait_event(comp[b])
                host_g[b].copy_(gflats[b], non_blocking=True)
                done[b].record(s_back)
        s_copy.wait_stream(s_back)

    # untimed warm-up of the copy path, at least 0.1 s of it: right after the
    # device-only phases the first uploads ran at ~21 GB/s and only then at ~50
    # (tools/h2d_probe.py: 20 x 7.8 MB at 20.8 GB/s, the next 20 at 49.2 GB/s)
    # (a step count, not a deadline, so every rank issues the same collectives)
    est_ms = max(ms_per_step, h2d / 20e6)  # the step, or its upload at the slow rate
    n_w = torch.tensor([max(3, args.warmup, math.ceil(100.0 / est_ms))], device=dev)
    if world > 1:
        dist.all_reduce(n_w, op=dist.ReduceOp.MAX)
    pipeline(int(n_w.item()))
    torch.cuda.synchronize()
    flush.zero_()
    torch.cuda.synchronize()
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_copy)
    t_host = time.perf_counter()
    pipeline(n_e2e)
    t_host = time.perf_counter() - t_host
    b_.record(s_copy)
    b_.synchronize()
    e2e_total = a.elapsed_time(b_)
    print(f"e2e: host enqueue {1e3 * t_host / n_e2e:.3f} ms/step, device {e2e_total / n_e2e:.3f} "
          f"ms/step over {n_e2e} steps, {nsets} buffer sets", file=sys.stderr)
    e2e_mode = ("pipelined: step k+1's inputs uploaded (H2D stream) and step k-1's "
                "gradients downloaded (D2H stream) while step k computes"
                + (" (its gradient all_reduce on the compute stream)" if exchange else ""))
    link = host_link(host_pflat, host_dL, host_g[0], sets[0][0], sets[0][1], gflats[0],
                     s_copy, s_back, e2e_total / n_e2e)
    os.sched_setaffinity(0, saved_aff)
    te = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = (world if not shared else 1) * n_e2e / (float(te[0]) / 1e3)

    # ---- roofline of the dominant render kernel -----------------------------
    n_cand, n_ell, n_con = r.render_stats()
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    p32, psfu, alu_src = load_alu_peaks(clk)
    fwd_t = kt["render_fwd"][0] / max(kt["render_fwd"][1], 1) / 1e3
    bwd_t = kt["render_bwd"][0] / max(kt["render_bwd"][1], 1) / 1e3
    dom = "render_bwd" if kt["render_bwd"][0] >= kt["render_fwd"][0] else "render_fwd"
    E, m = (BWD_WORK if dom == "render_bwd" else FWD_WORK)[blend]
    tdom = bwd_t if dom == "render_bwd" else fwd_t
    launches_dom = kt[dom][1] / args.steps
    work32 = (CAND_FP32 * n_cand + E * n_ell) / launches_dom if launches_dom else 0
    worksfu = m * n_ell / launches_dom if launches_dom else 0
    f32frac = work32 / tdom / p32 if tdom else 0
    sfufrac = worksfu / tdom / psfu if tdom else 0
    pipe = "fp32" if f32frac >= sfufrac else "mufu"
    useful32 = (CAND_FP32 + E) * n_ell / max(launches_dom, 1)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{name}:{dom}")
    roof = {"bound": "alu", "kernel": dom, "pipe": pipe,
            "achieved": (work32 if pipe == "fp32" else worksfu) / tdom / 1e9,
            "peak": (p32 if pipe == "fp32" else psfu) / 1e9,
            "unit": f"G{pipe} instr/s (tile-method algorithmic work; peak {alu_src} x 148 SMs x "
                    f"{clk / 1e6:.0f} MHz)",
            "frac": max(f32frac, sfufrac), "frac_fp32": f32frac, "frac_mufu": sfufrac,
            "frac_useful_fp32": useful32 / tdom / p32 if tdom else 0,
            "kernel_ms": tdom * 1e3, "traffic": traffic,
            "pairs": {"tile_candidates": n_cand, "in_ellipse": n_ell, "contributing": n_con}}

    line = {"metric": "fwd+bwd iters/s", "value": value, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if shared else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(name, c, world, args),
            "dup": int(n_tot2),
            "render_fps": render_fps,
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "mode": e2e_mode, "host_link": link,
                    "host_cpus": f"{len(local_cpus)} cores local to GPU {bus}" if local_cpus
                                 else "no NUMA pinning (sysfs unavailable)"},
            "gpu_launches": int(launches), "cuda_graph": True,
            "process_group": ({"backend": dist.get_backend(), "ranks": dist.get_world_size()}
                              if world > 1 else None),
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items() if v[1]},
            "roofline": roof,
            "hbm_kernels": hbm_fractions(
                kt, args.steps,
                dict(BN=Bl * N, dup=int(n_tot2), cap=int(r.cap),
                     BT=Bl * (-(-W // args.tile)) * (-(-H // args.tile)),
                     alpha=blend == "alpha", B=Bl,
                     param_bytes=sum(v.numel() * 4 for v in params.values()),
                     grad_bytes=sum(v.numel() * 4 for v in grads.values())),
                float(peaks.get("hbm_gbs", 6450.9))),
            "paper_context": "render FPS on one A6000: Kodak 1708-1779 (Table 1, PAPER.md:148-149); "
                             "Mip-NeRF360 95.7 (Table 2, PAPER.md:239)"}
    if c["kind"] == "2d" and not rows and not args.no_fit:
        line["fit"] = fit_rate(H, W, N, args, flush, dev, c["params"])
    if name == "c2" and not args.no_c3:
        line["nvs_c3"] = nvs_subrecord(args, rank, world, dev, flush)
    if not args.no_mlp and (c["kind"] == "6d" or name == "c2"):
        line["mlp"] = mlp_rate(args, flush, dev, peaks)
        line["mlp_bf16"] = mlp_rate(args, flush, dev, peaks, precision="bf16")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, fac, cores = cpu_oracle_sample(c, args.cpu_pixels, seed=123)
        line["cpu_baseline"] = {"value": 1.0 / (dt * fac), "unit": "iters/s", "cores": cores,
                                "kind": "oracle",
                                "sample": f"{args.cpu_pixels} random pixels, fwd+bwd against all "
                                          f"{N} primitives ({dt:.1f} s), extrapolated x{fac:.0f} "
                                          "to the full frame"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
